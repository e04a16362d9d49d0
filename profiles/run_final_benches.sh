#!/bin/bash
# Round-2 closing bench lines: bash profiles/run_final_benches.sh n1 | n2 | n4
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
case "$1" in
  n1)
    for c in c4 c3 c2 c1; do
      timeout 900 python bench.py --config $c > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err
    done ;;
  n2|n4)
    N=${1#n}
    for c in c4 c3; do
      timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 29533 bench.py --gpus $N --config $c > gpurun_out/final_${c}_n$N.json 2> gpurun_out/final_${c}_n$N.err
    done
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29534 tests/multigpu_parity.py > gpurun_out/final_mg_n$N.log 2>&1 ;;
esac
