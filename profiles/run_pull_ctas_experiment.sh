#!/bin/bash
cd $GRAFT_REPO_ROOT
for c in 296 148 74 37; do
  VK_PULL_CTAS_EXPERIMENT=$c timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 12 --warmup 3 > gpurun_out/pull_$c.json 2> gpurun_out/pull_$c.err
  echo "$c $(python -c "import json;d=json.load(open('gpurun_out/pull_$c.json'));print(round(d['value']), round(d['ms_per_step'],2), round(d['roofline']['ms_per_launch'],2), round(d['sampler']['ms_per_wave'],2))")"
done
