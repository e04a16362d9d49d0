#!/bin/bash
# 2-GPU bench with rank 0 under ncu (kernel list + NVLink counters of the
# miss exchange); rank 1 runs unprofiled. usage: bash profiles/run_n2_rank0_ncu.sh <tag> [bench args]
cd ${GRAFT_REPO_ROOT:-.}
TAG=$1; shift
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29577 WORLD_SIZE=2
RANK=1 LOCAL_RANK=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/r02_n2_${TAG}_r1.log 2>&1 &
RANK=0 LOCAL_RANK=0 timeout 900 ncu --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum \
  -k regex:'k_remote|k_word_popc|k_scan_u32|k_emit_list|k_gather|k_bucket|k_sample|k_prepare' --launch-skip 200 -c 120 --csv \
  --log-file gpurun_out/r02_n2_${TAG}_r0.csv python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/r02_n2_${TAG}_r0.log 2>&1
wait
