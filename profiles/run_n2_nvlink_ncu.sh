#!/bin/bash
# NVLink counters of the miss exchange: a 2-GPU C3 bench with rank 0 under
# ncu, profiling only k_remote_pull (nvlrx/nvltx bytes) and the gather;
# rank 1 runs unprofiled. usage: bash profiles/run_n2_nvlink_ncu.sh
cd ${GRAFT_REPO_ROOT:-.}
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29577 WORLD_SIZE=2
RANK=1 LOCAL_RANK=1 timeout 900 python bench.py --gpus 2 --config c3 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/r02_nvl_r1.log 2>&1 &
RANK=0 LOCAL_RANK=0 timeout 900 ncu --clock-control none \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:'k_remote_pull' --launch-skip 3 -c 3 --csv --log-file gpurun_out/r02_nvl_r0.csv \
  python bench.py --gpus 2 --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_nvl_r0.log 2>&1
wait
