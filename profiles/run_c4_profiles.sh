#!/bin/bash
# C4 (default wave) launch list and ncu --set full capture of one steady-state wave (one B200).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
K='k_bucket|k_small|k_sample|k_prepare|k_gather|k_compact|k_relabel|k_allidx'
timeout 600 ncu --metrics $M --clock-control none -k regex:"$K" -c 60 --csv --log-file gpurun_out/r02_launches_c4.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip 20 -c 20 \
  -o gpurun_out/r02_ncu_full_c4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_full_c4.log 2>&1
