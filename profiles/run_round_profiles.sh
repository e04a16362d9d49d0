#!/bin/bash
# Round-2 measurement record (one B200): C4/C3 launch lists of the bench's
# timed waves and ncu --set full captures of the top kernels.
cd ${GRAFT_REPO_ROOT:-.}
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
K='k_bucket|k_small|k_sample|k_prepare|k_gather|k_compact|k_relabel|k_allidx'
timeout 600 ncu --metrics $M --clock-control none -k regex:"$K" -c 60 --csv --log-file gpurun_out/r02_launches_c4.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches_c4.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"$K" -c 60 --csv --log-file gpurun_out/r02_launches_c3.csv \
  python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches_c3.log 2>&1
# full captures: C4 gather + sampler kernels of one steady-state wave (skip warm-up wave 0)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" --launch-skip 20 -c 20 \
  -o gpurun_out/r02_ncu_full_c4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_full_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name-base function -k regex:'^k_gather$' --launch-skip 4 -c 1 \
  -o gpurun_out/r02_ncu_full_c3_gather python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_full_c3.log 2>&1
