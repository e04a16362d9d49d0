#!/bin/bash
# C4 launch list (one timed wave) for the current build: bash profiles/run_c4_launches.sh <tag>
cd ${GRAFT_REPO_ROOT:-.}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_bucket|k_small|k_sample|k_prepare|k_gather|k_compact|k_relabel|k_allidx' -c 60 --csv \
  --log-file gpurun_out/r02_lb_$1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_lb_$1.log 2>&1
