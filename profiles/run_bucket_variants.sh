#!/bin/bash
# quick C4 launch lists for bucket-size variants
cd $GRAFT_REPO_ROOT
for cfg in "1024 19" "1024 17" "1024 16" "4096 18"; do
  set -- $cfg
  VK_BUCKET_TARGET=$1 VK_BUCKET_MAXBB=$2 timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_bucket|k_sample|k_prepare|k_gather' -c 60 --csv --log-file gpurun_out/r02_lb_$1_$2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_lb_$1_$2.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_bucket_dedup' -c 4 -o gpurun_out/r02_dedup_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_dedup_full.log 2>&1
