#!/bin/bash
# source-level ncu capture of the grouping kernels + one scatter + one count pass at 2^30 (cfg3)
mkdir -p gpurun_out
TAG=${1:-r02h}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"local_rows|local_cols|msd_scatter|msd_count2" -c 6 -o gpurun_out/prof_$TAG python tools/profile_target.py 30 > gpurun_out/ncu_log_$TAG.txt 2>&1
tail -3 gpurun_out/ncu_log_$TAG.txt
