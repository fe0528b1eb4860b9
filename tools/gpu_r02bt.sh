#!/bin/bash
# source-level ncu capture of one cfg3 call after r02bs: six scatters + both grouping kernels
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"local_rows|local_cols|msd_scatter" -c 8 -o gpurun_out/prof_bt python tools/profile_target.py 30 reps=1 > gpurun_out/ncu_log_bt.txt 2>&1
tail -3 gpurun_out/ncu_log_bt.txt
