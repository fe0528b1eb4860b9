#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"merge_add|msd_scatter|local_rows|local_cols" -c 12 --csv python tools/merge_target.py 27 > gpurun_out/r02p_merge.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"msd_scatter|local_rows|local_cols|seg_scatter" -c 12 --csv python tools/profile_target.py 30 reps=1 > gpurun_out/r02p_cfg3.csv 2>&1
timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/r02p_cfg3.txt 2>&1
timeout 300 python bench.py --config cfg4 --no-e2e --no-cpu --steps 5 > gpurun_out/r02p_cfg4.txt 2>&1
