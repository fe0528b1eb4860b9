#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bm_cfg4_launches.csv python tools/one_call.py 30 powerlaw > gpurun_out/bm_cfg4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bm_cfg3_launches.csv python tools/one_call.py 30 > gpurun_out/bm_cfg3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"local_rows|local_cols" -c 2 -o gpurun_out/bm_loc python tools/one_call.py 30 > gpurun_out/bm_ncu.log 2>&1
