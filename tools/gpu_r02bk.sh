#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"local_rows|local_cols" -c 2 -o gpurun_out/bk_loc python tools/one_call.py 30 > gpurun_out/bk_ncu.log 2>&1
