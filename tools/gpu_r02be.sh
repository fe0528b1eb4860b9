#!/bin/bash
mkdir -p gpurun_out
for v in 1 0; do
NMX_NARROW=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:local_cols -c 1 -o gpurun_out/be_lc_n$v python tools/one_call.py 30 > gpurun_out/be_ncu_n$v.log 2>&1
done
NMX_NARROW=1 timeout 600 ncu --set full --clock-control none -k regex:msd_scatter -c 6 -o gpurun_out/be_sc_n1 python tools/one_call.py 30 > gpurun_out/be_ncu_sc.log 2>&1
