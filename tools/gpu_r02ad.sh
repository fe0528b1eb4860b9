#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ad_launches.csv python tools/coo_target.py 28 1 > gpurun_out/ad_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"local_sort" -c 1 -o gpurun_out/prof_sort python tools/coo_target.py 28 1 > gpurun_out/ad_ncu2.log 2>&1
python tools/src_lines.py gpurun_out/prof_sort.ncu-rep local_sort 30 > gpurun_out/ad_src_sort.txt 2>&1
python tools/smem_lines.py gpurun_out/prof_sort.ncu-rep local_sort 20 > gpurun_out/ad_smem_sort.txt 2>&1
ncu -i gpurun_out/prof_sort.ncu-rep --page raw --csv > gpurun_out/prof_sort.raw.csv 2>/dev/null
rm -f gpurun_out/prof_sort.ncu-rep
