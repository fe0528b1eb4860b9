#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/time_paths.py 28 27 > gpurun_out/y_paths.txt 2>&1
timeout 300 python tools/time_windows.py > gpurun_out/y_windows.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"merge_add" -s 1 -c 1 -o gpurun_out/prof_ymerge python tools/merge_target.py 27 > gpurun_out/ncu_ymerge.log 2>&1
python tools/src_lines.py gpurun_out/prof_ymerge.ncu-rep merge_add 30 > gpurun_out/y_src_merge.txt 2>&1
ncu -i gpurun_out/prof_ymerge.ncu-rep --page raw --csv > gpurun_out/prof_ymerge.raw.csv 2>/dev/null
rm -f gpurun_out/prof_ymerge.ncu-rep
