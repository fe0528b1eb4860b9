#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:part_scatter -s 16 -c 1 -o gpurun_out/prof_part python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu > gpurun_out/al_ncu.log 2>&1
ncu -i gpurun_out/prof_part.ncu-rep --page raw --csv > gpurun_out/prof_part.raw.csv 2>/dev/null
python tools/src_lines.py gpurun_out/prof_part.ncu-rep part_scatter 25 > gpurun_out/al_src.txt 2>&1
rm -f gpurun_out/prof_part.ncu-rep
