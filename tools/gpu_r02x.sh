#!/bin/bash
mkdir -p gpurun_out
for v in 5 3 8 9 7; do
  NMX_PASS_VARIANT=$v timeout 300 python tools/time_paths.py 28 0 2>&1 | sed "s/^/v$v /" >> gpurun_out/x_sweep.txt
done
NMX_PATH=lsd timeout 600 ncu --set full --clock-control none --import-source on -k regex:"onesweep" -s 2 -c 1 -o gpurun_out/prof_xlsd python tools/profile_target.py 28 reps=1 > gpurun_out/ncu_xlsd.log 2>&1
python tools/src_lines.py gpurun_out/prof_xlsd.ncu-rep onesweep 40 > gpurun_out/x_src_onesweep.txt 2>&1
ncu -i gpurun_out/prof_xlsd.ncu-rep --page raw --csv > gpurun_out/prof_xlsd.raw.csv 2>/dev/null
rm -f gpurun_out/prof_xlsd.ncu-rep
