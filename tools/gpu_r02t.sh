#!/bin/bash
# r02t: source-level ncu of the scatter, grouping kernels (2^30 cfg3) and the LSD pass (2^28)
mkdir -p gpurun_out
timeout 300 python tools/profile_target.py 30 reps=3 > gpurun_out/t_live30.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"local_rows|local_cols|msd_scatter" -c 5 -o gpurun_out/prof_t30 python tools/profile_target.py 30 reps=1 > gpurun_out/ncu_t30.log 2>&1
NMX_PATH=lsd timeout 600 ncu --set full --clock-control none --import-source on -k regex:"onesweep" -c 3 -o gpurun_out/prof_tlsd python tools/profile_target.py 28 reps=1 > gpurun_out/ncu_tlsd.log 2>&1
for r in prof_t30 prof_tlsd; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null; done
for k in local_rows local_cols msd_scatter; do python tools/src_lines.py gpurun_out/prof_t30.ncu-rep $k 60 > gpurun_out/src_$k.txt 2>&1; done
python tools/src_lines.py gpurun_out/prof_tlsd.ncu-rep onesweep 60 > gpurun_out/src_onesweep.txt 2>&1
ncu -i gpurun_out/prof_t30.ncu-rep --page details --csv > gpurun_out/prof_t30.details.csv 2>/dev/null
ncu -i gpurun_out/prof_tlsd.ncu-rep --page details --csv > gpurun_out/prof_tlsd.details.csv 2>/dev/null
du -sh gpurun_out/*
