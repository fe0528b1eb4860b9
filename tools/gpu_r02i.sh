#!/bin/bash
# r02i: per-call DRAM traffic of cfg3 / cfg4 (metrics only, every kernel of one call),
# merge-add full capture, LSD onesweep full capture at 2^28
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -o gpurun_out/tr_cfg3 python tools/profile_target.py 30 reps=1 > gpurun_out/tr_cfg3.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -o gpurun_out/tr_cfg4 python tools/profile_target.py 30 powerlaw reps=1 > gpurun_out/tr_cfg4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"merge_add|merge_partition" -c 4 -o gpurun_out/prof_merge python tools/merge_target.py 27 > gpurun_out/prof_merge.log 2>&1
NMX_PATH=lsd timeout 900 ncu --set full --clock-control none --import-source on -k regex:"onesweep|hist_kernel|link_row|col_kernel" -c 16 -o gpurun_out/prof_lsd python tools/profile_target.py 28 reps=1 > gpurun_out/prof_lsd.log 2>&1
NMX_PATH=lsd timeout 300 python tools/profile_target.py 28 reps=3 > gpurun_out/lsd_live.txt 2>&1
timeout 300 python tools/profile_target.py 28 reps=3 > gpurun_out/msd_live_28.txt 2>&1
ls -la gpurun_out/*.ncu-rep
for r in tr_cfg3 tr_cfg4 prof_merge prof_lsd; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null; done
ncu -i gpurun_out/prof_lsd.ncu-rep --page source --csv -k regex:onesweep --print-source cuda,sass > gpurun_out/prof_lsd_src.csv 2>/dev/null
python tools/ncu_traffic.py gpurun_out/tr_cfg3.ncu-rep gpurun_out/traffic_cfg3.json 1073741824 1 > /dev/null
python tools/ncu_traffic.py gpurun_out/tr_cfg4.ncu-rep gpurun_out/traffic_cfg4.json 1073741824 1 > /dev/null
rm -f gpurun_out/prof_lsd.ncu-rep gpurun_out/tr_cfg3.ncu-rep gpurun_out/tr_cfg4.ncu-rep
du -sh gpurun_out
