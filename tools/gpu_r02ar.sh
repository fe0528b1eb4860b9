#!/bin/bash
# round-2 evidence: ncu launch list of the bench command, per-kernel DRAM traffic of one cfg3 / cfg4 call,
# a full capture of the dominant scatter (level 2) for the roofline traffic
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ar_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-side > gpurun_out/ar_bench_under_ncu.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -o gpurun_out/ar_tr_cfg3 python tools/profile_target.py 30 reps=1 > gpurun_out/ar_tr_cfg3.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -o gpurun_out/ar_tr_cfg4 python tools/profile_target.py 30 powerlaw reps=1 > gpurun_out/ar_tr_cfg4.log 2>&1
python tools/ncu_traffic.py gpurun_out/ar_tr_cfg3.ncu-rep gpurun_out/ar_traffic_cfg3.json 1073741824 1 > /dev/null
python tools/ncu_traffic.py gpurun_out/ar_tr_cfg4.ncu-rep gpurun_out/ar_traffic_cfg4.json 1073741824 1 > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:msd_scatter -s 1 -c 1 -o gpurun_out/ar_scatter python tools/profile_target.py 30 reps=1 > gpurun_out/ar_scatter.log 2>&1
ncu -i gpurun_out/ar_scatter.ncu-rep --page raw --csv > gpurun_out/ar_scatter.raw.csv 2>/dev/null
python tools/ncu_traffic.py gpurun_out/ar_scatter.ncu-rep gpurun_out/ar_traffic_scatter.json 1073741824 1 > /dev/null
rm -f gpurun_out/ar_tr_cfg3.ncu-rep gpurun_out/ar_tr_cfg4.ncu-rep
ls -la gpurun_out/ar_*
