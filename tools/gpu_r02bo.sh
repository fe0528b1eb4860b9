#!/bin/bash
# per-kernel DRAM traffic of one cfg3 / cfg4 call (narrowed columns, specialised grouping
# kernels), launch list of the bench command, full capture of the narrowed column levels
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -o gpurun_out/bo_tr_cfg3 python tools/profile_target.py 30 reps=1 > gpurun_out/bo_tr_cfg3.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -o gpurun_out/bo_tr_cfg4 python tools/profile_target.py 30 powerlaw reps=1 > gpurun_out/bo_tr_cfg4.log 2>&1
python tools/ncu_traffic.py gpurun_out/bo_tr_cfg3.ncu-rep gpurun_out/bo_traffic_cfg3.json 1073741824 1 > /dev/null
python tools/ncu_traffic.py gpurun_out/bo_tr_cfg4.ncu-rep gpurun_out/bo_traffic_cfg4.json 1073741824 1 > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bo_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-side > gpurun_out/bo_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"msd_scatter|local_rows|local_cols|count23" -c 10 -o gpurun_out/bo_full python tools/profile_target.py 30 reps=1 > gpurun_out/bo_full.log 2>&1
ncu -i gpurun_out/bo_full.ncu-rep --page raw --csv > gpurun_out/bo_full.raw.csv 2>/dev/null
rm -f gpurun_out/bo_tr_cfg3.ncu-rep gpurun_out/bo_tr_cfg4.ncu-rep
