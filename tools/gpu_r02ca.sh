#!/bin/bash
# final-state evidence: per-kernel DRAM traffic of one cfg3 / cfg4 call, launch list of the bench command
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -o gpurun_out/ca_tr_cfg3 python tools/profile_target.py 30 reps=1 > gpurun_out/ca_tr_cfg3.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -o gpurun_out/ca_tr_cfg4 python tools/profile_target.py 30 powerlaw reps=1 > gpurun_out/ca_tr_cfg4.log 2>&1
python tools/ncu_traffic.py gpurun_out/ca_tr_cfg3.ncu-rep gpurun_out/ca_traffic_cfg3.json 1073741824 1 > gpurun_out/ca_traffic_cfg3.txt
python tools/ncu_traffic.py gpurun_out/ca_tr_cfg4.ncu-rep gpurun_out/ca_traffic_cfg4.json 1073741824 1 > gpurun_out/ca_traffic_cfg4.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ca_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-side > gpurun_out/ca_bench_under_ncu.log 2>&1
rm -f gpurun_out/ca_tr_cfg3.ncu-rep gpurun_out/ca_tr_cfg4.ncu-rep
