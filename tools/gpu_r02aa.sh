#!/bin/bash
# cfg4 anatomy: level plan of the heavy paths + per-kernel launch times of one call
mkdir -p gpurun_out
NMX_DEBUG=1 timeout 300 python tools/profile_target.py 30 powerlaw reps=2 > gpurun_out/aa_debug.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/aa_launches.csv python tools/profile_target.py 30 powerlaw reps=1 > gpurun_out/aa_ncu.log 2>&1
