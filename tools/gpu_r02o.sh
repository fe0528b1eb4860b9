#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_merge.py tests/test_gpu_stream.py -q -m gpu -x 2>&1 | tail -5 > gpurun_out/r02o_pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"merge_add" -c 2 -o gpurun_out/prof_merge2 python tools/merge_target.py 27 > gpurun_out/prof_merge2.log 2>&1
ncu -i gpurun_out/prof_merge2.ncu-rep --page raw --csv > gpurun_out/prof_merge2.raw.csv 2>/dev/null
rm -f gpurun_out/prof_merge2.ncu-rep
