#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heavy.py tests/test_gpu_full_size.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/bb_pytest.txt
for v in 1 1; do timeout 300 python tools/quick_bench.py 30 2>&1 | sed "s/^/v2 /" >> gpurun_out/bb_quick.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:msd_count23 -c 2 --csv python tools/profile_target.py 30 reps=1 2>/dev/null | grep gpu__time >> gpurun_out/bb_quick.txt
