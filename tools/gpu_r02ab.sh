#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_group.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/ab_pytest.txt
timeout 300 python tools/time_windows.py > gpurun_out/ab_windows.txt 2>&1
timeout 300 python tools/quick_bench.py 23 30 > gpurun_out/ab_quick.txt 2>&1
