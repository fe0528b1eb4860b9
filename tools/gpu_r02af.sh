#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/quick_bench.py 26 30 > gpurun_out/af_quick.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heavy.py tests/test_gpu_full_size.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/af_pytest.txt
