#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_graphs.py tests/test_gpu_group.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/as_pytest.txt
timeout 300 python tools/time_windows.py > gpurun_out/as_windows.txt 2>&1
