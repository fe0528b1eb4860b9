#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_stream.py -q -m gpu -x --durations=8 2>&1 | tail -25 > gpurun_out/r02d_pytest.txt
