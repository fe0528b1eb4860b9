#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_group.py tests/reference_suite -q -m gpu -x --durations=10 2>&1 | tail -40 > gpurun_out/r02b_pytest.txt
