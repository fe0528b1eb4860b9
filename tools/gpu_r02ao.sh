#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_stream.py tests/reference_suite -x -q -m gpu 2>&1 | tail -3 > gpurun_out/ao_pytest.txt
timeout 900 python bench.py --no-cpu --no-side > gpurun_out/ao_bench.txt 2> gpurun_out/ao_bench.err
