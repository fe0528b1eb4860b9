#!/bin/bash
# r02u: new batches test + LSD / merge parity, live LSD / merge timings, bench with pipelined e2e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batches.py tests/test_gpu_merge.py tests/test_gpu_parity.py tests/test_gpu_stream.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/u_pytest.txt
timeout 300 python tools/time_paths.py 28 27 > gpurun_out/u_paths.txt 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/u_bench.txt 2> gpurun_out/u_bench.err
