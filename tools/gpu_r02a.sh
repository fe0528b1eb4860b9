#!/bin/bash
# r02 first session: full GPU suite (incl. the 2^30 golden parity), default bench, reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_gpu.txt
nproc >> gpurun_out/r02a_gpu.txt; free -g >> gpurun_out/r02a_gpu.txt
timeout 1800 python -m pytest tests -q -m gpu -x --durations=15 2>&1 | tail -40 > gpurun_out/r02a_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r02a_bench.txt 2> gpurun_out/r02a_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02a_bench_ref.txt 2>&1
