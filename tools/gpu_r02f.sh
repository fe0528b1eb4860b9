#!/bin/bash
# r02 re-entry: full GPU suite on the restored tree, default bench, reference arm, cfg4/cfg2/cfg1.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x --durations=10 2>&1 | tail -30 > gpurun_out/r02f_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r02f_bench.txt 2> gpurun_out/r02f_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02f_bench_ref.txt 2>&1
timeout 300 python bench.py --config cfg4 --no-e2e --no-cpu --steps 5 > gpurun_out/r02f_cfg4.txt 2>&1
timeout 300 python bench.py --config cfg2 --no-cpu --steps 10 > gpurun_out/r02f_cfg2.txt 2>&1
timeout 300 python bench.py --config cfg1 --no-cpu --steps 10 > gpurun_out/r02f_cfg1.txt 2>&1
