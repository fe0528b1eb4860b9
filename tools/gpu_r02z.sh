#!/bin/bash
# full GPU suite + smoke + default bench (cfg3 + cfg4 side line, pipelined e2e) + reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x --durations=8 2>&1 | tail -20 > gpurun_out/z_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/z_bench.txt 2> gpurun_out/z_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/z_bench_ref.txt 2>&1
