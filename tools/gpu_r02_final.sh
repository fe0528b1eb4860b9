#!/bin/bash
# full GPU suite + smoke + default bench (cfg3 + cfg4 side line) + reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x --durations=8 2>&1 | tail -20 > gpurun_out/fin_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/fin_bench.txt 2> gpurun_out/fin_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/fin_bench_ref.txt 2>&1
