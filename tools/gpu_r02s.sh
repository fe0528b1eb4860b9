#!/bin/bash
# full GPU suite + default bench + reference arm + smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x --durations=12 2>&1 | tail -30 > gpurun_out/r02s_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02s_bench.txt 2> gpurun_out/r02s_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02s_bench_ref.txt 2>&1
