#!/bin/bash
# narrowed column items: parity (2^27 cases, 2^30 goldens), A/B of cfg3 / cfg4 with NMX_NARROW=0
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -q -m gpu -x -k "narrowed or large_vs_packed or golden or full" 2>&1 | tail -8 > gpurun_out/bc_pytest.txt
for v in 1 0 1; do
  NMX_NARROW=$v timeout 300 python bench.py --no-e2e --no-cpu --steps 10 > gpurun_out/bc_bench_n$v.txt 2>&1
done
NMX_DEBUG=1 timeout 300 python bench.py --no-e2e --no-cpu --no-side --steps 3 > gpurun_out/bc_debug.txt 2>&1
