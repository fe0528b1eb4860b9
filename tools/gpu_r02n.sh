#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_heavy.py tests/test_gpu_random.py tests/test_gpu_full_size.py -q -m gpu -x 2>&1 | tail -5 > gpurun_out/r02n_pytest.txt
for sb in 8 7 8; do NMX_SEG_BITS=$sb timeout 300 python bench.py --config cfg4 --no-e2e --no-cpu --steps 5 > gpurun_out/r02n_cfg4_sb$sb.txt 2>&1; done
timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/r02n_cfg3.txt 2>&1
