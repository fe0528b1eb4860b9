#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heavy.py tests/test_gpu_full_size.py tests/test_gpu_stream.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/az_pytest.txt
for v in 0 1 0 1; do NMX_COUNT23=$v timeout 300 python tools/quick_bench.py 30 2>&1 | sed "s/^/c23=$v /" >> gpurun_out/az_quick.txt; done
