#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_heavy.py tests/test_gpu_parity.py tests/test_gpu_full_size.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/aq_pytest.txt
for cfg in "NMX_SEG_UNIFORM=0" "NMX_SEG_UNIFORM=1" "NMX_SEG_UNIFORM=1 NMX_SEG_R0=0"; do
  env $cfg timeout 300 python tools/quick_bench.py 30 2>&1 | grep "kind=1" | sed "s/^/$cfg /" >> gpurun_out/aq_quick.txt
done
NMX_DEBUG=1 timeout 300 python tools/profile_target.py 30 powerlaw reps=1 2>&1 | grep heavy_rows > gpurun_out/aq_plan.txt
