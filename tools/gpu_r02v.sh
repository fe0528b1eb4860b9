#!/bin/bash
# r02v: onesweep variant sweep (LSD path at 2^28), parity of the LSD path under the best ones
mkdir -p gpurun_out
for v in 5 8 9 10 11 12; do
  NMX_PASS_VARIANT=$v timeout 300 python tools/time_paths.py 28 0 2>&1 | sed "s/^/v$v /" >> gpurun_out/v_sweep.txt
done
for v in 8 10; do
  NMX_PASS_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -x -q -m gpu 2>&1 | tail -2 | sed "s/^/v$v /" >> gpurun_out/v_pytest.txt
done
