#!/bin/bash
# quick iteration: parity tests on the MSD path + bench lines (cfg3, cfg4, cfg2), A/B env toggle
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heavy.py tests/test_gpu_full_size.py -q -m gpu -x 2>&1 | tail -5 > gpurun_out/${TAG}_pytest.txt
for cfg in cfg3 cfg4 cfg2; do
  timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 5 2>&1 | tail -1 > gpurun_out/${TAG}_${cfg}.json
  NMX_LOCROWS_GENERAL=1 timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 5 2>&1 | tail -1 > gpurun_out/${TAG}_${cfg}_general.json
done
