#!/bin/bash
# local_cols direct / hashed loops: parity + bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heavy.py tests/test_gpu_random.py tests/test_gpu_graphs.py -q -m gpu -x 2>&1 | tail -4 > gpurun_out/bn_pytest.txt
for v in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --steps 10 > gpurun_out/bn_bench_$v.txt 2>&1
  python -c "
import json
for l in open('gpurun_out/bn_bench_$v.txt'):
    if l.startswith('{'):
        j=json.loads(l); c=j['other_configs']['cfg4']; print('run $v', round(j['ms_per_step'],3), j['parity']['equal'], j['whole_step']['stages_ms'], 'cfg4', round(c['ms_per_step'],3), c['parity']['equal'], c['stages_ms'])
" >> gpurun_out/bn_summary.txt
done
