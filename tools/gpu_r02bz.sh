#!/bin/bash
# A/B: u64 scatter levels with high-word 32-bit digit math (new)
mkdir -p gpurun_out
L=paper_2510_14050_b200/libnmx.so
for v in old new old new; do
  cp tools/ab/libnmx_$v.so $L
  timeout 300 python bench.py --no-e2e --no-cpu --steps 10 > gpurun_out/bz_bench_$v.txt 2>&1
  python -c "
import json
for l in open('gpurun_out/bz_bench_$v.txt'):
    if l.startswith('{'):
        j=json.loads(l); c=j['other_configs']['cfg4']; print('$v', round(j['ms_per_step'],3), c.get('stages_ms'), j['parity']['equal'], [round(x['ms'],3) for x in j['roofline']['per_launch']], 'cfg4', round(c['ms_per_step'],3), c['parity']['equal'])
" >> gpurun_out/bz_summary.txt
done
cp tools/ab/libnmx_new.so $L
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py tests/test_gpu_heavy.py tests/test_gpu_random.py tests/test_gpu_graphs.py tests/test_gpu_dropin.py -q -m gpu -x 2>&1 | tail -4 > gpurun_out/bz_pytest.txt
