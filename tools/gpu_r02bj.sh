#!/bin/bash
# narrowed column items, tile parent table + cheap decode: parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "narrowed or large_vs_packed" 2>&1 | tail -4 > gpurun_out/bj_pytest.txt
for v in 1 0 1 0; do
  NMX_NARROW=$v timeout 300 python bench.py --no-e2e --no-cpu --steps 10 > gpurun_out/bj_bench_n$v.txt 2>&1
  python -c "
import json
for l in open('gpurun_out/bj_bench_n$v.txt'):
    if l.startswith('{'):
        j=json.loads(l); print('narrow=$v', round(j['ms_per_step'],3), j['parity']['equal'], j['whole_step']['stages_ms'], j.get('other_configs'))
" >> gpurun_out/bj_summary.txt
done
