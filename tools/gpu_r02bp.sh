#!/bin/bash
# cfg4 heavy rows: width of the first (source-bit) segmented level, A/B
mkdir -p gpurun_out
for r0 in def 0 3 def 0; do
  if [ $r0 = def ]; then unset NMX_HEAVY_R0; else export NMX_HEAVY_R0=$r0; fi
  timeout 300 python bench.py --config cfg4 --no-e2e --no-cpu --steps 5 > gpurun_out/bp_$r0.txt 2>&1
  python -c "
import json
for l in open('gpurun_out/bp_$r0.txt'):
    if l.startswith('{'):
        j=json.loads(l); print('r0=$r0', round(j['ms_per_step'],3), j['parity']['equal'], j['whole_step']['stages_ms'])
" >> gpurun_out/bp_summary.txt
done
unset NMX_HEAVY_R0
NMX_DEBUG=1 NMX_HEAVY_R0=0 timeout 300 python tools/one_call.py 30 powerlaw > gpurun_out/bp_debug0.txt 2>&1
