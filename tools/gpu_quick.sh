#!/bin/bash
# Timing-only iteration: bench lines for the given configs (default cfg3), no tests.
TAG=${1:-q}
shift
mkdir -p gpurun_out
for cfg in ${@:-cfg3}; do
  timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 5 2>&1 | tail -1 > gpurun_out/quick_${cfg}_$TAG.txt
  python -c "
import json,sys
d=json.loads(open('gpurun_out/quick_${cfg}_$TAG.txt').read())
print('$cfg', round(d['ms_per_step'],3), d['stats9'], d.get('whole_step',{}).get('stages_ms'))"
done
