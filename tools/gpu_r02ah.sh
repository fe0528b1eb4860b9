#!/bin/bash
mkdir -p gpurun_out
NMX_DEBUG=1 timeout 900 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu > gpurun_out/ah_cfg5.txt 2> gpurun_out/ah_cfg5.err
grep -a "stream_parts" gpurun_out/ah_cfg5.err | tail -8
