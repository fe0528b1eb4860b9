#!/bin/bash
mkdir -p gpurun_out
NMX_DEBUG=1 timeout 900 python bench.py --config cfg5 --steps 1 --warmup 1 --no-cpu > gpurun_out/aj_cfg5_dbg.txt 2> gpurun_out/aj_cfg5_dbg.err
grep -a "stream_parts\|  part" gpurun_out/aj_cfg5_dbg.err | tail -14
