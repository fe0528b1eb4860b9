#!/bin/bash
mkdir -p gpurun_out
NMX_DEBUG=1 timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu > gpurun_out/ai_cfg5_dbg.txt 2> gpurun_out/ai_cfg5_dbg.err
grep -a "stream_parts" gpurun_out/ai_cfg5_dbg.err | tail -9
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 1 --no-cpu > gpurun_out/ai_cfg5.txt 2> gpurun_out/ai_cfg5.err
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/ai_pytest.txt
