#!/bin/bash
mkdir -p gpurun_out
NMX_DEBUG=1 timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu > gpurun_out/am_cfg5_dbg.txt 2> gpurun_out/am_cfg5_dbg.err
grep -a "stream_parts\|  part" gpurun_out/am_cfg5_dbg.err | tail -7
timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_distributed.py tests/test_gpu_group.py tests/test_gpu_full_size.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/am_pytest.txt
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 1 --no-cpu > gpurun_out/am_cfg5.txt 2> gpurun_out/am_cfg5.err
