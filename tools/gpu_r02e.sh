#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_stream.py -q -m gpu -x --durations=4 2>&1 | tail -8 > gpurun_out/r02e_pytest.txt
nvidia-smi --query-gpu=memory.total --format=csv >> gpurun_out/r02e_pytest.txt
timeout 600 python bench.py --config cfg5 --log2n 32 --no-cpu --steps 2 > gpurun_out/r02e_cfg5_32.json 2>&1
