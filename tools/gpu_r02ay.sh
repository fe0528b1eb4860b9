#!/bin/bash
mkdir -p gpurun_out
NMX_PATH=lsd timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/ay_pytest_lsd.txt
timeout 1500 python -m pytest tests/test_gpu_merge.py tests/test_gpu_anonymize.py tests/test_gpu_random.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/ay_pytest.txt
for v in 0 1; do NMX_PASS_TMA=$v timeout 300 python tools/time_paths.py 28 0 2>&1 | sed "s/^/tma=$v /" >> gpurun_out/ay_lsd.txt; done
NMX_PATH=lsd timeout 600 compute-sanitizer --tool memcheck python tools/profile_target.py 20 reps=1 > gpurun_out/ay_san.txt 2>&1
tail -2 gpurun_out/ay_san.txt
