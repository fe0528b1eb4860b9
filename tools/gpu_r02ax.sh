#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_merge.py tests/test_gpu_dropin.py tests/test_gpu_parity.py tests/test_gpu_anonymize.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/ax_pytest.txt
timeout 300 python tools/time_windows.py > gpurun_out/ax_windows.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ax_launches.csv python tools/coo_target.py 28 1 > gpurun_out/ax_ncu.log 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/coo_target.py 20 1 > gpurun_out/ax_san.txt 2>&1
tail -3 gpurun_out/ax_san.txt
