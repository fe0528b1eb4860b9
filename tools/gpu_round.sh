#!/bin/bash
# One GPU session: tests, bench (both arms), launch list, one full ncu capture.
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/pytest_gpu_$TAG.txt
cat gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py 2>&1 | tee gpurun_out/bench_$TAG.txt | tail -3
timeout 600 python bench.py --impl reference 2>&1 | tee gpurun_out/bench_ref_$TAG.txt | tail -2
timeout 300 python bench.py --config cfg4 --no-e2e --no-cpu --steps 3 2>&1 | tee gpurun_out/bench_cfg4_$TAG.txt | tail -1
timeout 300 python bench.py --config cfg2 --no-cpu --steps 10 2>&1 | tee gpurun_out/bench_cfg2_$TAG.txt | tail -1
timeout 300 python bench.py --config cfg1 --no-cpu --steps 10 2>&1 | tee gpurun_out/bench_cfg1_$TAG.txt | tail -1
timeout 600 python bench.py --config cfg5 --no-cpu --steps 3 2>&1 | tee gpurun_out/bench_cfg5_$TAG.txt | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"msd_scatter|local_rows|local_cols|msd_count2|msd_hist1" -c 13 -o gpurun_out/prof_$TAG python tools/profile_target.py 30 > gpurun_out/ncu_full_log_$TAG.txt 2>&1
tail -2 gpurun_out/ncu_full_log_$TAG.txt
