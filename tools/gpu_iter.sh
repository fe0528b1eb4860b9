#!/bin/bash
# Quick GPU iteration: new tests first, full GPU suite, then cfg3 / cfg4 bench lines.
TAG=${1:-iter}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu ${TESTS:-} 2>&1 | tail -30 > gpurun_out/pytest_$TAG.txt
cat gpurun_out/pytest_$TAG.txt
for cfg in ${CFGS:-cfg4 cfg3}; do
  timeout 300 python bench.py --config $cfg --no-e2e --no-cpu --steps 3 2>&1 | tail -1 | tee gpurun_out/bench_${cfg}_$TAG.txt
done
