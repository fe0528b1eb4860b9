#!/bin/bash
# quick GPU check of selected test files: tools/gpu_quick2.sh TAG file...
TAG=$1; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest "$@" -q -m gpu -x 2>&1 | tail -25 > gpurun_out/${TAG}_pytest.txt
