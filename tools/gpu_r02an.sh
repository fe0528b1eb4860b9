#!/bin/bash
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python tools/san_parts.py > gpurun_out/an_san.txt 2>&1
head -60 gpurun_out/an_san.txt
