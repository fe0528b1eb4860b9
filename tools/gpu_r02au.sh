#!/bin/bash
mkdir -p gpurun_out
for lib in paper_2510_14050_b200/libnmx.so tools/probe/libnmx_mg12.so tools/probe/libnmx_mg16.so; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:merge_add_kernel -c 2 --csv python tools/merge_ab.py $lib 2>/dev/null | grep -E "gpu__time|dram__bytes" | sed "s|^|$lib |" >> gpurun_out/au_merge.txt
done
