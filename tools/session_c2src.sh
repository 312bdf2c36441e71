#!/bin/bash
# C2 fused kernel: one --set full capture with the source page (stall
# sampling per SASS line), exported to CSV
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_filter_b -s 2 -c 1 -o gpurun_out/ncu_c2src python tools/prof_run.py c2 28 4 > gpurun_out/ncu_c2src.log 2>&1
ncu -i gpurun_out/ncu_c2src.ncu-rep --page source --csv > gpurun_out/ncu_c2src_source.csv 2>/dev/null
ncu -i gpurun_out/ncu_c2src.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu_c2src_cuda.csv 2>/dev/null
rm -f gpurun_out/ncu_c2src.ncu-rep
tail -2 gpurun_out/ncu_c2src.log
