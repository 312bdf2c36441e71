#!/bin/bash
# C2 mkFlags scan: one full ncu capture (k_scan<.., EpiSegStarts>) in the bench's own step
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_scan -s 4 -c 1 -o gpurun_out/ncu_mkflags python bench.py --config c2 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_mkflags.log 2>&1
ncu -i gpurun_out/ncu_mkflags.ncu-rep --page raw --csv > gpurun_out/ncu_mkflags_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_mkflags.ncu-rep --page source --csv > gpurun_out/ncu_mkflags_src.csv 2>/dev/null
rm -f gpurun_out/ncu_mkflags.ncu-rep
tail -2 gpurun_out/ncu_mkflags.log
