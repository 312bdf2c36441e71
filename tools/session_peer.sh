#!/bin/bash
# sharded partition2 peer kernel: parity (dist + full-size tests), launch times
# of the one-read dual placement against the two-segment form, and one full
# ncu capture of the dual kernel
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/peer_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/peer_pytest.txt
IXG_PEER_DUAL=0 timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -x -q -k peer >> gpurun_out/peer_pytest.txt 2>&1
echo "pytest (two-segment form) rc=$?" >> gpurun_out/peer_pytest.txt
for d in 3 0; do
  IXG_PEER_DUAL=$d timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_filter_b --csv \
    --log-file gpurun_out/peer_launch_dual$d.csv python tools/prof_run.py peer 28 6 > gpurun_out/peer_ncu_dual$d.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_filter_b -s 2 -c 1 -o gpurun_out/ncu_peer_dual python tools/prof_run.py peer 28 4 > gpurun_out/ncu_peer_full.log 2>&1
ncu -i gpurun_out/ncu_peer_dual.ncu-rep --page raw --csv > gpurun_out/ncu_peer_dual_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_peer_dual.ncu-rep --page source --csv > gpurun_out/ncu_peer_dual_src.csv 2>/dev/null
rm -f gpurun_out/ncu_peer_dual.ncu-rep
tail -3 gpurun_out/peer_pytest.txt
