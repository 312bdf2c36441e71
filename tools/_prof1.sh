set -x
python tools/prof_run.py filter 28 2 && ncu --set full --clock-control none --import-source on -k regex:k_filter -s 1 -c 1 -o gpurun_out/filter_lb8 python tools/prof_run.py filter 28 2 > gpurun_out/ncu1.log 2>&1
IXGPU_LIB=paper_2506_23058_b200/libixgpu_lb1.so python tools/prof_run.py filter 28 2 && IXGPU_LIB=paper_2506_23058_b200/libixgpu_lb1.so ncu --set full --clock-control none --import-source on -k regex:k_filter -s 1 -c 1 -o gpurun_out/filter_lb1 python tools/prof_run.py filter 28 2 > gpurun_out/ncu2.log 2>&1
IXGPU_LIB=paper_2506_23058_b200/libixgpu_lb1.so python tools/kbench.py 28 > gpurun_out/kbench_lb1.json 2>&1
tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
