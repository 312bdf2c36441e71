echo "== big filter"; IXG_TILE=24576 IXGPU_LIB=paper_2506_23058_b200/libixgpu_tr.so python tools/trace_filter.py filter 28
python tools/prof_run.py filter 28 2 && ncu --set full --clock-control none --import-source on -k regex:"k_filter_b" -s 1 -c 1 -o gpurun_out/filter_b python tools/prof_run.py filter 28 2 > gpurun_out/ncu1.log 2>&1
python tools/prof_run.py c2 28 2 && ncu --set full --clock-control none --import-source on -k regex:"k_segsum_b" -s 1 -c 1 -o gpurun_out/segsum_b python tools/prof_run.py c2 28 2 > gpurun_out/ncu2.log 2>&1
echo profiled
