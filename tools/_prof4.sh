# ncu --set full of the fused C2 kernel and the plain filter kernel (2^28 int32)
python tools/prof_run.py c2 28 2 > /dev/null && python tools/prof_run.py filter 28 2 > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_filter_b" -s 1 -c 1 -o gpurun_out/c2fused_full python tools/prof_run.py c2 28 2 > gpurun_out/ncu_full1.log 2>&1; echo c2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_filter_b" -s 1 -c 1 -o gpurun_out/filter_full python tools/prof_run.py filter 28 2 > gpurun_out/ncu_full2.log 2>&1; echo filter rc=$?
