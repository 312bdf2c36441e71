# ncu --set full (source-correlated) of the current fused C2 kernel at 2^28
python tools/prof_run.py c2 28 2 > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_filter_b" -s 1 -c 1 -o gpurun_out/c2_r5 python tools/prof_run.py c2 28 2 > gpurun_out/ncu_r5.log 2>&1; echo c2 rc=$?
