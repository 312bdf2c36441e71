CMD="python bench.py --steps 3 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
python tools/prof_run.py c2 28 2 > /dev/null && ncu --set full --clock-control none --import-source on -k regex:"k_filter_b|k_segsum_b" -s 2 -c 2 -o gpurun_out/c2_full python tools/prof_run.py c2 28 2 > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
