# partition2L pipeline: timing, then the per-kernel launch list of one call
timeout 300 python tools/jagged_bench.py 24 > gpurun_out/jagged.json && cat gpurun_out/jagged.json | head -30
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/jg_launches.csv python tools/jagged_bench.py 20 > /dev/null 2>&1; echo ncu rc=$?
