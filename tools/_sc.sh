timeout 600 python -m pytest tests -q -m gpu -x -k "scatter or c3 or executor" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
B="python bench.py --config c3 --steps 5 --warmup 3"
timeout 600 $B > gpurun_out/c3_new.json 2>gpurun_out/c3_new.err; echo "bench rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_scatter_t -c 1 -o gpurun_out/scatter_t_full $B --no-cpu > /dev/null 2>&1; echo "ncu rc=$?"
