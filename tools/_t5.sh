python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
python bench.py --config c3 --steps 20 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"; head -c 2500 gpurun_out/bench_c3.json; tail -2 gpurun_out/bench_c3.err
