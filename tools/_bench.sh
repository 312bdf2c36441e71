python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc=$?; cat gpurun_out/bench_c2.json; tail -3 gpurun_out/bench_c2.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo ref rc=$?; cat gpurun_out/bench_ref.json
python bench.py --config c1 --no-cpu > gpurun_out/bench_c1.json 2>&1; echo c1 rc=$?; tail -c 600 gpurun_out/bench_c1.json
python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
