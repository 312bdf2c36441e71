# every bench config once (ours), on one GPU
export PYTHONPATH=$PWD
for c in c2 c1 c5 c3 c4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --config c3 --perm random --steps 10 --warmup 3 > gpurun_out/bench_c3r.json 2> gpurun_out/bench_c3r.err; echo "c3r rc=$?"
