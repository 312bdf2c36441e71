# multi-rank functional runs on one GPU (gloo for the host-side exchanges) + the full bench set
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider > gpurun_out/pytest_dist.txt 2>&1; tail -3 gpurun_out/pytest_dist.txt
for c in c5 c2; do
  IXG_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --config $c --quick --steps 3 --warmup 3 > gpurun_out/bench_${c}_2r.json 2> gpurun_out/bench_${c}_2r.err; echo "$c 2r rc=$?"; tail -c 300 gpurun_out/bench_${c}_2r.json
done
for c in c2 c5 c3 c4 c1; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --config c3 --perm random --steps 10 --warmup 3 > gpurun_out/bench_c3r.json 2> gpurun_out/bench_c3r.err; echo "c3r rc=$?"
for c in c2 c3 c4; do timeout 600 python bench.py --impl reference --config $c --steps 2 --warmup 1 > gpurun_out/ref_$c.json 2> gpurun_out/ref_$c.err; echo "ref $c rc=$?"; done
nproc
