# One GPU session: the GPU test suite, smoke, every bench config (ours + the
# reference arm), ncu launch lists of each config's step and --set full
# captures of the dominant kernels.  Outputs under gpurun_out/ (copy the
# summaries worth keeping to profiles/rNN/).
export PYTHONPATH=$PWD
set -u
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
for c in c2 c1 c5 c3 c4; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/ref_$c.json 2> gpurun_out/ref_$c.err; echo "ref $c rc=$?"
done
timeout 900 python bench.py --config c3 --perm random --steps 20 --warmup 5 > gpurun_out/bench_c3r.json 2> gpurun_out/bench_c3r.err; echo "bench c3r rc=$?"
for c in c2 c5; do
  IXG_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --config $c --quick --steps 3 --warmup 3 > gpurun_out/bench_${c}_2r.json 2> gpurun_out/bench_${c}_2r.err; echo "2 ranks $c rc=$?"
done
# launch lists (cold-cache, serialised: the kernels' shares of a step)
for c in c2 c1 c3 c4; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
  echo "launches $c rc=$?"
done
# --set full of the dominant kernels
cap() {  # name, kernel regex, launch-skip, command...
  local name=$1 kre=$2 skip=$3; shift 3
  ncu --set full --import-source on --clock-control none -k regex:"$kre" -s $skip -c 1 -o gpurun_out/full_$name "$@" > gpurun_out/full_$name.log 2>&1
  local rc=$?
  ncu -i gpurun_out/full_$name.ncu-rep --page raw --csv > gpurun_out/full_${name}_raw.csv 2>/dev/null
  rm -f gpurun_out/full_$name.ncu-rep
  echo "full $name rc=$rc"
}
cap c2_fused "k_filter_b" 2 python tools/prof_run.py c2 28 4
cap c5_place "k_filter_b" 2 python tools/prof_run.py partition2 28 4
cap c4_gather "k_csr_gather" 2 python tools/prof_run.py csr 28 4
cap c3_scatter "k_scatter_t" 1 python tools/c3prof.py streams
