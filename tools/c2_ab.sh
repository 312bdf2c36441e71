# A/B of library builds on the C2 bench step (development tool):
#   bash tools/c2_ab.sh lib1.so lib2.so ...   (each run twice, interleaved)
export PYTHONPATH=$PWD
for rep in 1 2; do
  for l in "$@"; do
    IXGPU_LIB=$PWD/$l python bench.py --config ${AB_CONFIG:-c2} --steps 50 --warmup 5 --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$l', d['ms_per_step'], r['kernel_ms'], r['frac'], d['clocks']['sm_mhz'])"
  done
done
