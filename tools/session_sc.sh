export PYTHONPATH=$PWD
python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "scatter or stream" > gpurun_out/pytest_sc.txt 2>&1; tail -5 gpurun_out/pytest_sc.txt
for p in streams random; do timeout 600 python bench.py --config c3 --perm $p --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c3_$p.json 2> gpurun_out/bench_c3_$p.err; echo "c3 $p rc=$?"; done
cat > /tmp/c3prof.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2506_23058_b200 import ops, _lib as L
n = 1 << 29
dev = torch.device('cuda')
g = torch.Generator(device=dev); g.manual_seed(11)
for kind in sys.argv[1:]:
    if kind.startswith('random'):
        is_ = torch.randperm(n, generator=g, device=dev, dtype=torch.int64)
    else:
        xs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 11, torch.int32)
        c = xs < 0; t = torch.cumsum(c, 0, dtype=torch.int64); i1 = torch.arange(1, n + 1, device=dev, dtype=torch.int64)
        is_ = torch.where(c, t - 1, t[-1] + (i1 - t) - 1); del xs, c, t, i1
    vs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 12, torch.int32)
    out = torch.zeros(n, dtype=torch.int32, device=dev)
    st = ops.Status(dev)
    bits = L.V_CONFLICT | L.V_INIT if kind.endswith('chk') else 0
    for _ in range(2):
        ops.scatter(out, is_, vs, bits, st)
    torch.cuda.synchronize()
    del is_, vs, out
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum --clock-control none -k regex:"k_scatter|k_bin" --csv python /tmp/c3prof.py streams streams_chk random random_chk > gpurun_out/ncu_c3.csv 2> gpurun_out/ncu_c3.err
