"""Time the generic-operator paths (development tool): jit_fold's tiled
scan for an associative operator (min, segmented max), the CAS hist, and
the kmeans row loop compiled from corpus/kmeans_rows.ixl (a map calling a
looping row function, inlined by jit.py) next to the registered
ixg_kmeans_ker pipeline.

python tools/fold_bench.py [log2 n]
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import _lib as L  # noqa: E402
from paper_2506_23058_b200 import ir, jit, jit_fold, ops  # noqa: E402

V = ir.VarE
DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_23058_b200", "data")


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    n = 1 << lg
    dev = torch.device("cuda")
    st = ops.Status(dev)
    out = {"n": n}
    xs = ops.gen_uniform(n, -(1 << 40), 1 << 40, 1, torch.int64, device=dev)
    fl = (ops.gen_uniform(n, 0, 63, 2, torch.int64, device=dev) == 0).to(torch.uint8)
    mn = ir.Lambda(("a", "b"), ir.If(ir.BinOp("<", V("a"), V("b")), V("a"), V("b")))
    segmax = ir.Lambda(("f1", "v1", "f2", "v2"), ir.TupleE((ir.BinOp("||", V("f1"), V("f2")), ir.If(
        V("f2"), V("v2"), ir.If(ir.BinOp("<", V("v1"), V("v2")), V("v2"), V("v1"))))))
    bits = lambda node: 0  # noqa: E731
    ms = timeit(lambda: jit_fold.scan(mn, [0], [xs], {}, bits, st, device=dev))
    out["scan_min_i64"] = {"ms": ms, "Gelem/s": n / ms / 1e6, "alg_GB/s": 16 * n / ms / 1e6}
    ms = timeit(lambda: jit_fold.scan(segmax, [0, 0], [fl, xs], {}, bits, st, device=dev))
    out["scan_segmax_u8_i64"] = {"ms": ms, "Gelem/s": n / ms / 1e6, "alg_GB/s": 25 * n / ms / 1e6}
    ms = timeit(lambda: ops.scan_add(xs, 0))
    out["scan_add_i64_builtin"] = {"ms": ms, "Gelem/s": n / ms / 1e6}
    m = n // 4
    is_ = ops.gen_uniform(m, 0, (1 << 20) - 1, 3, torch.int64, device=dev)
    vs = ops.gen_uniform(m, -1, 1, 4, torch.int64, device=dev)
    mul = ir.Lambda(("a", "b"), ir.BinOp("*", V("a"), V("b")))
    ms = timeit(lambda: jit_fold.hist(mul, 1, 1 << 20, is_, vs, {}, bits, st))
    out["hist_mul_cas"] = {"ms": ms, "Gelem/s": m / ms / 1e6, "bins": 1 << 20}
    ms = timeit(lambda: ops.hist(L.HIST_MIN, 1 << 40, 1 << 20, is_, vs))
    out["hist_min_builtin"] = {"ms": ms, "Gelem/s": m / ms / 1e6}
    # kmeans rows: inlined JIT map vs the registered pipeline
    prog = ir.from_json(json.load(open(os.path.join(DATA, "programs.json")))["own:kmeans_rows.ixl"]["program"])
    funs = {f.name: f for f in prog.defs}
    body = funs["all_rows"].body
    while ir.kind(body) == "Let":
        body = body.body
    lam = body.args[0]
    rows_n, ncols = 1 << 20, 1 << 12
    lens = ops.gen_uniform(rows_n, 0, 127, 22, torch.int64, device=dev)
    ptr = torch.zeros(rows_n + 1, dtype=torch.int64, device=dev)
    ptr[1:] = torch.cumsum(lens, 0)
    nnz = int(ptr[-1].item())
    vals = torch.rand(nnz, dtype=torch.float64, device=dev)
    idx = ops.gen_uniform(nnz, 0, ncols - 1, 23, torch.int64, device=dev)
    cl = torch.rand(ncols, dtype=torch.float64, device=dev)
    rows = torch.arange(rows_n, dtype=torch.int64, device=dev)
    env = {"ptr": ("array", ptr), "cl": ("array", cl), "vals": ("array", vals), "cols": ("array", idx)}
    f_jit = lambda: jit.map_jit(lam, [rows], env, bits, rows_n, st, device=dev, funs=funs,  # noqa: E731
                                bits_for=lambda name: bits)
    got, _ = f_jit()
    ref = ops.kmeans_ker(rows, ptr, cl, vals, idx, L.VARIANT_ELIDED, st)
    out["kmeans_rows_equal"] = bool(torch.equal(got, ref))
    ms = timeit(f_jit)
    out["kmeans_rows_jit"] = {"ms": ms, "Gnnz/s": nnz / ms / 1e6}
    ms = timeit(lambda: ops.kmeans_ker(rows, ptr, cl, vals, idx, L.VARIANT_ELIDED, st))
    out["kmeans_rows_pipeline"] = {"ms": ms, "Gnnz/s": nnz / ms / 1e6}
    out["status_ok"] = st.read().ok
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
