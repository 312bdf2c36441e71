"""Throughput of the generic map (the register VM, ixg_map) on corpus
lambdas over device arrays (development tool).  python tools/vm_bench.py [log2n]"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import ops, vm  # noqa: E402
from paper_2506_23058_b200.ir import BinOp, Const, If, Lambda, VarE  # noqa: E402


def timeit(fn, reps=10):
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
    n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 26)
    dev = torch.device("cuda")
    c = ops.gen_uniform(n, 0, 1, 1, torch.int64, device=dev)
    t = ops.gen_uniform(n, 1, 1000, 2, torch.int64, device=dev)
    f = ops.gen_uniform(n, 1, 1000, 3, torch.int64, device=dev)
    st = ops.Status(dev)
    # partition2.ixl:15-16: \\c t f -> if c then t - 1 else f - 1  (c as 0/1)
    lam = Lambda(["c", "t", "f"], If(BinOp("!=", VarE("c"), Const(0)), BinOp("-", VarE("t"), Const(1)),
                                     BinOp("-", VarE("f"), Const(1))))
    comp = vm.compile_map(lam, [c, t, f], {})
    ms = timeit(lambda: ops.map_vm(comp, n, st, device=dev))
    print(f"vm map3 (partition2 indices) n=2^{n.bit_length() - 1}: {ms:.3f} ms, {n / ms / 1e6:.1f} Gelem/s, "
          f"{32 * n / ms / 1e6:.0f} GB/s")
    ref = torch.where(c != 0, t - 1, f - 1)
    out = ops.map_vm(comp, n, st, device=dev)
    assert torch.equal(out, ref)
    from paper_2506_23058_b200 import jit

    out, _ = jit.map_jit(lam, [c, t, f], {}, lambda node: 0, n, st, device=dev)
    assert torch.equal(out, ref)
    ms = timeit(lambda: jit.map_jit(lam, [c, t, f], {}, lambda node: 0, n, st, device=dev))
    print(f"jit map3 (NVRTC kernel): {ms:.3f} ms, {n / ms / 1e6:.1f} Gelem/s, {32 * n / ms / 1e6:.0f} GB/s")
    ms = timeit(lambda: torch.where(c != 0, t - 1, f - 1))
    print(f"torch.where equivalent: {ms:.3f} ms")


if __name__ == "__main__":
    main()
