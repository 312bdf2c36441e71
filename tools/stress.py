"""Randomised parity sweep of the ELIDED and CHECKED kernels against the C restatement
(test infrastructure: development tool, not part of the product).

Random sizes (ragged tiles, one-tile, multi-wave), predicates (selectivity
0 .. 1, edge thresholds), element types, for filter / partition2 /
partition3 / C2 / scan (+) / segmented scan / scatter (ELIDED permutation and
CHECKED with OOB and duplicates) / CSR gather / hist, each checked bit for
bit against oracle/ixoracle.  Runs
for --seconds (default 300) and prints a JSON summary; exits 1 on the first
mismatch.

python tools/stress.py [--seconds S] [--max-log2 L] [--seed N]
"""

import argparse
import json
import os
import random
import sys
import time

import numpy as np
import torch

os.environ.setdefault("IXG_BIN_SHIFT", "12")  # binned scatters with many windows at these sizes

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ixoracle as O  # noqa: E402
from paper_2506_23058_b200 import _lib as L  # noqa: E402
from paper_2506_23058_b200 import gen, ops  # noqa: E402
from paper_2506_23058_b200.pred import Pred  # noqa: E402


def rand_pred(rng, lo, hi):
    kind = rng.choice(["lt", "ge", "gt", "le", "eq", "ne", "hash", "true", "false"])
    thr = rng.choice([0, -1, 1, lo, hi, rng.randint(lo, hi)])
    if kind == "hash":
        return Pred.hash(rng.getrandbits(63))
    if kind == "true":
        return Pred(7)
    if kind == "false":
        return Pred(8)
    return {"lt": Pred.lt, "ge": Pred.ge, "gt": Pred.gt, "le": Pred.le, "eq": lambda t: Pred(4, t),
            "ne": lambda t: Pred(5, t)}[kind](thr)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--max-log2", type=int, default=25)
    ap.add_argument("--seed", type=int, default=1234)
    a = ap.parse_args()
    dev = torch.device("cuda")
    rng = random.Random(a.seed)
    t_end = time.time() + a.seconds
    counts = {}
    it = 0
    while time.time() < t_end:
        it += 1
        op = rng.choice(["filter", "partition2", "partition3", "c2", "scan", "segscan", "scatter", "csr", "hist",
                         "filter_chk", "partition2_chk", "partition3_chk", "c2_chk", "scatter_binned",
                         "scatter_streams", "scatter_conflict", "flags", "peer"])
        dt = rng.choice([np.int32, np.int64])
        lg = rng.randint(0, a.max_log2)
        n = max(0, (1 << lg) + rng.randint(-7, 7) * rng.choice([1, 17, 4099]))
        span = rng.choice([(-128, 127), (-(1 << 31), (1 << 31) - 1), (0, 3)])
        xs_h = gen.uniform(it, n, span[0], span[1], dt)
        xs = torch.from_numpy(xs_h).to(dev)
        st = ops.Status(dev)
        p = rand_pred(rng, *span)
        chk = op.endswith("_chk")
        variant = L.VARIANT_CHECKED if chk else L.VARIANT_ELIDED
        op = op.replace("_chk", "")
        if op == "filter":
            ys, dk = ops.filter(xs, p, variant, st)
            k = int(dk.item())
            want = O.filter_(p, xs_h)
            ok = k == len(want) and np.array_equal(ys[:k].cpu().numpy().astype(np.int64), want)
        elif op == "partition2":
            ys, dnt = ops.partition2(xs, p, variant, st)
            wnt, wys = O.partition2(p, xs_h)
            ok = int(dnt.item()) == wnt and np.array_equal(ys.cpu().numpy().astype(np.int64), wys)
        elif op == "partition3":
            q = rand_pred(rng, *span)
            ys, dm = ops.partition3(xs, p, q, variant, st)
            w1, w2, wys = O.partition3(p, q, xs_h)
            ok = dm.cpu().tolist() == [w1, w2] and np.array_equal(ys.cpu().numpy().astype(np.int64), wys)
        elif op == "scan":
            ne = rng.randint(-1000, 1000)
            v_h = gen.uniform(it, n, -(1 << 20), 1 << 20, dt)
            got = ops.scan_add(torch.from_numpy(v_h).to(dev), ne)
            ok = np.array_equal(got.cpu().numpy(), O.scan_add(v_h, ne))
        elif op == "segscan":
            v_h = gen.uniform(it, n, -(1 << 20), 1 << 20, np.int64)
            f_h = (gen.uniform(it + 1, n, 0, rng.choice([1, 5, 100, 10000]), np.int64) == 0).astype(np.uint8)
            got = ops.segscan_add(torch.from_numpy(f_h).to(dev), torch.from_numpy(v_h).to(dev))
            ok = np.array_equal(got.cpu().numpy(), O.sgmsum(f_h.astype(np.int64), v_h))
        elif op == "scatter":
            # a permutation (ELIDED Sc1) or random indices with OOB (CHECKED: no conflicts -> equal values)
            vs_h = gen.uniform(it, n, -(1 << 30), 1 << 30, np.int64)
            if rng.random() < 0.5:
                is_h = np.random.default_rng(it).permutation(n).astype(np.int64)
                bits, dst_h = 0, np.zeros(n, dtype=np.int64)
            else:
                is_h = gen.uniform(it + 2, n, -3, n + 3, np.int64)
                vs_h = is_h * 7 + 1  # duplicates carry equal values: never a conflict
                bits, dst_h = L.V_BOUNDS | L.V_CONFLICT | L.V_INIT, gen.uniform(it + 3, n, -9, 9, np.int64)
            out = torch.from_numpy(dst_h.copy()).to(dev)
            ops.scatter(out, torch.from_numpy(is_h).to(dev), torch.from_numpy(vs_h).to(dev), bits, st)
            ok = np.array_equal(out.cpu().numpy(), O.scatter(dst_h, is_h, vs_h))
        elif op == "scatter_binned":
            # destination-window binning (4096-destination windows here, IXG_BIN_SHIFT) in every form
            vs_h = gen.uniform(it, n, -(1 << 30), 1 << 30, np.int64)
            mode = rng.randrange(3)
            if mode == 0:  # Sc1: a permutation
                is_h = np.random.default_rng(it).permutation(n).astype(np.int64)
                bits, dst_h = 0, np.zeros(n, dtype=np.int64)
            elif mode == 1:  # injective only: a permutation of a larger range, some OOB
                is_h = np.random.default_rng(it).permutation(n + 50).astype(np.int64)[:n] - 3
                bits, dst_h = L.V_INIT, gen.uniform(it + 3, n, -9, 9, np.int64)
            else:  # CHECKED: duplicates with equal values, OOB
                is_h = gen.uniform(it + 2, n, -3, n + 3, np.int64)
                vs_h = is_h * 5 - 2
                bits, dst_h = L.V_BOUNDS | L.V_CONFLICT | L.V_INIT, gen.uniform(it + 3, n, -9, 9, np.int64)
            out = torch.from_numpy(dst_h.copy()).to(dev)
            ops.scatter(out, torch.from_numpy(is_h).to(dev), torch.from_numpy(vs_h).to(dev), bits, st,
                        layout=L.SCATTER_BINNED)
            ok = np.array_equal(out.cpu().numpy(), O.scatter(dst_h, is_h, vs_h))
        elif op == "scatter_streams":
            # CHECKED over C3's index pattern (two interleaved monotone streams: the set-associative
            # claim windows' fast path), a few indices moved out of range
            c_h = gen.uniform(it, n, 0, 1, np.int64) == 0
            t = np.cumsum(c_h)
            is_h = np.where(c_h, t - 1, (t[-1] if n else 0) + (np.arange(1, n + 1) - t) - 1).astype(np.int64)
            if n:
                is_h[gen.uniform(it + 1, max(1, n // 97), 0, n - 1, np.int64)] = -1
            vs_h = gen.uniform(it + 2, n, -(1 << 30), 1 << 30, np.int64)
            dst_h = gen.uniform(it + 3, n, -9, 9, np.int64)
            out = torch.from_numpy(dst_h.copy()).to(dev)
            ops.scatter(out, torch.from_numpy(is_h).to(dev), torch.from_numpy(vs_h).to(dev),
                        L.V_BOUNDS | L.V_CONFLICT | L.V_INIT, st)
            ok = np.array_equal(out.cpu().numpy(), O.scatter(dst_h, is_h, vs_h))
        elif op == "scatter_conflict":
            # CHECKED with ONE conflicting duplicate among equal-valued ones: NonIdempotentScatter
            if n < 2:
                continue
            is_h = gen.uniform(it + 2, n, 0, max(0, n - 1), np.int64)
            vs_h = is_h * 3 + 1
            j = rng.randrange(n)
            k2 = rng.randrange(n)
            is_h[k2] = is_h[j]
            if j != k2:
                vs_h[k2] = vs_h[j] + 1
            out = torch.from_numpy(np.zeros(n, np.int64)).to(dev)
            ops.scatter(out, torch.from_numpy(is_h).to(dev), torch.from_numpy(vs_h).to(dev),
                        L.V_BOUNDS | L.V_CONFLICT | L.V_INIT, st)
            s2 = st.read()
            ok = (not s2.ok and bool(s2.codes & (1 << L.CONFLICT))) if j != k2 else s2.ok
            st = ops.Status(dev)  # the expected failure is checked; the common check below sees a clean status
        elif op == "flags":
            # mkFlags as a bitmap (the C2 chain's clear + big-tile scan), empty / negative segments
            m = max(0, n // rng.choice([1, 3, 64]))
            shape_h = gen.uniform(it, m, rng.choice([0, -3]), rng.choice([1, 8, 300]), np.int64)
            scn = np.concatenate([[0], np.cumsum(shape_h)[:-1]]) if m else np.zeros(0, np.int64)
            nbits = int(shape_h[shape_h > 0].sum()) + rng.choice([0, 1, 77]) if m else rng.choice([1, 33])
            bits = ops.flag_bitmap(torch.from_numpy(shape_h).to(dev), nbits)
            got = bits.cpu().numpy().view(np.uint32)[: (nbits + 31) // 32].copy()
            if nbits % 32:
                got[-1] &= np.uint32((1 << (nbits % 32)) - 1)
            want = np.zeros((nbits + 31) // 32, np.uint32)
            sel = (shape_h > 0) & (scn >= 0) & (scn < nbits)
            np.bitwise_or.at(want, (scn[sel] >> 5).astype(np.int64), (np.uint32(1) << (scn[sel] & 31).astype(np.uint32)))
            ok = np.array_equal(got, want)
        elif op == "peer":
            # the sharded partition2 (one read, both classes placed) for G simulated ranks
            G = rng.choice([1, 2, 3, 5, 8])
            ep = 4 if dt == np.int32 else 2
            per = max(ep, (n // G) // ep * ep)
            xs_h = gen.uniform(it, G * per, span[0], span[1], dt)
            wnt, wys = O.partition2(p, xs_h)
            tdt = xs.dtype
            bufs = [torch.empty(per, dtype=tdt, device=dev) for _ in range(G)]
            shards = [torch.from_numpy(xs_h[r * per:(r + 1) * per].copy()).to(dev) for r in range(G)]
            d_counts = torch.cat([ops.partition_counts(x, p) for x in shards])
            for r in range(G):
                ops.partition2_peer(shards[r], p, [b.data_ptr() for b in bufs], per, d_counts, r)
            ok = int(d_counts.sum().item()) == wnt and np.array_equal(
                torch.cat(bufs).cpu().numpy().astype(np.int64), wys)
        elif op == "csr":
            ncols = rng.choice([1, 97, 1 << 16])
            x_h = gen.uniform(it, ncols, -(1 << 15), (1 << 15) - 1, np.int64)
            v_h = gen.uniform(it + 1, n, -(1 << 15), (1 << 15) - 1, np.int64)
            i_h = gen.uniform(it + 2, n, 0, ncols - 1, np.int64)
            got = ops.csr_gather(torch.from_numpy(x_h).to(dev), torch.from_numpy(v_h).to(dev),
                                 torch.from_numpy(i_h).to(dev), L.VARIANT_ELIDED, st)
            ok = np.array_equal(got.cpu().numpy(), O.csrg(x_h, v_h, i_h))
        elif op == "hist":
            dlen = rng.choice([0, 1, 100, n // 3 + 1])
            hop = rng.choice([O.HIST_MIN, O.HIST_MAX, O.HIST_ADD])
            is_h = gen.uniform(it, n, -2, dlen + 2, np.int64)
            vs_h = gen.uniform(it + 1, n, -(1 << 30), 1 << 30, np.int64)
            ne = rng.randint(-5, 5)
            got = ops.hist(hop, ne, dlen, torch.from_numpy(is_h).to(dev), torch.from_numpy(vs_h).to(dev))
            ok = np.array_equal(got.cpu().numpy(), O.hist(hop, ne, dlen, is_h, vs_h))
        else:
            xs_h = gen.uniform(it, n, -128, 127, dt)
            xs = torch.from_numpy(xs_h).to(dev)
            p = Pred.ge(rng.choice([0, -50, 50, -200, 200]))
            k = len(O.filter_(p, xs_h))
            m = max(1, rng.choice([1, 7, k // 64 + 1, k // 3 + 1]))
            shape = gen.segment_shape(it, m, k)
            ys, zs, dk = ops.c2(xs, p, torch.from_numpy(shape).to(dev), variant, st)
            kk = int(dk.item())
            wys, wzs = O.c2(p, xs_h, shape)
            # int32 zs: NARROW is flagged iff some exact sum leaves int32 (then zs wraps, as documented)
            fits = dt == np.int64 or len(wzs) == 0 or int(np.abs(wzs).max()) < (1 << 31) - 1 or \
                (int(wzs.max()) <= (1 << 31) - 1 and int(wzs.min()) >= -(1 << 31))
            narrow = st.read().narrow
            ok = kk == len(wys) and np.array_equal(ys[:kk].cpu().numpy().astype(np.int64), wys) and \
                narrow == (not fits) and (narrow or np.array_equal(zs[:kk].cpu().numpy().astype(np.int64), wzs))
            counts["c2_narrow"] = counts.get("c2_narrow", 0) + int(narrow)
        s = st.read()
        ok = ok and s.ok  # NARROW is a flag, not a failure code
        op = op + ("_chk" if chk else "")
        counts[op] = counts.get(op, 0) + 1
        if not ok:
            print(json.dumps({"mismatch": op, "n": n, "dtype": np.dtype(dt).name, "pred": repr(p), "iter": it}))
            sys.exit(1)
    print(json.dumps({"seed": a.seed, "iterations": it, "per_op": counts, "ok": True}))


if __name__ == "__main__":
    main()
