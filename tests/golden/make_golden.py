"""Generate the golden fixtures from the Python reference itself.

Run in the build container (the reference is importable there, never on the
GPU box):

    python tests/golden/make_golden.py

Writes
  tests/golden/cases.json                  -- (program, fun, args) -> result or
                                              exception, computed by
                                              ixverify.oracle.eval_program
  paper_2506_23058_b200/data/programs.json -- normalized ASTs (ir.to_json) of
                                              every corpus program
  paper_2506_23058_b200/data/selection.json -- the verifier's per-site verdicts
                                              (select.select) keyed by
                                              function fingerprint

Inputs: the reference's own generator ``gen_args`` (oracle.py:602-620; sizes
0-12, precondition-satisfying) with its predicate callables replaced by
``Pred`` descriptors drawn from the same RNG (``x < thr``, ``x > thr`` or a
hash table, mirroring oracle.py:686-696), plus larger counter-generated
inputs, the SPEC/paper demo values and hand-made unsafe inputs that exercise
the CHECKED error paths.
"""

from __future__ import annotations

import glob
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402
from ixverify.normalize import check_well_formed, normalize  # noqa: E402
from ixverify.oracle import Interp, OracleError, eval_program, gen_args  # noqa: E402
from ixverify.oracle import _check_pre_atom, _conjuncts, chk_bij, chk_inj  # noqa: E402
from ixverify.parser import parse_program  # noqa: E402

import bigtrack  # noqa: E402
from paper_2506_23058_b200 import gen, ir  # noqa: E402
from paper_2506_23058_b200 import select as sel  # noqa: E402
from paper_2506_23058_b200.pred import GT, HASH, LT, Pred  # noqa: E402

BUDGET = 10**9


def corpus_files():
    ref = sorted(glob.glob("/root/reference/pkg/corpus/*.ixl"))
    own = sorted(glob.glob(os.path.join(ROOT, "corpus", "*.ixl")))
    return [("ref", p) for p in ref] + [("own", p) for p in own]


def key_of(origin, path):
    return f"{origin}:{os.path.basename(path)}"


def enc(v):
    if isinstance(v, Pred):
        return v.to_json()
    if isinstance(v, bool):
        return v
    if isinstance(v, int):
        return v
    if isinstance(v, float):
        return {"f": v.hex()}
    if isinstance(v, tuple):
        return {"tuple": [enc(x) for x in v]}
    if isinstance(v, list):
        return [enc(x) for x in v]
    raise TypeError(type(v))


def run(program, fun, args, budget=BUDGET):
    """the reference's answer; "big" when its evaluation left int64 (bigtrack.py)"""
    with bigtrack.tracking() as big:
        try:
            d = {"result": enc(eval_program(program, fun, args, budget))}
        except OracleError as e:
            d = {"error": type(e).__name__}
            if hasattr(e, "site"):
                d["site"] = e.site
            if getattr(e, "pos", None) is not None:
                d["pos"] = list(e.pos)
    if big[0] or not bigtrack.fits([a for a in args if not isinstance(a, Pred)]):
        d["big"] = True
    return d


PROPERTY_HEADS = {"Range", "Equiv", "Mono", "Inj", "Bij", "FiltPart", "InvFiltPart", "OrthogPreds"}


def ref_pre_holds(program, fun, args, required=None):
    """Do the entry function's annotations hold for these arguments, by the
    reference's own concrete predicates?  Range / Mono through
    oracle.py:712-734 _check_pre_atom, Inj / Bij over their codomain interval
    through chk_inj / chk_bij (oracle.py:492-520; the interval is what the
    verifier assumes, infer.py:306-324).  None = no annotations; False also
    for properties with no concrete check (Equiv, FiltPart, ...)."""
    interp = Interp(program, BUDGET)
    f = interp.funs[fun]
    if all(p.pre is None for p in f.params) or len(args) != len(f.params):
        return None
    env = {p.name: a for p, a in zip(f.params, args)}
    interp._bind_sizes(f, args, env)
    need = None if required is None else set(required)
    for p in f.params:
        if p.pre is None:
            continue
        for atom in _conjuncts(p.pre):
            if need is not None and sel.atom_key(p.name, atom) not in need:
                continue  # no elided check depends on it (select.required_atoms)
            head = atom.fun.name if type(atom).__name__ == "App" and type(atom.fun).__name__ == "VarE" else None
            try:
                if head in ("Inj", "Bij"):
                    x = env[atom.args[0].name]
                    lo, hi = (interp.eval(e, env) for e in atom.args[1].items)
                    if head == "Inj":
                        ok = chk_inj(x, lo, hi)
                    else:
                        ok = chk_bij(x, (lo, hi), None, [tuple(interp.eval(e, env) for e in atom.args[2].items)])
                elif head in PROPERTY_HEADS and head not in ("Range", "Mono"):
                    ok = False
                else:
                    ok = _check_pre_atom(atom, p, env, interp)
            except Exception:
                ok = False
            if not ok:
                return False
    return True


def swap_preds(args, rng):
    out = []
    for a in args:
        if callable(a):
            mode = rng.randrange(3)
            thr = rng.randint(-2, 9)
            out.append(Pred(LT, thr) if mode == 0 else Pred(GT, thr) if mode == 1 else Pred(HASH, 0, rng.getrandbits(64)))
        else:
            out.append(a)
    return out


def big_cases(fun):
    """Larger counter-generated inputs for the pipeline functions."""
    out = []
    for lg, seed in ((10, 1), (12, 2)):
        n = 1 << lg
        xs = gen.uniform(seed, n, -500, 500, np.int64).tolist()
        if fun in ("filter", "partition2"):
            out.append([Pred(LT, 7), xs])
            out.append([Pred(HASH, 0, 0xDEADBEEF + seed), xs])
        elif fun == "partition3":
            out.append([Pred(LT, -100), Pred(HASH, 0, 77), xs])
        elif fun == "filter_by":
            cs = [bool(c) for c in (gen.uniform(seed + 5, n, 0, 2, np.int64) == 0)]
            out.append([cs, xs])
        elif fun == "sum":
            out.append([xs])
        elif fun == "c2":
            k = sum(1 for x in xs if x >= 0)
            shape = gen.segment_shape(seed, 37, k).tolist()
            out.append([Pred.ge(0), xs, shape])
        elif fun in ("mkSgmDescr",):
            m = n // 16
            shape = gen.uniform(seed + 1, m, 0, 9, np.int64).tolist()
            out.append([shape, gen.uniform(seed + 2, m, -9, 9, np.int64).tolist()])
        elif fun == "mkII":
            out.append([gen.uniform(seed + 1, n // 16, 0, 9, np.int64).tolist()])
        elif fun == "sgmSum":
            flags = [bool(c) for c in (gen.uniform(seed + 3, n, 0, 7, np.int64) == 0)]
            out.append([flags, xs])
        elif fun == "mkFlags":
            m = 64
            shape = gen.segment_shape(seed, m, n // 2).tolist()
            out.append([n // 2, shape])
        elif fun in ("sc_bij", "sc_inj", "sc_any"):
            perm = np.argsort(np.argsort(np.array(xs), kind="stable"), kind="stable").tolist()
            out.append([[0] * n, perm, gen.uniform(seed + 4, n, -99, 99, np.int64).tolist()])
        elif fun in ("csrg", "csrg_any"):
            ncols = 97
            out.append([gen.uniform(seed + 6, ncols, -300, 300, np.int64).tolist(),
                        gen.uniform(seed + 7, n, -300, 300, np.int64).tolist(),
                        gen.uniform(seed + 8, n, 0, ncols - 1, np.int64).tolist()])
        elif fun in ("partition2L", "filter_seg"):
            m = n // 16
            shp = gen.uniform(seed + 10, m, 0, 31, np.int64)
            shp[::7] = 0  # empty rows
            nn = int(shp.sum())
            cs = [bool(c) for c in (gen.uniform(seed + 11, nn, 0, 2, np.int64) == 0)]
            out.append([shp.tolist(), cs, gen.uniform(seed + 12, nn, -500, 500, np.int64).tolist()])
        elif fun in ("scan_min", "scan_max", "scan_clip"):
            out.append([xs])
        elif fun == "scan_mul":
            out.append([[1 if v >= 0 else -1 for v in xs]])  # bounded products
        elif fun == "scan_and":
            out.append([[bool(c) for c in (gen.uniform(seed + 13, n, 0, 300, np.int64) != 0)]])
        elif fun == "scan_pair":
            out.append([xs, gen.uniform(seed + 14, n, -900, 900, np.int64).tolist()])
        elif fun == "scan_segmax":
            out.append([[bool(c) for c in (gen.uniform(seed + 15, n, 0, 9, np.int64) == 0)], xs])
        elif fun == "scan_lookup":
            out.append([gen.uniform(seed + 16, 97, -50, 50, np.int64).tolist(),
                        gen.uniform(seed + 17, n, 0, 96, np.int64).tolist()])
        elif fun == "pairs":
            out.append([xs])
        elif fun == "unpair":
            out.append([list(zip(xs, gen.uniform(seed + 25, n, -500, 500, np.int64).tolist()))])
        elif fun == "pair_pick":
            out += [[xs, 0], [xs, n - 1], [xs, n // 3]]
        elif fun in ("scan_fsum", "scan_fmax"):
            out.append([[round(float(v), 3) for v in np.random.default_rng(seed + 22).uniform(-50, 50, n)]])
        elif fun == "scan_decay":
            out.append([xs])
        elif fun in ("hist_fadd", "hist_fmin"):
            out.append([n // 4, gen.uniform(seed + 23, n, -3, n // 4 + 2, np.int64).tolist(),
                        [round(float(v), 3) for v in np.random.default_rng(seed + 24).uniform(-9, 9, n)]])
        elif fun in ("hist_mul", "hist_lmin", "hist_last", "hist_horner"):
            bins = n // 4 if fun != "hist_horner" else 2 * n
            out.append([bins, gen.uniform(seed + 18, n, -3, bins + 2, np.int64).tolist(),
                        gen.uniform(seed + 19, n, -3, 3, np.int64).tolist()])
        elif fun == "countdown":
            out.append([gen.uniform(seed + 21, n, 0, 3000, np.int64).tolist()])
        elif fun in ("all_rows", "row_corr"):
            rng = np.random.default_rng(seed + 20)
            rows = n // 16
            ptr = [0] + np.cumsum(rng.integers(0, 40, rows)).tolist()
            nnz, m = ptr[-1], 37
            args = [ptr, [round(float(v), 3) for v in rng.uniform(-4, 9, m)],
                    [round(float(v), 3) for v in rng.uniform(-4, 9, nnz)], rng.integers(0, m, nnz).tolist()]
            if fun == "all_rows":
                out.append(args)
            else:
                out += [[r] + args for r in (0, rows // 2, rows - 1)]
        elif fun == "get_smallest_pairs":
            nv = 50
            es = gen.uniform(seed + 9, 200, 0, nv - 1, np.int64).tolist()
            is_ = np.random.default_rng(seed).permutation(1000)[:200].tolist()
            out.append([nv, 10**6, es, is_])
    return out


def kmeans_cases(rng_seed):
    rng = np.random.default_rng(rng_seed)
    out = []
    for nrows in (1, 4, 9):
        lens = rng.integers(0, 7, nrows)
        ptr = [0] + np.cumsum(lens).tolist()
        nnz = ptr[-1]
        ncols = int(rng.integers(1, 6))
        vals = [round(float(v), 2) for v in rng.uniform(-4, 9, nnz)]
        cols = rng.integers(0, ncols, nnz).tolist()
        cl = [round(float(v), 2) for v in rng.uniform(-4, 9, ncols)]
        for row in range(nrows):
            out.append([row, ptr, cl, vals, cols])
    return out


BIG = 1 << 62


def overflow_cases(fun):
    """Values whose results leave int64 in the reference (its ints are
    unbounded: scan of [2^62, 2^62, 2^62] = [.., 3*2^62]),
    and ones that come close without leaving it."""
    if fun == "sum":
        return [[[BIG, BIG, BIG]], [[BIG, BIG - 1, -BIG]], [[-BIG, -BIG, -1]], [[(1 << 63) - 1, 1]],
                [[-BIG, -BIG]]]
    if fun == "sgmSum":
        return [[[True, False, False, True, False], [BIG, BIG, 5, BIG, BIG - 1]],
                [[True, False, True, False], [BIG, BIG, BIG, -BIG]]]
    if fun in ("csrg", "csrg_any"):
        return [[[1 << 40, 3], [1 << 30, 1 << 20], [0, 1]], [[1 << 31, 3], [1 << 31, -(1 << 31)], [0, 0]]]
    if fun == "c2":
        return [[Pred.ge(0), [BIG, BIG, -1, 3], [2, 1]], [Pred.ge(0), [BIG, BIG, -1, 3], [1, 1, 1]]]
    if fun in ("scan_mul",):
        return [[[1 << 40, 1 << 30, 1]], [[1 << 31, -(1 << 31), 2]], [[3] * 50]]
    if fun in ("hist_mul",):
        return [[2, [0, 0, 0, 1], [1 << 40, 1 << 30, 0, 5]], [2, [0, 0, 1], [1 << 40, 1 << 30, 5]]]
    if fun == "scan_pair":
        return [[[BIG, BIG], [1, 2]]]
    return []


def error_cases(fun):
    """Inputs that violate the annotations, so the CHECKED paths fire."""
    if fun == "sc_any":
        return [[[0, 0, 0, 0], [0, 2, 0], [1, 2, 3]],      # conflicting duplicate
                [[0, 0, 0], [1, 1, 7, -1], [5, 5, 9, 9]],  # equal duplicate + OOB
                [[0, 0, 0], [0, 1, 2], [7, 8]]]            # zip truncation
    if fun in ("csrg_any", "csrg"):  # csrg: its Range annotation violated
        return [[[1, 2, 3], [4, 5, 6, 7], [0, 2, 3, 1]], [[1, 2, 3], [4, 5], [-1, 0]], [[1, 2, 3], [4, 5], [0, 3]]]
    if fun == "sc_bij":  # Inj / Bij violated: conflict, equal duplicate, out of range, not onto
        return [[[0, 0, 0], [0, 0, 1], [5, 6, 7]], [[0, 0, 0], [0, 0, 1], [5, 5, 7]],
                [[9, 9, 9], [0, 5, 1], [1, 2, 3]], [[9, 9, 9], [2, 1, 1], [4, 4, 4]]]
    if fun == "sc_inj":
        return [[[0, 0, 0], [1, 1, 2], [4, 5, 6]], [[0, 0, 0], [1, 1, 2], [4, 4, 6]]]
    if fun == "c2":  # Range shape (0, inf) violated
        return [[Pred.ge(0), [1, -2, 3, 4, 0], [2, -1, 1, 1]], [Pred.ge(0), [5, 6, 7], [-2, 3, 2]]]
    if fun == "kmeans_ker":
        return [[2, [0, 1, 2], [1.5, 2.5], [0.5, 1.0], [0, 1]],         # pointers[row+1] OOB
                [0, [0, 3], [1.0], [0.5, 1.0, 2.0], [0, 0, 0]],          # values[...] OOB at j=2
                [0, [0, 2], [1.0, 2.0], [0.5, 1.0], [1, 5]],             # cluster[column] OOB
                [3, [0, 1, 2], [1.5, 2.5], [0.5, 1.0], [0, 1]],          # pointers[row] OOB
                [-1, [0, 1, 2], [1.5, 2.5], [0.5, 1.0], [0, 1]],         # negative row
                [0, [0, 2, 1], [1.5], [0.5, 1.0], [0, 0]]]               # Range pointers holds, row 1 empty
    if fun == "mkSgmDescr":
        return [[[3, -3, 4, 1], [1, 2, 3, 4]],                           # negative shape -> conflict
                [[2, 1, 3], [7, 8]], [[2, 0, 1], [1, 2, 3, 4]]]          # zip truncation: short / long xs
    if fun == "get_smallest_pairs":
        return [[3, 99, [0, 5, 1], [4, 2, 7]],                           # H[i] OOB
                [3, 99, [0, 1, 2, 1], [4, 4, 7, 7]]]                     # Inj is violated
    if fun == "all_rows":
        return [[[0, 2, 5], [1.5, 2.0], [0.5, 1.0, 2.0, 3.0], [0, 1, 1, 0]],     # vals[lo + j] OOB in row 1
                [[0, 1, 3], [1.5], [0.5, 1.0, 2.0], [0, 0, 4]]]                  # cl[cols[lo + j]] OOB
    if fun == "row_corr":
        return [[2, [0, 1, 2], [1.5, 2.5], [0.5, 1.0], [0, 1]],                  # ptr[row + 1] OOB
                [0, [0, 3], [1.0], [0.5, 1.0, 2.0], [0, 0, 0]]]                  # vals[lo + j] OOB at j = 2
    if fun == "pair_pick":
        return [[[1, 2, 3], 3], [[1, 2, 3], -1], [[], 0]]
    if fun == "countdown":
        return [[[3, -1, 5]], [[0] * 40 + [-2]]]                         # never-ending while loop
    if fun == "scan_lookup":
        return [[[1, 2, 3], [0, 2, 5, 1, 9]],                            # tbl[5] at element 2 (first)
                [[1, 2], [-1]],                                          # negative index
                [[4] * 40, list(range(40)) + [40]]]                      # last element only
    return []


DEMOS = {
    ("ref:partition2.ixl", "partition2"): [[Pred(LT, 5), [5, 4, 2, 8, 7, 3]]],
    ("ref:mksgmdescr.ixl", "mkSgmDescr"): [[[0, 2, 1, 0, 3], [1, 2, 3, 4, 5]]],
    ("own:mkii.ixl", "mkII"): [[[0, 2, 1, 0, 3]]],
    ("own:partition2l.ixl", "partition2L"): [[[3, 0, 2, 4], [True, False, True, False, True, False, False, True,
                                                               True], [10, 11, 12, 13, 14, 15, 16, 17, 18]],
                                             [[2, 1], [True, False, True, False], [1, 2, 3, 4]]],  # n != sum shp
    ("own:filter_seg.ixl", "filter_seg"): [[[3, 0, 2, 4], [True, False, True, False, True, False, False, True,
                                                             True], [10, 11, 12, 13, 14, 15, 16, 17, 18]],
                                           [[4], [True, False], [1, 2]]],  # n != sum shp
}


def main():
    programs, selection, cases = {}, {}, []
    for origin, path in corpus_files():
        key = key_of(origin, path)
        src = open(path).read()
        prog = normalize(parse_program(src, os.path.basename(path)))
        check_well_formed(prog)
        programs[key] = {"source": src, "program": ir.to_json(prog)}
        s = sel.select(prog)
        for name, fs in s.funcs.items():
            selection[f"{key}:{name}"] = fs.to_json()
        interp = Interp(prog, BUDGET)
        for f in prog.defs:
            rng = random.Random(hash((key, f.name)) & 0xFFFF if False else sum(map(ord, key + f.name)))
            draws = []
            if f.name in ("partition2L", "filter_seg"):
                # jagged inputs need n == sum shp, which the language cannot
                # state (gen_args would draw unrelated lengths; with sum shp > n
                # the reference's own scan indexes past the shorter array)
                for _ in range(40):
                    shp = [rng.randint(0, 4) for _ in range(rng.randint(0, 5))]
                    nn = sum(shp)
                    draws.append(("jagged", [shp, [rng.random() < 0.5 for _ in range(nn)],
                                             [rng.randint(-9, 9) for _ in range(nn)]]))
            elif f.name != "kmeans_ker":
                for _ in range(40):
                    a = gen_args(f, rng, interp)
                    if a is not None:
                        draws.append(("gen_args", swap_preds(a, rng)))
            else:
                draws += [("kmeans", a) for a in kmeans_cases(sum(map(ord, key)))]
            draws += [("big", a) for a in big_cases(f.name)]
            draws += [("error", a) for a in error_cases(f.name)]
            draws += [("overflow", a) for a in overflow_cases(f.name)]
            draws += [("demo", a) for a in DEMOS.get((key, f.name), [])]
            for origin_kind, a in draws:
                rec = {"program": key, "fun": f.name, "kind": origin_kind, "args": enc(a)}
                # a never-ending loop is cut by the default budget (oracle.py:118)
                bud = 10**6 if (f.name, origin_kind) == ("countdown", "error") else BUDGET
                rec.update(run(prog, f.name, a, bud))
                rec["pre"] = ref_pre_holds(prog, f.name, a, s.funcs[f.name].required)
                rec["budget"] = bud  # the step budget the reference ran with
                cases.append(rec)
    data = os.path.join(ROOT, "paper_2506_23058_b200", "data")
    os.makedirs(data, exist_ok=True)
    with open(os.path.join(data, "programs.json"), "w") as fh:
        json.dump(programs, fh)
    with open(os.path.join(data, "selection.json"), "w") as fh:
        json.dump(selection, fh, indent=1)
    with open(os.path.join(ROOT, "tests", "golden", "cases.json"), "w") as fh:
        json.dump(cases, fh)
    errs = sum(1 for c in cases if "error" in c)
    print(f"{len(programs)} programs, {len(selection)} function verdicts, {len(cases)} cases ({errs} raising)")


if __name__ == "__main__":
    main()
