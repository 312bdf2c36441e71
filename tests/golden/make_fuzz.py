"""Random programs for the generic executor's code generators (jit.py,
jit_fold.py), with their results computed by the Python reference itself.

Run in the build container (the reference is importable there):

    python tests/golden/make_fuzz.py

Writes tests/golden/fuzz.json: {"programs": {key: normalized AST}, "cases":
[{program, fun, args, result | error, site, pos}]}.  Every program is one
function of the shapes

    map  (\\x y -> E) xs ys          (+ a captured table `tbl` and scalar `s`)
    scan (\\a b -> E) c xs           (any operator: associative or not)
    hist (\\a b -> E) c m is vs
    map  (\\x -> loop (acc) = (c) for j < 3 do E) xs
    map  (\\x y -> F) xs ys                   (f64: Python float arithmetic)

with E drawn from + - *, comparisons, && || !, if / let, and table reads
tbl[E] that may fall outside the table (CHECKED sites raise OutOfBounds).
Operands stay small so that no value leaves int64.
"""

from __future__ import annotations

import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from ixverify.normalize import check_well_formed, normalize  # noqa: E402
from ixverify.oracle import OracleError, eval_program  # noqa: E402
from ixverify.parser import parse_program  # noqa: E402

import bigtrack  # noqa: E402
from paper_2506_23058_b200 import ir  # noqa: E402


def expr(rng, vars_, depth, tbl=True):
    """an integer expression over vars_ (names) of bounded magnitude"""
    if depth <= 0 or rng.random() < 0.25:
        if rng.random() < 0.7:
            return rng.choice(vars_)
        return str(rng.randint(0, 9))
    k = rng.random()
    if k < 0.45:
        op = rng.choice(["+", "-", "*", "+", "-"])
        return f"({expr(rng, vars_, depth - 1, tbl)} {op} {expr(rng, vars_, depth - 1, tbl)})"
    if k < 0.7:
        return f"(if {cond(rng, vars_, depth - 1, tbl)} then {expr(rng, vars_, depth - 1, tbl)} else " \
               f"{expr(rng, vars_, depth - 1, tbl)})"
    if k < 0.85 and tbl:
        return f"tbl[{expr(rng, vars_, depth - 1, False)}]"
    v = f"t{depth}"
    return f"(let {v} = {expr(rng, vars_, depth - 1, tbl)} in {expr(rng, vars_ + [v], depth - 1, tbl)})"


def cond(rng, vars_, depth, tbl):
    k = rng.random()
    if depth <= 0 or k < 0.6:
        op = rng.choice(["<", "<=", ">", ">=", "==", "!="])
        return f"({expr(rng, vars_, depth - 1, tbl)} {op} {expr(rng, vars_, depth - 1, tbl)})"
    if k < 0.8:
        op = rng.choice(["&&", "||"])
        return f"({cond(rng, vars_, depth - 1, tbl)} {op} {cond(rng, vars_, depth - 1, tbl)})"
    return f"(!{cond(rng, vars_, depth - 1, tbl)})"


ASSOC = ["a + b", "a * b", "if a < b then a else b", "if b <= a then a else b", "b", "a"]


def fexpr(rng, vars_, depth):
    """a float expression (Python floats: IEEE double, no contraction)"""
    if depth <= 0 or rng.random() < 0.25:
        if rng.random() < 0.7:
            return rng.choice(vars_)
        return rng.choice(["0.5", "1.25", "3.0", "0.1", "2"])
    k = rng.random()
    if k < 0.6:
        op = rng.choice(["+", "-", "*"])
        return f"({fexpr(rng, vars_, depth - 1)} {op} {fexpr(rng, vars_, depth - 1)})"
    if k < 0.85:
        c = rng.choice(["<", "<=", ">", ">="])
        return f"(if ({fexpr(rng, vars_, depth - 1)} {c} {fexpr(rng, vars_, depth - 1)}) then " \
               f"{fexpr(rng, vars_, depth - 1)} else {fexpr(rng, vars_, depth - 1)})"
    v = f"u{depth}"
    return f"(let {v} = {fexpr(rng, vars_, depth - 1)} in {fexpr(rng, vars_ + [v], depth - 1)})"


def program(rng, i):
    kind = rng.choice(["map", "map", "scan", "hist", "loop", "fmap"])
    if kind == "fmap":
        body = fexpr(rng, ["x", "y"], 3)
        src = (f"def f{i} [n] (xs: [n]f64) (ys: [n]f64) : [n]f64 =\n"
               f"  map (\\x y -> {body}) xs ys\n")
        return kind, src
    if kind == "map":
        body = expr(rng, ["x", "y", "s"], 3)
        src = (f"def f{i} [n] [m] (tbl: [m]i64) (s: i64) (xs: [n]i64) (ys: [n]i64) : [n]i64 =\n"
               f"  map (\\x y -> {body}) xs ys\n")
    elif kind == "scan":
        body = rng.choice(ASSOC) if rng.random() < 0.4 else expr(rng, ["a", "b"], 2, tbl=rng.random() < 0.3)
        src = (f"def f{i} [n] [m] (tbl: [m]i64) (xs: [n]i64) : [n]i64 =\n"
               f"  scan (\\a b -> {body}) {rng.randint(0, 5)} xs\n")
    elif kind == "hist":
        body = rng.choice(ASSOC[:4]) if rng.random() < 0.4 else expr(rng, ["a", "b"], 2, tbl=False)
        src = (f"def f{i} [n] (k: i64) (is: [n]i64) (vs: [n]i64) : []i64 =\n"
               f"  hist (\\a b -> {body}) {rng.randint(0, 5)} k is vs\n")
    else:
        body = expr(rng, ["acc", "x", "j"], 2)
        src = (f"def f{i} [n] [m] (tbl: [m]i64) (xs: [n]i64) : [n]i64 =\n"
               f"  map (\\x -> loop (acc) = ({rng.randint(0, 3)}) for j < 3 do {body}) xs\n")
    return kind, src


def args_for(rng, kind, n):
    xs = [rng.randint(-9, 9) for _ in range(n)]
    tbl = [rng.randint(-20, 20) for _ in range(rng.randint(1, 12))]
    if kind == "map":
        return [tbl, rng.randint(-5, 5), xs, [rng.randint(-9, 9) for _ in range(n)]]
    if kind in ("scan", "loop"):
        return [tbl, xs]
    if kind == "fmap":
        return [[round(rng.uniform(-9, 9), 3) for _ in range(n)], [round(rng.uniform(-9, 9), 3) for _ in range(n)]]
    k = rng.randint(0, 8)
    return [k, [rng.randint(-2, k + 1) for _ in range(n)], xs]


def main():
    rng = random.Random(2506)
    programs, cases = {}, []
    budget = 10**7
    made = 0
    import signal

    def _slow(*_):
        raise TimeoutError

    signal.signal(signal.SIGALRM, _slow)
    while made < 300:
        kind, src = program(rng, made)
        signal.alarm(5)  # a candidate the reference needs seconds for is dropped
        # keep value magnitudes bounded: the reference's ints are unbounded
        try:
            prog = normalize(parse_program(src, f"fuzz{made}.ixl"))
            check_well_formed(prog)
        except Exception:
            signal.alarm(0)
            continue
        fname = prog.defs[0].name
        key = f"fuzz:{made}"
        rows = []
        ok = True
        for n in (0, 1, 5, 33, 300):
            a = args_for(rng, kind, n)
            # values are NOT bounded: a result or intermediate that leaves int64
            # is kept and marked "big" (bigtrack.py) -- the GPU must then raise
            # IntegerOverflow (or still match), never return a wrapped value
            with bigtrack.tracking() as big:
                try:
                    res = eval_program(prog, fname, a, budget)
                    d = {"program": key, "fun": fname, "kind": kind, "args": a, "result": res}
                except TimeoutError:
                    ok = False
                    break
                except OracleError as e:
                    d = {"program": key, "fun": fname, "kind": kind, "args": a, "error": type(e).__name__}
                    if hasattr(e, "site"):
                        d["site"] = e.site
                    if getattr(e, "pos", None) is not None:
                        d["pos"] = list(e.pos)
            if big[0]:
                d["big"] = True
            rows.append(d)
        signal.alarm(0)
        if not ok:
            print("dropped (slow or huge):", src.strip()[:160], file=sys.stderr)
            continue
        programs[key] = {"source": src, "program": ir.to_json(prog)}
        cases += rows
        made += 1
    with open(os.path.join(ROOT, "tests", "golden", "fuzz.json"), "w") as fh:
        json.dump({"programs": programs, "cases": cases}, fh)
    errs = sum(1 for c in cases if "error" in c)
    print(f"{len(programs)} programs, {len(cases)} cases ({errs} raising)")


if __name__ == "__main__":
    main()
