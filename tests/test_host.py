"""CPU tests of the host side: program snapshots, fingerprints, the selector
against the live reference verifier, the lambda compiler, the C-ABI exports."""

import ctypes
import json
import os
import re

import pytest

from paper_2506_23058_b200 import _lib as L
from paper_2506_23058_b200 import ir, vm
from paper_2506_23058_b200 import select as sel
from paper_2506_23058_b200.pred import Pred

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROGRAMS = json.load(open(os.path.join(ROOT, "paper_2506_23058_b200", "data", "programs.json")))
SELECTION = json.load(open(os.path.join(ROOT, "paper_2506_23058_b200", "data", "selection.json")))


def test_abi_exports_every_declared_symbol():
    """libixgpu.so loads (no GPU needed) and exports every function include/ixgpu.h declares."""
    hdr = open(os.path.join(ROOT, "include", "ixgpu.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(ixg_\w+)\(", hdr, re.M))
    assert len(declared) >= 25
    lib = L.load(require_device=False)
    for name in declared:
        assert hasattr(lib, name), name
        assert name in L.SIGNATURES, name
    assert lib.ixg_version() == 1
    assert lib.ixg_ws_bytes(L.OP_C2, 1 << 20, 1 << 10) > (1 << 20) // 8


def test_oracle_not_imported_by_product():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2506_23058_b200")):
        for fn in files:
            if fn.endswith(".py"):
                src = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(from\s+oracle\b|import\s+oracle\b)", src, re.M), fn
                assert not re.search(r"^\s*(from|import)\s+\S*ixoracle", src, re.M), fn
                assert "libixoracle" not in src, fn


def test_snapshot_round_trip_and_fingerprints():
    for key, d in PROGRAMS.items():
        prog = ir.from_json(d["program"])
        assert ir.to_json(prog) == d["program"]
        for f in prog.defs:
            assert SELECTION[f"{key}:{f.name}"]["fingerprint"] == ir.fingerprint(f)


def test_frozen_selection_golden():
    """SURVEY.md Appendix B, as frozen in data/selection.json."""
    def bits(key):
        return [(s["kind"], tuple(s["pos"]), sel.SiteVerdict(**{**s, "pos": tuple(s["pos"])}).bits)
                for s in SELECTION[key]["sites"]]
    assert bits("ref:partition2.ixl:partition2") == [("bounds", (12, 40), 0), ("scatter-safety", (18, 12), 0)]
    assert bits("ref:filter.ixl:filter") == [("bounds", (11, 33), 0), ("scatter-safety", (14, 12), 0)]
    assert bits("ref:partition3.ixl:partition3")[-1] == ("scatter-safety", (26, 12), 0)
    assert bits("ref:maxmatching.ixl:get_smallest_pairs") == [("bounds", (18, 27), 0)]
    assert all(b == 0 for _, _, b in bits("ref:kmeans_ker.ixl:kmeans_ker"))
    # mkSgmDescr: bounds proved, the scatter never reached -> fully CHECKED
    mk = bits("ref:mksgmdescr.ixl:mkSgmDescr")
    assert [b for _, _, b in mk[:3]] == [0, 0, 0] and mk[3][2] == L.V_CONFLICT | L.V_INIT
    # mkFlags: Ss2 proved (no conflict check) but no conversion rule: init kept
    assert bits("own:c2_filter_sgmsum.ixl:mkFlags")[-1][2] == L.V_INIT
    assert bits("own:c3_scatter.ixl:sc_bij") == [("scatter-safety", (6, 12), 0)]
    assert bits("own:c3_scatter.ixl:sc_inj")[0][2] == L.V_INIT
    assert bits("own:c3_scatter.ixl:sc_any")[0][2] == L.V_CONFLICT | L.V_INIT
    assert bits("own:c4_csr_gather.ixl:csrg")[0][2] == 0
    assert bits("own:c4_csr_gather.ixl:csrg_any")[0][2] == L.V_BOUNDS


@pytest.mark.reference
def test_live_selector_matches_frozen(reference):
    from ixverify.normalize import normalize
    from ixverify.parser import parse_program

    for key, d in PROGRAMS.items():
        prog = normalize(parse_program(d["source"], key.split(":")[1]))
        s = sel.select(prog)
        for name, fs in s.funcs.items():
            assert fs.to_json() == SELECTION[f"{key}:{name}"], (key, name)


@pytest.mark.reference
def test_snapshot_matches_reference_parse(reference):
    """A program parsed by the reference fingerprints like its snapshot (the
    fingerprint ignores the fresh %aN names normalization invents)."""
    from ixverify.normalize import normalize
    from ixverify.parser import parse_program

    for key, d in PROGRAMS.items():
        a = normalize(parse_program(d["source"]))
        b = ir.from_json(d["program"])
        for fa, fb in zip(a.defs, b.defs):
            assert ir.fingerprint(fa) == ir.fingerprint(fb)
            assert [(k, p) for k, p, _ in ir.sites(fa)] == [(k, p) for k, p, _ in ir.sites(fb)]


def test_expr_str_matches_reference_sites():
    prog = ir.from_json(PROGRAMS["ref:kmeans_ker.ixl"]["program"])
    f = ir.find_def(prog, "kmeans_ker")
    assert [ir.expr_str(n) for _, _, n in ir.sites(f)] == [
        "pointers[row]", "pointers[row + 1]", "values[index_start + j]", "indices[index_start + j]",
        "cluster[column]"]


def _calls_program_function(e, prog):
    """loops, tuples and calls of program functions inside a lambda are
    compiled by the NVRTC path only (jit.py), not the register VM"""
    names = {f.name for f in prog.defs}
    if ir.kind(e) in ("Loop", "TupleE") or (ir.kind(e) == "App" and ir.kind(e.fun) == "VarE" and e.fun.name in names):
        return True
    if ir.kind(e) == "Let" and len(e.names) > 1:
        return True
    return any(_calls_program_function(c, prog) for c in ir.children(e))


def test_vm_compiles_corpus_lambdas():
    """Every map lambda of the corpus compiles to the register program."""
    n = 0
    for key, d in PROGRAMS.items():
        prog = ir.from_json(d["program"])
        for f in prog.defs:
            lets = set()

            def collect(e):
                if ir.kind(e) == "Let":
                    lets.update(e.names)
                for c in ir.children(e):
                    collect(c)
            collect(f.body)

            def walk(e):
                nonlocal n
                if ir.kind(e) == "App" and ir.kind(e.fun) == "VarE" and e.fun.name == "map" and ir.kind(e.args[0]) == "Lambda":
                    lam = e.args[0]
                    env = {}
                    for p in f.params:
                        env[p.name] = ("pred", object()) if ir.kind(p.type) == "TFun" else ("array", object())
                    env.update({s: ("scalar", 3) for s in f.sizes})
                    for nm in ("num_true", "m1", "m2", "count", "len"):
                        env.setdefault(nm, ("scalar", 1))
                    for nm in ("H", "shape", "x"):
                        env.setdefault(nm, ("array", object()))
                    for nm in lets:  # let-bound names of the body (arrays, except the scalars above)
                        env.setdefault(nm, ("array", object()))
                    arrs = [object() for _ in lam.params]
                    if _calls_program_function(lam, prog):
                        return  # inlined calls (loops, f64) are the NVRTC path's: jit.py
                    c = vm.compile_map(lam, arrs, env)
                    assert c.insns[-1][0] == L.VM_OUT and len(c.insns) <= L.VM_MAX_INSN
                    n += 1
                for c in ir.children(e):
                    walk(c)
            walk(f.body)
    assert n >= 20


def test_vm_short_circuit_and_if_guard_indexing():
    # \i -> if i == 0 then 0 else shape[i-1]: the IndexE sits behind a jump
    lam = ir.Lambda(("i",), ir.If(ir.BinOp("==", ir.VarE("i"), ir.Const(0)), ir.Const(0),
                                   ir.IndexE(ir.VarE("shape"), ir.BinOp("-", ir.VarE("i"), ir.Const(1)), (6, 51))),
                    (0, 0))
    c = vm.compile_map(lam, [object()], {"shape": ("array", object())})
    ops = [i[0] for i in c.insns]
    jz = ops.index(L.VM_JZ)
    assert ops.index(L.VM_IDX) > jz
    assert c.sites[0].pos == (6, 51)


def test_errors_mirror():
    from paper_2506_23058_b200 import errors

    e = errors.OutOfBounds("xs[i]", (3, 4))
    assert str(e) == "out of bounds: xs[i]" and e.site == "xs[i]" and e.pos == (3, 4)
    assert isinstance(errors.NonIdempotentScatter((1, 2)), errors.OracleError)


def test_jit_generates_and_compiles_corpus_lambdas():
    """Every map lambda of the corpus becomes a CUDA kernel that NVRTC
    compiles for sm_100a (no GPU needed to compile)."""
    import torch

    from paper_2506_23058_b200 import jit

    nvrtc = pytest.importorskip("cuda.bindings.nvrtc")
    seen = set()
    for key, d in PROGRAMS.items():
        prog = ir.from_json(d["program"])
        for f in prog.defs:
            lets = set()

            def collect(e):
                if ir.kind(e) == "Let":
                    lets.update(e.names)
                for c in ir.children(e):
                    collect(c)
            collect(f.body)

            def walk(e):
                if ir.kind(e) == "App" and ir.kind(e.fun) == "VarE" and e.fun.name == "map" and ir.kind(e.args[0]) == "Lambda":
                    lam = e.args[0]
                    env = {}
                    for p in f.params:
                        env[p.name] = ("pred", Pred.lt(3)) if ir.kind(p.type) == "TFun" else ("array", torch.zeros(4, dtype=torch.int64))
                    env.update({s: ("scalar", 3) for s in f.sizes})
                    for nm in ("num_true", "m1", "m2", "count", "len"):
                        env.setdefault(nm, ("scalar", 1))
                    for nm in ("H", "shape", "x"):
                        env.setdefault(nm, ("array", torch.zeros(4, dtype=torch.int64)))
                    for nm in lets:
                        env.setdefault(nm, ("array", torch.zeros(4, dtype=torch.int64)))
                    funs = {g.name: g for g in prog.defs}
                    tup = {}  # parameters destructured by a tuple let: arrays of tuples

                    def find(x):
                        if ir.kind(x) == "Let" and len(x.names) > 1 and ir.kind(x.rhs) == "VarE":
                            tup[x.rhs.name] = len(x.names)
                        for c in ir.children(x):
                            find(c)
                    find(lam.body)
                    arrs = [jit.TupleCols([torch.zeros(4, dtype=torch.int64)] * tup[p]) if p in tup else
                            torch.zeros(4, dtype=torch.int64) for p in lam.params]
                    src, spec = jit.generate(lam, arrs, env, funs=funs, k_out=jit.tuple_arity(lam.body, funs))
                    if src not in seen:
                        seen.add(src)
                        err, prog_ = nvrtc.nvrtcCreateProgram(src.encode(), b"m.cu", 0, [], [])
                        opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-default-device"]
                        (err,) = nvrtc.nvrtcCompileProgram(prog_, len(opts), opts)
                        assert int(err) == 0, src
                for c in ir.children(e):
                    walk(c)
            walk(f.body)
    assert len(seen) >= 15


def _scanops_lambdas():
    prog = ir.from_json(PROGRAMS["own:scanops.ixl"]["program"])
    out = {}
    for f in prog.defs:
        def walk(e):
            if ir.kind(e) == "App" and ir.kind(e.fun) == "VarE" and e.fun.name in ("scan", "hist"):
                out[f.name] = (e.fun.name, e.args[0], (len(e.args) - 1) // 2)
            for c in ir.children(e):
                walk(c)
        walk(f.body)
    return out


def test_fold_classifier():
    """jit_fold's structural classifier: associative scan operators take the
    tiled parallel scan, commutative+associative hist operators the CAS loop,
    everything else the in-order device fold (oracle.py:281-316)."""
    from paper_2506_23058_b200 import jit_fold

    lams = _scanops_lambdas()
    par = {name for name, (kind, lam, k) in lams.items() if kind == "scan" and jit_fold.classify_scan(lam, k)}
    # (structural: a float accumulator still takes the in-order fold at run time, jit_fold.scan)
    assert par == {"scan_min", "scan_max", "scan_mul", "scan_and", "scan_pair", "scan_segmax", "scan_fsum",
                   "scan_fmax"}
    hk = {name: jit_fold.classify_hist(lam) for name, (kind, lam, k) in lams.items() if kind == "hist"}
    assert hk == {"hist_mul": "mul", "hist_lmin": "min", "hist_last": None, "hist_horner": None, "hist_fadd": "add",
                  "hist_fmin": None}
    assert jit_fold.fold_types(lams["scan_decay"][1], 1, [False], [False]) == ["f"]  # int ne, float operator
    assert jit_fold.fold_types(lams["scan_min"][1], 1, [False], [False]) == ["i"]
    # the corpus' own (+) and segmented (+) are associative too
    c2 = ir.from_json(PROGRAMS["own:c2_filter_sgmsum.ixl"]["program"])
    seg = [e for f in c2.defs if f.name == "sgmSum" for e in [f.body]][0]
    while ir.kind(seg) == "Let":
        seg = seg.rhs
    assert jit_fold.classify_scan(seg.args[0], 2)
    # min / max / projections from every comparison
    for op, want in (("<", "min"), ("<=", "min"), (">", "max"), (">=", "max")):
        lam = ir.Lambda(("a", "b"), ir.If(ir.BinOp(op, ir.VarE("a"), ir.VarE("b")), ir.VarE("a"), ir.VarE("b")))
        assert jit_fold.classify_hist(lam) == want
        lam2 = ir.Lambda(("a", "b"), ir.If(ir.BinOp(op, ir.VarE("b"), ir.VarE("a")), ir.VarE("a"), ir.VarE("b")))
        assert jit_fold.classify_hist(lam2) == {"min": "max", "max": "min"}[want]
    lam = ir.Lambda(("a", "b"), ir.BinOp("-", ir.VarE("a"), ir.VarE("b")))
    assert not jit_fold.classify_scan(lam, 1) and jit_fold.classify_hist(lam) is None


def test_fold_kernels_compile():
    """Every scanops operator's generated kernels (parallel and in-order
    forms) compile with NVRTC for sm_100a (no GPU needed)."""
    import torch

    from paper_2506_23058_b200 import jit_fold

    nvrtc = pytest.importorskip("cuda.bindings.nvrtc")

    def compile_ok(src):
        err, prog_ = nvrtc.nvrtcCreateProgram(src.encode(), b"f.cu", 0, [], [])
        opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-default-device"]
        (err,) = nvrtc.nvrtcCompileProgram(prog_, len(opts), opts)
        if err != nvrtc.nvrtcResult.NVRTC_SUCCESS:
            _, size = nvrtc.nvrtcGetProgramLogSize(prog_)
            log = b" " * size
            nvrtc.nvrtcGetProgramLog(prog_, log)
            raise AssertionError(log.decode() + "\n" + src)

    env = {"tbl": ("array", torch.zeros(4, dtype=torch.int64))}
    for name, (kind, lam, k) in _scanops_lambdas().items():
        if ir.kind(lam) != "Lambda":
            continue  # a named operator (i64.min): the executor builds its lambda
        if kind == "scan":
            types = ["long long"] * k
            if jit_fold.classify_scan(lam, k):
                compile_ok(jit_fold._par_scan_source(lam, k, types)[0])
            compile_ok(jit_fold._seq_scan_source(lam, k, types, env, lambda node: L.V_BOUNDS)[0])
        else:
            if jit_fold.classify_hist(lam):
                compile_ok(jit_fold._hist_cas_source(lam, "long long"))
            compile_ok(jit_fold._hist_seq_source(lam, "long long", env, lambda node: L.V_BOUNDS)[0])


def test_jit_loops_floats_and_inlining_compile():
    """A function-level loop (kmeans_ker, oracle.py:242-262) and a map that
    calls a looping row function (corpus/kmeans_rows.ixl) generate kernels
    NVRTC compiles; float arithmetic uses the round-to-nearest intrinsics."""
    import torch

    from paper_2506_23058_b200 import jit

    nvrtc = pytest.importorskip("cuda.bindings.nvrtc")
    prog = ir.from_json(PROGRAMS["own:kmeans_rows.ixl"]["program"])
    funs = {f.name: f for f in prog.defs}
    allrows = funs["all_rows"]
    lam = allrows.body
    while ir.kind(lam) == "Let":
        lam = lam.body
    lam = lam.args[0]
    f64, i64 = torch.zeros(4, dtype=torch.float64), torch.zeros(4, dtype=torch.int64)
    env = {"ptr": ("array", i64), "cl": ("array", f64), "vals": ("array", f64), "cols": ("array", i64)}
    src, spec = jit.generate(lam, [i64], env, funs=funs)
    assert "__dmul_rn" in src and "__dsub_rn" in src and "__dadd_rn" in src
    assert spec.out_types == ["f"] and len(spec.sites) == 5
    kprog = ir.from_json(PROGRAMS["ref:kmeans_ker.ixl"]["program"])
    body = kprog.defs[0].body
    while ir.kind(body) == "Let":
        body = body.body
    assert ir.kind(body) == "Loop"
    kenv = {"index_start": ("scalar", 0), "nnz_sgm": ("scalar", 3), "values": ("array", f64),
            "indices": ("array", i64), "cluster": ("array", f64)}
    src2, spec2 = jit.generate(ir.Lambda((), body), [], kenv)
    for s in (src, src2):
        err, p_ = nvrtc.nvrtcCreateProgram(s.encode(), b"l.cu", 0, [], [])
        opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-default-device"]
        (err,) = nvrtc.nvrtcCompileProgram(p_, len(opts), opts)
        assert err == nvrtc.nvrtcResult.NVRTC_SUCCESS, s


def test_fuzz_fixtures_load():
    """tests/golden/fuzz.json (the reference's results on random programs,
    replayed on the GPU by test_gpu_fuzz.py) is well formed."""
    fz = json.load(open(os.path.join(ROOT, "tests", "golden", "fuzz.json")))
    assert len(fz["programs"]) >= 200 and len(fz["cases"]) >= 1000
    kinds = set()
    for key, d in fz["programs"].items():
        prog = ir.from_json(d["program"])
        assert len(prog.defs) == 1 and len(ir.fingerprint(prog.defs[0])) == 16
    for c in fz["cases"]:
        assert c["program"] in fz["programs"] and ("result" in c) != ("error" in c)
        kinds.add(c["kind"])
    assert kinds == {"map", "scan", "hist", "loop", "fmap"}


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the reference's CPU path on the host cores)
    prints one JSON line with the contract's keys; runs without a GPU."""
    import subprocess
    import sys

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["warmup"] >= 3 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in line["config"]


# ----------------------------------------------------------------- soundness of the selection
def _prog(key):
    return ir.from_json(PROGRAMS[key]["program"])


def test_closure_keys_distinguish_annotations():
    """csrg / csrg_any and sc_bij / sc_inj share a body but not their
    annotations: their verdicts must not share a key."""
    def key(k, fn):
        p = _prog(k)
        return ir.closure_fingerprint(p, ir.find_def(p, fn))

    c4, c3 = "own:c4_csr_gather.ixl", "own:c3_scatter.ixl"
    assert ir.fingerprint(ir.find_def(_prog(c4), "csrg")) == ir.fingerprint(ir.find_def(_prog(c4), "csrg_any"))
    assert key(c4, "csrg") != key(c4, "csrg_any")
    assert key(c3, "sc_bij") != key(c3, "sc_inj") != key(c3, "sc_any")
    assert key("ref:kmeans_ker.ixl", "kmeans_ker") != key("own:kmeans_noann.ixl", "kmeans_ker")


def test_frozen_table_unambiguous_and_selects_by_contract():
    fz = sel.frozen()
    assert not sel.AMBIGUOUS, sel.AMBIGUOUS
    assert all(fs.closure for fs in fz.values())
    bits = lambda k, fn: [s.bits for s in sel.selection_for(_prog(k), ir.find_def(_prog(k), fn), live=False).sites]
    assert bits("own:c4_csr_gather.ixl", "csrg") == [0]
    assert bits("own:c4_csr_gather.ixl", "csrg_any") == [L.V_BOUNDS]
    assert bits("own:c3_scatter.ixl", "sc_bij") == [0]
    assert bits("own:c3_scatter.ixl", "sc_inj") == [L.V_INIT]
    assert bits("own:c3_scatter.ixl", "sc_any") == [L.V_CONFLICT | L.V_INIT]
    # kmeans_ker without its Range annotations: every site CHECKED
    assert bits("ref:kmeans_ker.ixl", "kmeans_ker") == [0] * 5
    assert bits("own:kmeans_noann.ixl", "kmeans_ker") == [L.V_BOUNDS] * 5


def _strip_pre(prog, fn):
    d = ir.to_json(prog)
    for f in d["defs"]:
        if f["name"] == fn:
            for p in f["params"]:
                p["pre"] = None
    return ir.from_json(d)


def test_unannotated_copy_never_inherits_verdicts():
    """The same body with its annotations removed (or a different postcondition)
    is not in the table: all CHECKED, never the corpus verdict."""
    for key, fn in (("ref:kmeans_ker.ixl", "kmeans_ker"), ("own:c4_csr_gather.ixl", "csrg"),
                    ("own:c3_scatter.ixl", "sc_bij"), ("ref:maxmatching.ixl", "get_smallest_pairs")):
        p = _strip_pre(_prog(key), fn)
        fs = sel.selection_for(p, ir.find_def(p, fn), live=False)
        assert not fs.elides, (key, fn, fs.source)


def test_redefined_callee_changes_caller_key():
    """A caller's verdicts come from its callees' analysis (infer.py:1387-1420):
    redefining a helper must change the caller's key, so the caller does not
    inherit the corpus verdicts."""
    prog = _prog("ref:maxmatching.ixl")
    gsp = ir.find_def(prog, "get_smallest_pairs")
    assert sel.selection_for(prog, gsp, live=False).source == "frozen"
    d = ir.to_json(prog)
    for f in d["defs"]:
        if f["name"] == "filter_by":  # a different helper under the same name
            f["body"] = {"$": "VarE", "name": "xs", "pos": [1, 1]}
    prog2 = ir.from_json(d)
    assert ir.fingerprint(ir.find_def(prog2, "get_smallest_pairs")) == ir.fingerprint(gsp)
    assert ir.closure_fingerprint(prog2, ir.find_def(prog2, "get_smallest_pairs")) != ir.closure_fingerprint(prog, gsp)
    assert sel.selection_for(prog2, ir.find_def(prog2, "get_smallest_pairs"), live=False).source == "checked"


@pytest.mark.reference
def test_live_verifier_wins_over_frozen(reference):
    """With the reference importable, a reference AST is verified live, even
    when the frozen table holds the same key."""
    from ixverify.normalize import normalize
    from ixverify.parser import parse_program

    src = PROGRAMS["own:kmeans_noann.ixl"]["source"]
    prog = normalize(parse_program(src, "kmeans_noann.ixl"))
    fs = sel.selection_for(prog, ir.find_def(prog, "kmeans_ker"))
    assert fs.source == "live" and [s.bits for s in fs.sites] == [L.V_BOUNDS] * 5
    src = PROGRAMS["ref:kmeans_ker.ixl"]["source"]
    prog = normalize(parse_program(src, "kmeans_ker.ixl"))
    fs = sel.selection_for(prog, ir.find_def(prog, "kmeans_ker"))
    assert fs.source == "live" and [s.bits for s in fs.sites] == [0] * 5


def test_contract_host_side():
    """The host half of the precondition check: sizes, scalar annotations,
    intervals with inf (contract.py; oracle.py:712-734)."""
    from paper_2506_23058_b200 import contract

    prog = _prog("ref:kmeans_ker.ixl")
    f = ir.find_def(prog, "kmeans_ker")
    env = contract.bind_sizes(f, {"pointers": [0, 1, 2], "values": [0.5], "indices": [0], "cluster": [1.0, 2.0]})
    assert env["n"] == 2 and env["nnz"] == 1 and env["num_cols"] == 2
    row_pre = f.params[0].pre
    atom = next(contract.conjuncts(row_pre))
    assert contract._atom(atom, {**env, "row": 1}) is True
    assert contract._atom(atom, {**env, "row": 2}) is False
    assert contract._atom(atom, {**env, "row": -1}) is False
    ok, why = contract.check(f, {"row": 5, "pointers": [0, 1, 2]})
    assert not ok and "row" in why
    gsp = ir.find_def(_prog("ref:maxmatching.ixl"), "get_smallest_pairs")
    inj = list(contract.conjuncts(gsp.params[3].pre))[0]
    lo, hi = contract._interval(inj.args[1], {})
    assert lo == float("-inf") and hi == float("inf")
    assert contract._clamp_int(lo, hi, -5, 9) == (-5, 9)
    assert contract._clamp_int(0, 3, -5, 9) == (0, 3)


def test_required_annotations_by_ablation():
    """Only the annotations some elision depends on are checked at run time
    (select.required_atoms: the verifier re-run with each conjunct dropped).
    get_smallest_pairs' `Inj is (-inf, inf)` backs no elided check (the
    H[i] gather needs `Range es` only), so an input violating it still runs
    ELIDED; kmeans_ker needs all three of its Range annotations."""
    from paper_2506_23058_b200 import contract

    gsp = SELECTION["ref:maxmatching.ixl:get_smallest_pairs"]
    assert gsp["required"] == ["es|Range es ((0, n_verts - 1))"]
    km = SELECTION["ref:kmeans_ker.ixl:kmeans_ker"]
    assert len(km["required"]) == 3 and all(r.split("|")[1].startswith("Range") for r in km["required"])
    assert SELECTION["own:c3_scatter.ixl:sc_inj"]["required"] == ["is|Inj is ((0, n - 1))"]
    # the frozen verdict carries the list; nothing left to check -> no device work at all
    prog = _prog("ref:maxmatching.ixl")
    f = ir.find_def(prog, "get_smallest_pairs")
    fs = sel.selection_for(prog, f, live=False)
    assert fs.source == "frozen" and fs.required == gsp["required"]
    assert contract.check(f, {}, required=[]) == (True, "")
    assert not contract.has_preconditions(f, required=[]) and contract.has_preconditions(f)


@pytest.mark.reference
def test_required_annotations_live(reference):
    """The live selector computes the same required set as the frozen table."""
    from ixverify.normalize import normalize
    from ixverify.parser import parse_program

    src = PROGRAMS["ref:maxmatching.ixl"]["source"]
    prog = normalize(parse_program(src, "maxmatching.ixl"))
    fs = sel.selection_for(prog, ir.find_def(prog, "get_smallest_pairs"))
    assert fs.source == "live" and fs.required == ["es|Range es ((0, n_verts - 1))"]
