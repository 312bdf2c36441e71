"""Selector: the reference verifier's proved obligations -> kernel variant
bits per source site.

The verifier (``ixverify.infer.Analyzer``, /root/reference/pkg/src/ixverify/
infer.py:172-226) records an ``Obligation(kind, pos, text, proved)``
(infer.py:132-137) for every indexing site (two ``bounds`` obligations,
``_bounds_check`` infer.py:612-632) and every scatter (one
``scatter-safety`` obligation via Ss1/Ss2/Ss3, infer.py:1091-1100,
1129-1143).  ``analyze_program`` stops at the first failure, so the
selector runs ``Analyzer.analyze_fun`` per definition itself and keeps the
partial obligation list of a failing definition.

Per site:
  * bounds site  -> ELIDED iff every obligation recorded at its pos is proved;
  * scatter site -> the idempotence check is ELIDED iff scatter-safety is
    proved; destination init + OOB test are ELIDED only when the result is
    the Sc1 bijection ``for i < n . true => x[is^-1[i]]`` (detected with
    ``props._inv_pattern`` on the bound result, props.py:561-578,
    infer.py:1101-1122) -- Sc1 is not itself an Obligation.
  * unrecorded sites (after a failure, or in callers of a failed callee) are
    CHECKED.

The verifier only exists where the reference is installed; the verdicts for
the bundled corpus are frozen in ``data/selection.json`` (keyed by
``ir.closure_fingerprint``: body, annotations and callees) so the GPU box
can select without it.  The live verifier always wins when it is
importable; a frozen key held with two different verdicts is dropped.
"""

from __future__ import annotations

import json
import os
import sys
from dataclasses import asdict, dataclass, field
from typing import Optional

from . import _lib as L
from . import ir

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
REFERENCE_SRC = os.environ.get("IXVERIFY_SRC", "/root/reference/pkg/src")


@dataclass
class SiteVerdict:
    kind: str  # "bounds" | "scatter-safety"
    pos: tuple
    text: str
    recorded: bool = False
    proved: bool = False
    rule: str = ""
    sc1: bool = False

    @property
    def bits(self) -> int:
        if self.kind == "bounds":
            return 0 if (self.recorded and self.proved) else L.V_BOUNDS
        b = 0
        if not (self.recorded and self.proved):
            b |= L.V_CONFLICT
        if not self.sc1:
            b |= L.V_INIT
        return b


@dataclass
class FunSelection:
    name: str
    fingerprint: str
    status: str
    sites: list = field(default_factory=list)
    closure: str = ""  # ir.closure_fingerprint: the key the verdicts are valid for
    source: str = ""   # "live" | "frozen" | "checked" (where these verdicts came from)
    # the parameter annotations the elided sites' proofs need ("param|atom",
    # see required_atoms); None = all of them (no ablation ran)
    required: Optional[list] = None

    @property
    def elides(self) -> bool:
        """does any site run without its check?"""
        return any(s.bits != (L.V_BOUNDS if s.kind == "bounds" else L.V_CONFLICT | L.V_INIT) for s in self.sites)

    def bits(self, ordinal: int) -> int:
        return self.sites[ordinal].bits

    def by_pos(self, pos) -> Optional[SiteVerdict]:
        for s in self.sites:
            if tuple(s.pos) == tuple(pos):
                return s
        return None

    def to_json(self):
        d = asdict(self)
        d.pop("source", None)
        for s in d["sites"]:
            s["pos"] = list(s["pos"])
        return d

    @classmethod
    def from_json(cls, d):
        sites = [SiteVerdict(**{**s, "pos": tuple(s["pos"])}) for s in d["sites"]]
        return cls(d["name"], d["fingerprint"], d["status"], sites, d.get("closure", ""), "", d.get("required"))


@dataclass
class Selection:
    funcs: dict

    def __getitem__(self, name) -> FunSelection:
        return self.funcs[name]

    def to_json(self):
        return {k: v.to_json() for k, v in self.funcs.items()}


def _import_reference():
    if REFERENCE_SRC not in sys.path and os.path.isdir(REFERENCE_SRC):
        sys.path.insert(0, REFERENCE_SRC)
    import ixverify.infer as infer  # noqa: F401
    import ixverify.props as props  # noqa: F401

    return sys.modules["ixverify.infer"], sys.modules["ixverify.props"]


def reference_available() -> bool:
    try:
        _import_reference()
        return True
    except Exception:
        return False


def _scatter_result_names(fundef):
    """pos of each scatter App -> the let-bound name of its result."""
    out = {}

    def walk(e):
        if ir.kind(e) == "Let" and len(e.names) == 1:
            r = e.rhs
            if ir.kind(r) == "App" and ir.kind(r.fun) == "VarE" and r.fun.name == "scatter":
                out[tuple(r.pos)] = e.names[0]
        for c in ir.children(e):
            walk(c)

    walk(fundef.body)
    return out


def _analyze(a, infer, props, f):
    """(status, site verdicts, FunInfo or None) of one definition."""
    status, info = "verified", None
    try:
        info = a.analyze_fun(f)
    except infer.InferError as exc:  # keep the partial obligation list
        status = f"failed: {type(exc).__name__}: {exc}"
    obls = list(getattr(a, "obligations", []))
    names = _scatter_result_names(f)
    sites = []
    for kind, pos, node in ir.sites(f):
        rec = [o for o in obls if tuple(o.pos) == pos and o.kind == kind]
        v = SiteVerdict(kind, pos, ir.expr_str(node), recorded=bool(rec), proved=bool(rec) and all(o.proved for o in rec))
        if kind == "scatter-safety" and rec:
            v.rule = rec[0].text.replace("scatter via ", "").replace("scatter", "").strip()
            nm = names.get(pos)
            if v.proved and info is not None and nm in info.gamma:
                try:
                    v.sc1 = props._inv_pattern(info.gamma[nm]) is not None
                except Exception:
                    v.sc1 = False
        sites.append(v)
    return status, sites, info


def atom_key(param_name: str, atom) -> str:
    """The identity of one annotation conjunct (same text for the reference's
    AST and this package's IR mirror)."""
    return f"{param_name}|{ir.expr_str(atom)}"


def _conjuncts(e):
    if ir.kind(e) == "BinOp" and e.op == "&&":
        yield from _conjuncts(e.lhs)
        yield from _conjuncts(e.rhs)
    else:
        yield e


def required_atoms(a, infer, props, f, base_bits) -> Optional[list]:
    """Which parameter annotations do the verdicts depend on?  Ablation with
    the verifier itself: drop one conjunct at a time and re-analyze; a
    conjunct whose removal leaves every site's bits unchanged is not needed
    by any elision.  The conjuncts found free one by one are then dropped
    TOGETHER and re-checked (two may each be redundant only given the
    other); if that changes any bits, every conjunct stays required.  Only
    the required ones are checked on the device before ELIDED variants run
    (contract.py) -- an annotation no proof used cannot make an elided
    check unsafe."""
    import dataclasses

    atoms = [(pi, k, atom) for pi, q in enumerate(f.params) if q.pre is not None
             for k, atom in enumerate(_conjuncts(q.pre))]
    if not atoms:
        return []
    mod = sys.modules[type(atoms[0][2]).__module__]

    def bits_without(drop):
        params = list(f.params)
        for pi, q in enumerate(f.params):
            if q.pre is None:
                continue
            keep = [atom for k, atom in enumerate(_conjuncts(q.pre)) if (pi, k) not in drop]
            pre = None
            for atom in keep:
                pre = atom if pre is None else mod.BinOp("&&", pre, atom, atom.pos)
            params[pi] = dataclasses.replace(q, pre=pre)
        try:
            _, sites, _ = _analyze(a, infer, props, dataclasses.replace(f, params=tuple(params)))
        except Exception:
            return None
        return [s.bits for s in sites]

    free = {(pi, k) for pi, k, _ in atoms if bits_without({(pi, k)}) == base_bits}
    if free and len(free) > 1 and bits_without(free) != base_bits:
        free = set()
    return [atom_key(f.params[pi].name, atom) for pi, k, atom in atoms if (pi, k) not in free]


def select(program, max_rewrites: int = 1000, ablate: bool = True) -> Selection:
    """Run the reference verifier per definition and derive site verdicts.
    `program` must be the reference's normalized Program."""
    infer, props = _import_reference()
    a = infer.Analyzer(program, max_rewrites=max_rewrites)
    funcs = {}
    for f in program.defs:
        status, sites, info = _analyze(a, infer, props, f)
        if info is not None:
            a.infos[f.name] = info
        fs = FunSelection(f.name, ir.fingerprint(f), status, sites, ir.closure_fingerprint(program, f), "live")
        if ablate and fs.elides:
            fs.required = required_atoms(a, infer, props, f, [s.bits for s in sites])
        funcs[f.name] = fs
    return Selection(funcs)


# ----------------------------------------------------------------- frozen
_FROZEN = None
AMBIGUOUS: set = set()  # closure keys the frozen table holds with conflicting verdicts


def _verdict_key(fs: FunSelection):
    # the status text carries source positions; compare its class only
    return (":".join(fs.status.split(":")[:2]), tuple((s.kind, s.recorded, s.proved, s.sc1) for s in fs.sites))


def frozen() -> dict:
    """closure fingerprint -> FunSelection for the bundled corpus
    (data/selection.json).  A key that occurs with two different verdicts is
    dropped (it selects all-CHECKED), never resolved by load order."""
    global _FROZEN
    if _FROZEN is None:
        path = os.path.join(DATA, "selection.json")
        table: dict = {}
        if os.path.exists(path):
            with open(path) as fh:
                for d in json.load(fh).values():
                    fs = FunSelection.from_json(d)
                    if not fs.closure:
                        continue  # a verdict without its contract key is never trusted
                    prev = table.get(fs.closure)
                    if prev is not None and _verdict_key(prev) != _verdict_key(fs):
                        AMBIGUOUS.add(fs.closure)
                    table.setdefault(fs.closure, fs)
        for k in AMBIGUOUS:
            table.pop(k, None)
        _FROZEN = table
    return _FROZEN


_SEL_CACHE: dict = {}  # (id(program), id(fundef), live | checked) -> (program, fundef, selection)
_LIVE_CACHE: dict = {}  # id(program) -> (program, Selection)


def _cached(key, program, fundef, make):
    hit = _SEL_CACHE.get(key)
    if hit is not None and hit[0] is program and hit[1] is fundef:
        return hit[2]
    v = make()
    if len(_SEL_CACHE) > 4096:
        _SEL_CACHE.clear()
    _SEL_CACHE[key] = (program, fundef, v)
    return v


def checked_selection(fundef) -> FunSelection:
    """Every site CHECKED: the reference interpreter's own behaviour."""
    return _cached((None, id(fundef), "checked"), None, fundef, lambda: _checked_selection(fundef))


def _checked_selection(fundef) -> FunSelection:
    sites = [SiteVerdict(k, pos, ir.expr_str(n)) for k, pos, n in ir.sites(fundef)]
    return FunSelection(fundef.name, ir.fingerprint(fundef), "checked (no verdict)", sites, "", "checked")


def selection_for(program, fundef, live: bool = True) -> FunSelection:
    """Verdicts for one function, in this order:
      1. the live reference verifier, whenever it is importable and
         `program` is the reference's own AST (run once per program);
      2. the frozen corpus table, matched on the closure fingerprint (body,
         annotations and every callee, ``ir.closure_fingerprint``) -- an
         unannotated or re-annotated copy of a corpus function, or one whose
         helper was redefined, never inherits the corpus verdicts;
      3. otherwise every site CHECKED.
    Memoised per program and function object."""
    return _cached((id(program), id(fundef), live), program, fundef, lambda: _selection_for(program, fundef, live))


def _live(program) -> Selection:
    hit = _LIVE_CACHE.get(id(program))
    if hit is not None and hit[0] is program:
        return hit[1]
    s = select(program)
    if len(_LIVE_CACHE) > 256:
        _LIVE_CACHE.clear()
    _LIVE_CACHE[id(program)] = (program, s)
    return s


def _selection_for(program, fundef, live: bool) -> FunSelection:
    if live and program is not None and type(program).__module__.startswith("ixverify") and reference_available():
        fs = _live(program).funcs.get(fundef.name)
        if fs is not None:
            return fs
    if program is not None:
        key = ir.closure_fingerprint(program, fundef)
        fz = frozen().get(key)
        if fz is not None:
            # positions may differ from the frozen source: re-key by ordinal
            cur = ir.sites(fundef)
            if len(cur) == len(fz.sites) and all(a.kind == k for a, (k, _, _) in zip(fz.sites, cur)):
                sites = [SiteVerdict(**{**asdict(s), "pos": pos}) for s, (_, pos, _) in zip(fz.sites, cur)]
                return FunSelection(fundef.name, fz.fingerprint, fz.status, sites, key, "frozen", fz.required)
    return checked_selection(fundef)
