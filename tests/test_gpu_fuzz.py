"""Random programs (tests/golden/fuzz.json, made by make_fuzz.py from the
Python reference itself) through the drop-in: maps with captured tables and
scalars, scans and hists with arbitrary operators, loops -- every lambda
compiled by jit.py / jit_fold.py.  Results, exception classes and
OutOfBounds sites/positions must equal the reference's."""

import json
import os

import pytest

from paper_2506_23058_b200 import errors, ir

import bigtrack

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FUZZ = json.load(open(os.path.join(HERE, "golden", "fuzz.json")))
_PROGS = {}


def _program(key):
    if key not in _PROGS:
        _PROGS[key] = ir.from_json(FUZZ["programs"][key]["program"])
    return _PROGS[key]


@pytest.mark.parametrize("idx", range(len(FUZZ["cases"])))
def test_fuzz_program(cuda, idx):
    from paper_2506_23058_b200.executor import eval_program

    case = FUZZ["cases"][idx]
    prog = _program(case["program"])
    if case.get("big"):  # the reference left int64: IntegerOverflow, or still its exact answer
        try:
            got = eval_program(prog, case["fun"], case["args"], variant="checked")
        except errors.IntegerOverflow:
            return
        except errors.OracleError as ex:
            assert "error" in case and type(ex).__name__ == case["error"], ex
            return
        assert "result" in case and bigtrack.fits(case["result"]) and got == case["result"], (got, case)
        return
    if "error" in case:
        with pytest.raises(getattr(errors, case["error"])) as ei:
            eval_program(prog, case["fun"], case["args"], variant="checked")
        if "site" in case:
            assert ei.value.site == case["site"]
        if "pos" in case:
            assert list(ei.value.pos) == case["pos"]
        return
    got = eval_program(prog, case["fun"], case["args"], variant="checked")
    assert got == case["result"], (FUZZ["programs"][case["program"]]["source"], case["args"], got, case["result"])
