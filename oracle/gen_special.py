"""Golden outputs of the reference on non-finite / extreme inputs (run HERE,
where /root/reference exists): tests/golden/special_values.json.

    NUMBA_CACHE_DIR=/tmp/nb PYTHONPATH=/root/reference/pkg/src python oracle/gen_special.py

Each case records repr() of combinatoric / ryser / glynn (the reference's
float kernels all start their sums at zero = a[0,0] - a[0,0],
src/_kernels.py:30/117/228/375/533, so a non-finite a[0,0] gives NaN even
where the algebra gives +-inf; signed zeros follow Ryser's (-1)^n)."""
import json
import warnings
from pathlib import Path

import numpy as np
import permanent as R

warnings.filterwarnings("ignore")
CASES = {
    "nan_2x2": [[1.0, float("nan")], [2.0, 3.0]],
    "inf_a00_2x2": [[float("inf"), 1.0], [1.0, 1.0]],
    "inf_a01_2x2": [[1.0, float("inf")], [1.0, 1.0]],
    "neginf_3x3": [[1.0, 2.0, 3.0], [4.0, float("-inf"), 6.0], [7.0, 8.0, 9.0]],
    "tiny_4x4": [[1e-300] * 4] * 4,
    "huge_4x4": [[1e300] * 4] * 4,
    "zeros_5x5": [[0.0] * 5] * 5,
    "zeros_4x4": [[0.0] * 4] * 4,
    "rect_nan_1x3": [[1.0, float("nan"), 2.0]],
    "rect_inf_a00_2x4": [[float("inf"), 1.0, 2.0, 3.0], [1.0, 1.0, 1.0, 1.0]],
    "complex_inf_re_2x2": [[complex(float("inf"), 1.0), 1.0], [1.0, 1.0]],
}
out = {}
for k, rows in CASES.items():
    a = np.array(rows, dtype=complex if any(isinstance(x, complex) for r in rows for x in r) else float)
    rec = {"matrix": [[repr(x) for x in r] for r in rows], "complex": bool(np.iscomplexobj(a))}
    for name in ("combinatoric", "ryser", "glynn"):
        rec[name] = repr(getattr(R, name)(a))
    out[k] = rec
path = Path(__file__).resolve().parents[1] / "tests" / "golden" / "special_values.json"
path.write_text(json.dumps(out, indent=1))
print(json.dumps(out, indent=1))
