import sys, numpy as np, warnings
sys.path.insert(0, '.')
import paper_2510_03421_b200 as R
tests = {
 "nan": np.array([[1.0, np.nan],[2.0, 3.0]]),
 "inf": np.array([[np.inf, 1.0],[1.0, 1.0]]),
 "neginf_sq3": np.array([[1.0,2,3],[4,-np.inf,6],[7,8,9]]),
 "tiny": np.full((4,4), 1e-300),
 "huge": np.full((4,4), 1e300),
 "zeros": np.zeros((5,5)),
 "rect_nan": np.array([[1.0, np.nan, 2.0]]),
 "nan_20": np.where(np.eye(20) > 0, np.nan, 0.5),
 "tiny_20": np.full((20, 20), 1e-20),
 "huge_20": np.full((20, 20), 1e20),
 "zeros_21": np.zeros((21, 21)),
}
for k,a in tests.items():
    out=[]
    for fn in (R.combinatoric, R.ryser, R.glynn, R.opt):
        try: out.append(repr(fn(a)))
        except Exception as e: out.append(type(e).__name__+":"+str(e)[:40])
    print(k, out, flush=True)
