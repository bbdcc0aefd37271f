import csv, io, sys
sys.path.insert(0, '.')
from paper_2510_03421_b200 import precision as PR
from collections import defaultdict
def rows(text): return {(r["family"], r["algorithm"], int(r["m"]), int(r["n"]), r["kind"]): r for r in csv.DictReader(io.StringIO(text))}
ref = rows(open('tests/golden/precision_ref.csv').read())
txt = PR.precision_csv(PR.run_precision_suite(n_range=range(2, 17), seed=0, cauchy_attempts=200))
open('gpurun_out/precision_b200.csv','w').write(txt)
ours = rows(txt)
worst = defaultdict(lambda: [-9, -9]); diffs = defaultdict(list)
for k, r in ref.items():
    o = ours[k]
    if r["overflow"] == "true" or o["overflow"] == "true": continue
    dr, do = float(r["digits_lost"]), float(o["digits_lost"])
    g = (k[0], k[1], k[4]); worst[g][0] = max(worst[g][0], dr); worst[g][1] = max(worst[g][1], do); diffs[g].append(do - dr)
    if do > max(dr, 0) + 0.5: print("worse", k, round(do, 2), round(dr, 2))
for g in sorted(worst): print(g, "ref max %.2f ours max %.2f  mean diff %.2f" % (worst[g][0], worst[g][1], sum(diffs[g]) / len(diffs[g])))
