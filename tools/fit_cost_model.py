"""Fit simulate.ITER_COEF / CYCLES_PER_ITER, the first-run (cold) scheduling model.

The measured (warm) schedule orders each policy's instances by iterations x the policy's mean
device cycles per iteration, and that ordering is what a first run should reproduce. Iterations
are deterministic (no contention noise, unlike per-instance device cycles, whose rank
correlation with the work is ~0 within a policy), so per policy: least squares of
log(iterations) on simulate.cost_design(batch) over two C4 sweeps the bench does not run
(seeds 100-115 and 200-215, tools/dump_c4_costs.py), and each policy's mean device cycles per
iteration (for the SM split between policies). Reports the held-out rank correlation on the
bench's own sweep (seeds 0-15).
usage: python tools/fit_cost_model.py FIT.npz [FIT2.npz ...] --test TEST.npz > profiles/r02_cost_model.json"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from scipy.stats import spearmanr

from paper_2410_17840_b200 import configs as C
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate

NAMES = ("fcfs", "nopreempt", "trail_plus", "larry")


def load(path):
    d = np.load(path)
    s0 = int(d["first_seed"]) if "first_seed" in d else 0
    b = I.make_batch(C.c4_jobs(seeds=range(s0, s0 + 16)))
    return b, simulate.cost_design(b), d["warm_iterations"].astype(np.float64), d["warm_device_cycles"].astype(np.float64), s0


args = sys.argv[1:]
test = None
if "--test" in args:
    test = args[args.index("--test") + 1]
    args = [a for a in args if a not in ("--test", test)]
data = [load(a) for a in args]
pol = np.concatenate([d[0].instances["engine"]["policy"] for d in data])
X = np.concatenate([d[1] for d in data])
it = np.concatenate([d[2] for d in data])
cyc = np.concatenate([d[3] for d in data])
coef = np.zeros((4, X.shape[1]))
cpi = np.zeros(4)
rep = {"fit_seeds": [d[4] for d in data], "target": "log iterations", "policies": {}}
for p in range(4):
    m = pol == p
    coef[p], *_ = np.linalg.lstsq(X[m], np.log(it[m]), rcond=None)
    cpi[p] = cyc[m].sum() / it[m].sum()
    rep["policies"][NAMES[p]] = {"coef": [round(float(c), 4) for c in coef[p]], "cycles_per_iteration": round(float(cpi[p]), 1),
                                 "fit_spearman": float(spearmanr(X[m] @ coef[p], it[m]).statistic)}
if test:
    bt, Xt, itt, _, st0 = load(test)
    rep["test_seeds"] = st0
    pt = bt.instances["engine"]["policy"]
    for p in range(4):
        m = pt == p
        pr = Xt[m] @ coef[p]
        rep["policies"][NAMES[p]]["test_spearman"] = float(spearmanr(pr, itt[m]).statistic)
        rep["policies"][NAMES[p]]["test_rel_err_p50_p90"] = [float(v) for v in
                                                           np.percentile(abs(np.exp(pr) / itt[m] - 1), [50, 90])]
print(json.dumps(rep, indent=1))
print("ITER_COEF = " + repr(np.round(coef, 4).tolist()), file=sys.stderr)
print("CYCLES_PER_ITER = " + repr(np.round(cpi, 1).tolist()), file=sys.stderr)
