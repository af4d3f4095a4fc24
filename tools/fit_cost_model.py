"""Fit simulate.COST_COEF: per policy, least squares of log(device cycles) on
[1, log n, log rho, log iterations_est, (log rho)^2] (simulate.cost_features) over a C4
sweep the bench does not run (seeds 100-115, tools/dump_c4_costs.py ... 100), and report
the held-out rank correlation on the bench's own sweep (seeds 0-15).
usage: python tools/fit_cost_model.py FIT.npz [TEST.npz] > profiles/r02_cost_model.json"""
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
    f = simulate.cost_features(b)
    ln, lr, li = np.log(f[:, 0]), np.log(f[:, 1]), np.log(f[:, 2])
    X = np.stack([np.ones(len(f)), ln, lr, li, lr * lr], 1)
    return b, X, d["warm_device_cycles"].astype(np.float64), s0


b, X, y, s0 = load(sys.argv[1])
pol = b.instances["engine"]["policy"]
coef = np.zeros((4, 5))
rep = {"fit_seeds": [s0, s0 + 15], "policies": {}}
for p in range(4):
    m = pol == p
    coef[p], *_ = np.linalg.lstsq(X[m], np.log(y[m]), rcond=None)
    rep["policies"][NAMES[p]] = {"coef": [round(float(c), 3) for c in coef[p]],
                                 "fit_spearman": float(spearmanr(X[m] @ coef[p], y[m]).statistic)}
if len(sys.argv) > 2:
    bt, Xt, yt, st0 = load(sys.argv[2])
    rep["test_seeds"] = [st0, st0 + 15]
    pt = bt.instances["engine"]["policy"]
    old = None
    for p in range(4):
        m = pt == p
        pr = Xt[m] @ coef[p]
        rep["policies"][NAMES[p]]["test_spearman"] = float(spearmanr(pr, yt[m]).statistic)
        rep["policies"][NAMES[p]]["test_rel_err_p50_p90"] = [float(v) for v in
                                                           np.percentile(abs(np.exp(pr) / yt[m] - 1), [50, 90])]
print(json.dumps(rep, indent=1))
print("COST_COEF = " + repr(np.round(coef, 3).tolist()), file=sys.stderr)
