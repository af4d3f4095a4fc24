"""Generate the golden parity fixtures by running the PYTHON REFERENCE.

Run in the build container (the only place /root/reference exists):
    python tests/golden/make_golden.py [group ...]

For every scenario of tests/scenarios.py this imports servesim read-only from
/root/reference/pkg/src, runs it through the reference's own entry point
(Engine(...).run, engine.py:236, or run_cluster(..., engines=...),
cluster.py:65-79) and records:
  * counters: Σ iterations (engine.py:226), Σ request-steps and Σ batch tokens
    (a wrapper around Engine._form_batch, engine.py:300-323 — no reference edits),
    dispatch / preempt / park / finish event counts, peak batch tokens;
  * the decision digest: FNV-1a over each engine's event_log (engine.py:165,273)
    folded in server order (tests/golden_util.py);
  * a sha256 of the records (first_token, finish, preempt_count, server);
  * summarize() (metrics.py:80-99) of the records;
  * per engine: iterations, request-steps, batch tokens, peak batch tokens;
  * for the small groups, the full records, event streams and event_lines().
Output: tests/golden/<group>.json (committed). Nothing at test or bench time
reads /root/reference.
"""

from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from servesim import metrics as ref_metrics  # noqa: E402
from servesim.balancers import make_balancer  # noqa: E402,F401
from servesim.cluster import run_cluster  # noqa: E402
from servesim.config import BalancerSettings, ClusterSettings, EngineSettings  # noqa: E402
from servesim.costmodel import CostParams  # noqa: E402
from servesim.engine import Engine  # noqa: E402
from servesim.kvmem import KvBlockPool  # noqa: E402
from servesim.policies import make_policy  # noqa: E402
from servesim.workload import LengthDist, SynthSpec, TraceEntry, scale_qps, synthesize  # noqa: E402

import scenarios as S  # noqa: E402
from golden_util import EVENT_CODES, event_digest, fold_digests, records_sha, trace_sha  # noqa: E402

FULL_RECORD_GROUPS = {"engine_unit", "cluster_unit", "hetero"}
LEAN_GROUPS = {"c6", "c2", "c3"}  # many tiny instances: counters + digests only

_orig_form_batch = Engine._form_batch


def _counting_form_batch(self):
    plan = _orig_form_batch(self)
    self._g_rsteps = getattr(self, "_g_rsteps", 0) + len(plan.decode_ids) + len(plan.prefill_chunks)
    self._g_btok = getattr(self, "_g_btok", 0) + plan.total_tokens
    return plan


Engine._form_batch = _counting_form_batch


def make_trace(sc):
    t = sc["trace"]
    if "rows" in t:
        entries = [TraceEntry(a, p, o) for a, p, o in t["rows"]]
    else:
        kw = dict(t["synth"])
        for k in ("prompt_dist", "output_dist"):
            if k in kw:
                kw[k] = LengthDist(**kw[k])
        entries = synthesize(SynthSpec(**kw))
    if sc["qps_factor"] != 1.0:
        entries = scale_qps(entries, sc["qps_factor"])
    return entries


def _n_rows(sc):
    return len(sc["trace"]["rows"]) if "rows" in sc["trace"] else 10**9


def make_engine(e):
    return Engine(
        KvBlockPool(e["pool_blocks"], e["block_size"]),
        make_policy(e["policy"], alpha=e["alpha"], c=e["c"], max_output=e["max_output"]),
        CostParams(*e["cost"]),
        max_tokens_per_batch=e["cap"],
        max_running=e["max_running"],
        max_context=e["max_context"],
    )


def run_scenario(sc, full: bool):
    trace = make_trace(sc)
    e = sc["engine"]
    c = sc["cluster"]
    t0 = time.perf_counter()
    if sc["mode"] == "engine":
        engines = [make_engine(e)]
        records = engines[0].run(trace)
    else:
        settings = ClusterSettings(
            n_servers=c["n_servers"],
            engine=EngineSettings(max_tokens_per_batch=c.get("route_cap", e["cap"])),
            balancer=BalancerSettings(name=c["balancer"], poll_interval_s=c["poll_interval_s"],
                                      beta_prior=c["beta_prior"], beta_fixed=c["beta_fixed"]),
            seed=c["seed"],
        )
        engines = ([make_engine(x) for x in sc["engines"]] if "engines" in sc  # heterogeneous prebuilt engines
                   else [make_engine(e) for _ in range(c["n_servers"])])
        records = run_cluster(settings, trace, engines=engines)
    wall = time.perf_counter() - t0
    ev_lists = [[(EVENT_CODES[ev], rid, t) for ev, t, rid, _ in eng.event_log] for eng in engines]
    counts = {k: 0 for k in EVENT_CODES}
    for eng in engines:
        for ev, *_ in eng.event_log:
            counts[ev] += 1
    arr = np.array([x.arrival_time for x in trace], dtype=np.float64)
    out = {
        "name": sc["name"],
        "n_requests": len(records),
        "trace_sha": trace_sha(arr, [x.prompt_len for x in trace], [x.output_len for x in trace]),
        "iterations": sum(eng.iterations for eng in engines),
        "request_steps": sum(getattr(eng, "_g_rsteps", 0) for eng in engines),
        "batch_tokens": sum(getattr(eng, "_g_btok", 0) for eng in engines),
        "dispatches": counts["dispatch"],
        "preempts": counts["preempt"],
        "parks": counts["park"],
        "finished": counts["finish"],
        "peak_batch_tokens": max(eng.peak_batch_tokens for eng in engines),
        "digest": "%016x" % fold_digests([event_digest(ev) for ev in ev_lists]),
        "records_sha": records_sha([r.first_token_time for r in records], [r.finish_time for r in records],
                                   [r.preempt_count for r in records], [r.server for r in records]),
        "summary": ref_metrics.summarize(records).to_dict() if records else None,
        "ref_wall_s": wall,
        # per engine (server order): iterations (engine.py:226), request-steps, batch tokens,
        # peak_batch_tokens (engine.py:225) — the criterion-8 audit is per engine (test_acceptance.py:371-382)
        "per_engine": [[eng.iterations, getattr(eng, "_g_rsteps", 0), getattr(eng, "_g_btok", 0),
                        eng.peak_batch_tokens] for eng in engines],
    }
    if full:
        out["records"] = [[r.first_token_time, r.finish_time, r.preempt_count, r.server] for r in records]
        out["events"] = [[[code, rid, t] for code, rid, t in ev] for ev in ev_lists]
        out["event_lines"] = [eng.event_lines() for eng in engines]  # engine.py:267-269, incl. seq=/count=
    return out


def _json_default(o):
    if isinstance(o, float) and (math.isinf(o) or math.isnan(o)):
        return repr(o)
    raise TypeError(o)


def main(groups):
    for g in groups:
        scs = S.GROUPS[g]()
        t0 = time.perf_counter()
        res = []
        for sc in scs:
            try:
                r = run_scenario(sc, g in FULL_RECORD_GROUPS and _n_rows(sc) <= 200)
                if g in LEAN_GROUPS:
                    for k in ("summary", "ref_wall_s", "trace_sha"):
                        r.pop(k)
                res.append(r)
            except Exception as exc:  # the reference's own error is the golden
                res.append({"name": sc["name"], "error": type(exc).__name__, "message": str(exc)})
        dt = time.perf_counter() - t0
        path = HERE / f"{g}.json"
        path.write_text(json.dumps({"group": g, "generator": "tests/golden/make_golden.py",
                                    "reference": "/root/reference/pkg/src/servesim", "n": len(res),
                                    "results": res}, indent=None, separators=(",", ":")) + "\n")
        print(f"{g}: {len(res)} scenarios in {dt:.1f}s -> {path} ({path.stat().st_size/1e3:.0f} kB)")


if __name__ == "__main__":
    main(sys.argv[1:] or list(S.GROUPS))
