"""Build ssb_instance batches from tests/scenarios.py dicts and compare results
with the golden fixtures produced by the Python reference."""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
TESTS = Path(__file__).resolve().parent
for p in (str(ROOT), str(TESTS)):
    if p not in sys.path:
        sys.path.insert(0, p)

from golden_util import fold_digests, records_sha, trace_sha  # noqa: E402
from paper_2410_17840_b200 import instances as I  # noqa: E402
from paper_2410_17840_b200.policies import EngineLimits, make_policy  # noqa: E402
from paper_2410_17840_b200.settings import BalancerSettings, ClusterSettings, CostParams, EngineSettings  # noqa: E402
from paper_2410_17840_b200.workload import LengthDist, SynthSpec, Trace, synthesize  # noqa: E402

GOLDEN = TESTS / "golden"
_trace_cache: dict = {}


def load_golden(group: str) -> dict:
    d = json.loads((GOLDEN / f"{group}.json").read_text())
    return {r["name"]: r for r in d["results"]}


def scenario_trace(sc) -> Trace:
    t = sc["trace"]
    if "rows" in t:
        r = np.array(t["rows"], dtype=np.float64).reshape(-1, 3)
        return Trace(r[:, 0], r[:, 1].astype(np.int64), r[:, 2].astype(np.int64))
    key = json.dumps(t["synth"], sort_keys=True)
    if key not in _trace_cache:
        kw = dict(t["synth"])
        for k in ("prompt_dist", "output_dist"):
            if k in kw:
                kw[k] = LengthDist(**kw[k])
        _trace_cache[key] = synthesize(SynthSpec(**kw))
    return _trace_cache[key]


def engine_resolved(e) -> I.ResolvedEngine:
    """The prebuilt engine of one scenario engine dict (make_golden.make_engine)."""
    return I.ResolvedEngine(
        policy=make_policy(e["policy"], alpha=e["alpha"], c=e["c"], max_output=e["max_output"]),
        pool_blocks=e["pool_blocks"], block_size=e["block_size"], cost=CostParams(*e["cost"]),
        limits=EngineLimits(e["cap"], e["max_running"], e["max_context"]),
    )


def scenario_settings(sc) -> tuple[ClusterSettings, I.ResolvedEngine]:
    e, c = sc["engine"], sc["cluster"]
    es = EngineSettings(policy=e["policy"], alpha=e["alpha"], c=e["c"], max_output=e["max_output"],
                        pool_blocks=e["pool_blocks"], block_size=e["block_size"],
                        max_tokens_per_batch=c.get("route_cap", e["cap"]),
                        max_running=e["max_running"],
                        cost=dict(zip(["mem_base_s", "mem_per_kv_token_s", "compute_per_token_s", "overhead_s"],
                                      e["cost"])))
    re = I.ResolvedEngine(
        policy=make_policy(e["policy"], alpha=e["alpha"], c=e["c"], max_output=e["max_output"]),
        pool_blocks=e["pool_blocks"], block_size=e["block_size"], cost=CostParams(*e["cost"]),
        limits=EngineLimits(e["cap"], e["max_running"], e["max_context"]),
    )
    cs = ClusterSettings(n_servers=c["n_servers"], engine=es,
                         balancer=BalancerSettings(name=c["balancer"], poll_interval_s=c["poll_interval_s"],
                                                   beta_prior=c["beta_prior"], beta_fixed=c["beta_fixed"]),
                         seed=c["seed"])
    return cs, re


def scenario_batch(scs) -> I.Batch:
    traces, recs, toffs = [], [], {}
    servers = {}  # heterogeneous prebuilt engines: one parameter set per server
    n_trace = n_rec = 0
    for k, sc in enumerate(scs):
        if "engines" in sc:
            servers[k] = np.array([I.engine_params_record(engine_resolved(x)) for x in sc["engines"]],
                                  dtype=I._abi.ENGINE_PARAMS)
        t = scenario_trace(sc)
        key = id(t)
        if key not in toffs:
            toffs[key] = n_trace
            traces.append(t)
            n_trace += len(t)
        cs, re = scenario_settings(sc)
        recs.append(I.instance_record(cs, len(t), trace_offset=toffs[key], record_offset=n_rec,
                                      qps_factor=sc["qps_factor"], resolved=re))
        n_rec += len(t)
    tr = Trace(np.concatenate([t.arrival for t in traces]), np.concatenate([t.prompt for t in traces]),
               np.concatenate([t.output for t in traces]))
    return I.Batch(tr, np.array(recs, dtype=I._abi.INSTANCE), n_rec, [sc["name"] for sc in scs], servers)


PER_ENGINE_FIELDS = ("iterations", "request_steps", "batch_tokens", "peak_batch_tokens")


def compare_instance(sc, golden, batch, i, rec, stats, *, check_summary=None, engines=None) -> list[str]:
    """Return a list of mismatch descriptions (empty = bit-exact parity). engines: the
    instance's ENGINE_STATS rows, compared with the reference's per-engine counters."""
    g = golden[sc["name"]]
    bad = []
    st = stats[i]
    if "error" in g:
        if int(st["status"]) == 0:
            bad.append(f"reference raised {g['error']} but status 0")
        return bad
    if int(st["status"]) != 0:
        return [f"status {int(st['status'])}"]
    inst = batch.instances[i]
    n, o, to = int(inst["n_requests"]), int(inst["record_offset"]), int(inst["trace_offset"])
    arr = batch.trace.arrival[to:to + n] / float(inst["qps_factor"])
    if "trace_sha" in g and trace_sha(arr, batch.trace.prompt[to:to + n],
                                       batch.trace.output[to:to + n]) != g["trace_sha"]:
        bad.append("trace differs from the reference's")
    for k in ("iterations", "request_steps", "batch_tokens", "dispatches", "preempts", "parks", "finished",
              "peak_batch_tokens"):
        if int(st[k]) != int(g[k]):
            bad.append(f"{k}: got {int(st[k])} want {g[k]}")
    if "%016x" % int(st["digest"]) != g["digest"]:
        bad.append("event digest differs")
    if engines is not None and "per_engine" in g:
        got = [[int(r[k]) for k in PER_ENGINE_FIELDS] for r in engines]
        if got != g["per_engine"]:
            bad.append(f"per-engine counters differ: got {got[:3]} want {g['per_engine'][:3]}")
    sha = records_sha(rec.first_token[o:o + n], rec.finish[o:o + n], rec.preempt_count[o:o + n],
                      rec.server[o:o + n])
    if sha != g["records_sha"]:
        bad.append("records differ")
        if "records" in g:
            want = np.array(g["records"], dtype=np.float64).reshape(-1, 4)
            got = np.stack([rec.first_token[o:o + n], rec.finish[o:o + n], rec.preempt_count[o:o + n],
                            rec.server[o:o + n]], axis=1)
            diff = np.flatnonzero(np.any(want != got, axis=1))
            bad.append(f"first differing request {diff[:5].tolist()}: got {got[diff[:1]].tolist()} "
                       f"want {want[diff[:1]].tolist()}")
    if check_summary is not None and g.get("summary"):
        for k, v in g["summary"].items():
            gv = check_summary[k]
            if isinstance(v, float) and math.isinf(v):
                ok = math.isinf(gv)
            else:
                ok = gv == v
            if not ok:
                bad.append(f"summary {k}: got {gv!r} want {v!r}")
    return bad


__all__ = ["load_golden", "scenario_batch", "scenario_trace", "compare_instance", "fold_digests"]


def pooled_host_values(batch, rec):
    """Per-record metric arrays of every instance of `batch` concatenated (numpy,
    the reference's operation order), plus the preempt counts — the pooled set."""
    from paper_2410_17840_b200.pooled import metric_values

    cols = {k: [] for k in ("arrival", "prompt", "output", "first_token", "finish", "first_dispatch", "pc")}
    for inst in batch.instances:
        o, t, n, f = int(inst["record_offset"]), int(inst["trace_offset"]), int(inst["n_requests"]), float(inst["qps_factor"])
        cols["arrival"].append(batch.trace.arrival[t:t + n] / f)
        cols["prompt"].append(batch.trace.prompt[t:t + n])
        cols["output"].append(batch.trace.output[t:t + n])
        cols["first_token"].append(rec.first_token[o:o + n])
        cols["finish"].append(rec.finish[o:o + n])
        cols["first_dispatch"].append(rec.first_dispatch[o:o + n])
        cols["pc"].append(rec.preempt_count[o:o + n])
    c = {k: np.concatenate(v) for k, v in cols.items()}
    vals = metric_values(c["arrival"], c["prompt"], c["output"], c["first_token"], c["finish"], c["first_dispatch"])
    return vals, c["pc"]


def pooled_expected(vals, pc):
    """sorted(union)[ceil(p/100*n)-1] per slot (metrics.py:46-54) + counts."""
    import math

    from paper_2410_17840_b200.pooled import SLOTS

    out = {}
    for metric, p in SLOTS:
        v = np.sort(vals[metric], kind="stable")
        out[f"{metric}_p{p}"] = float(v[math.ceil(p / 100 * len(v)) - 1]) if len(v) else float("nan")
    n = len(vals["ttft"])
    out.update(n_requests=n, n_tpot=len(vals["tpot"]), n_preempted=int((pc > 0).sum()),
               preemption_rate=int((pc > 0).sum()) / n)
    return out
