"""The reference-side binding (paper_2410_17840_b200/servesim_bridge.py) driven through
the REFERENCE's own CLI (servesim.cli.main, cli.py:205-214) in the build container,
with the device call replaced by the CPU oracle (the checker) — so routing and exit
codes are tested without a GPU:

* ``--backend b200`` writes byte-identical records / summary / sweep files to
  ``--backend python`` (the reference's own engine);
* ``cmd_sweep`` becomes one batched device call (every factor x combo at once);
* exit codes 0 / 1 (InfeasibleRequestError from the reference's check_feasible) / 2
  (StallError from a device status, and no CUDA device at all).
Skipped where /root/reference is absent (the GPU box); tests/test_gpu_api.py runs the
same binding on the device."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="needs the reference package (build container only)")

if REF.exists() and str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

from oracle import oracle as O  # noqa: E402
from paper_2410_17840_b200 import _abi  # noqa: E402
from paper_2410_17840_b200 import servesim_bridge as B  # noqa: E402

CFG = {
    "seed": 3,
    "workload": {"synth": {"duration_s": 12.0, "mean_qps": 30.0, "burstiness": 2.5,
                           "prompt_dist": {"location": 6.45, "scale": 1.1},
                           "output_dist": {"location": 4.95, "scale": 0.9}}},
    "cluster": {"n_servers": 4, "engine": {"pool_blocks": 900, "c": 0.5},
                "balancer": {"poll_interval_s": 0.05}},
    "policies": ["fcfs", "larry", "trail_plus"],
    "balancers": ["rr", "p2c", "sal"],
    "sweep_factors": [0.5, 1.0, 2.0],
}


class OracleDevice:
    """Stands in for servesim_bridge._Device: same interface, results from the CPU oracle."""

    calls = []
    force_status = 0

    def __init__(self, inst, arr, prm, out, *, events=0, servers=None):
        from paper_2410_17840_b200.instances import Batch
        from paper_2410_17840_b200.workload import Trace

        OracleDevice.calls.append(len(inst))
        self.inst = np.ascontiguousarray(inst)
        self.batch = Batch(Trace(arr, prm, out), self.inst, int((inst["record_offset"] + inst["n_requests"]).max()),
                           servers={} if servers is None else {0: servers})

    def run(self):
        self.rec, st = O.run_batch(self.batch)
        if self.force_status:
            st["status"][:] = self.force_status
        est = np.zeros(int(self.inst["n_servers"].sum()), dtype=_abi.ENGINE_STATS)
        return st, est

    def records(self):
        return self.rec.first_token, self.rec.finish, self.rec.preempt_count, self.rec.server

    def summaries(self):
        out = np.zeros(len(self.inst), dtype=_abi.SUMMARY)
        tr = self.batch.trace
        for i, row in enumerate(self.inst):
            o, t, n, f = (int(row["record_offset"]), int(row["trace_offset"]), int(row["n_requests"]),
                          float(row["qps_factor"]))
            s = O.summarize(tr.arrival[t:t + n] / f, tr.prompt[t:t + n], tr.output[t:t + n],
                            self.rec.first_token[o:o + n], self.rec.finish[o:o + n], self.rec.preempt_count[o:o + n])
            for k in ("n_requests", "ttft_p50", "ttft_p95", "ttft_p99", "norm_ttft_p50", "norm_ttft_p95",
                      "gen_time_p50", "gen_time_p95", "preemption_rate", "throughput_rps"):
                out[i][k] = s[k]
        return out


@pytest.fixture
def cfg(tmp_path):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(CFG))
    return p


@pytest.fixture
def oracle_device(monkeypatch):
    OracleDevice.calls = []
    OracleDevice.force_status = 0
    monkeypatch.setattr(B, "_Device", OracleDevice)
    return OracleDevice


@pytest.mark.parametrize("cmd", ["run", "sweep"])
def test_b200_backend_writes_the_python_backends_bytes(cmd, cfg, tmp_path, oracle_device, capsys):
    py, dev = tmp_path / "py", tmp_path / "b200"
    assert B.cli_main([cmd, "--config", str(cfg), "--out-dir", str(py)]) == 0
    assert oracle_device.calls == []  # the python backend never touches the binding
    assert B.cli_main([cmd, "--backend", "b200", "--config", str(cfg), "--out-dir", str(dev)]) == 0
    combos = len(CFG["policies"]) * len(CFG["balancers"])
    if cmd == "run":
        assert oracle_device.calls == [1] * combos  # cmd_run: one run_cluster per combination
    else:
        assert oracle_device.calls == [combos * len(CFG["sweep_factors"])]  # cmd_sweep: ONE batched launch
    names = sorted(p.name for p in py.iterdir())
    assert names == sorted(p.name for p in dev.iterdir()) and names
    for name in names:
        assert (py / name).read_bytes() == (dev / name).read_bytes(), name
    from servesim import cli

    assert cli._COMMANDS["sweep"] is cli.cmd_sweep  # the patch is undone after the call


def test_exit_code_1_on_infeasible_request(cfg, tmp_path, oracle_device):
    rc = B.cli_main(["run", "--backend", "b200", "--config", str(cfg), "--out-dir", str(tmp_path / "o"),
                     "--set", "cluster.engine.pool_blocks=4"])
    assert rc == 1 and oracle_device.calls == []  # InfeasibleRequestError before any device call


def test_exit_code_2_on_device_stall(cfg, tmp_path, oracle_device, capsys):
    oracle_device.force_status = _abi.SSB_E_STALL
    rc = B.cli_main(["run", "--backend", "b200", "--config", str(cfg), "--out-dir", str(tmp_path / "o")])
    assert rc == 2
    assert "StallError" in capsys.readouterr().err


def test_exit_code_2_without_a_cuda_device(cfg, tmp_path, capsys):
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    rc = B.cli_main(["sweep", "--backend", "b200", "--config", str(cfg), "--out-dir", str(tmp_path / "o")])
    assert rc == 2 and "CUDA" in capsys.readouterr().err


def test_heterogeneous_prebuilt_engines_route_per_server(oracle_device):
    """run_cluster(settings, trace, engines=[...]) with the reference's own engines that differ
    in pool, cap, running limit and cost (cluster.py:66-79): the binding hands one parameter set
    per server to the device (here the oracle) and the records equal the reference's run, mixed
    policies included."""
    from servesim.cluster import build_engine, run_cluster
    from servesim.config import ClusterSettings, EngineSettings
    from servesim.workload import SynthSpec, synthesize

    trace = synthesize(SynthSpec(duration_s=10.0, mean_qps=40.0, burstiness=2.0, seed=5))
    for bal, pol in (("sal", "larry"), ("p2c", "trail_plus"), ("rr", "fcfs")):
        settings = ClusterSettings(n_servers=3, engine=EngineSettings(policy=pol, pool_blocks=900, c=0.5))
        settings.balancer.name = bal
        variants = [dict(pool_blocks=900), dict(pool_blocks=600, max_tokens_per_batch=256, max_running=12),
                    dict(pool_blocks=2500, cost={"mem_base_s": 2e-2})]
        mk = lambda: [build_engine(EngineSettings(policy=pol, c=0.5, **v)) for v in variants]  # noqa: E731
        want = run_cluster(settings, trace, engines=mk())
        engines = mk()
        got = B.run_cluster(settings, trace, engines=engines)
        assert [(r.first_token_time, r.finish_time, r.preempt_count, r.server) for r in got] == \
               [(r.first_token_time, r.finish_time, r.preempt_count, r.server) for r in want], (bal, pol)
    mk = lambda: [build_engine(EngineSettings(policy=p, pool_blocks=900, c=0.5)) for p in ("fcfs", "larry", "trail_plus")]  # noqa: E731
    want = run_cluster(settings, trace, engines=mk())
    got = B.run_cluster(settings, trace, engines=mk())
    assert [(r.first_token_time, r.finish_time, r.preempt_count, r.server) for r in got] == \
           [(r.first_token_time, r.finish_time, r.preempt_count, r.server) for r in want], "mixed policies"
