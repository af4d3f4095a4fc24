"""bench.py's N>1 path on CPU: `python bench.py --gpus 2 --dry-cpu` self-launches two
ranks under torch.distributed.run (gloo), shards the sweep (weak: seeds per rank;
strong: the one sweep split by estimated cost), runs the barrier / max-over-ranks /
all-gather plumbing with the oracle standing in for the kernels, and rank 0 alone
prints one JSON line. The request-step total must equal a single-process oracle run
of the same instances."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _bench(*extra):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-cpu", "--steps", "1",
                          *extra], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    return json.loads(lines[0])


def _oracle_rsteps(jobs):
    from oracle import oracle as O
    from paper_2410_17840_b200 import instances as I

    _, st = O.run_batch(I.make_batch(jobs), threads=2)
    assert (st["status"] == 0).all()
    return int(st["request_steps"].sum())


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_rank_dry_cpu(scaling):
    import bench
    from paper_2410_17840_b200 import configs as C

    line = _bench("--scaling", scaling)
    assert line["n_gpus"] == 2 and line["scaling"] == scaling and "dry_cpu" in line
    assert line["steps"] == 1 and line["warmup"] >= 3
    for k in ("value", "e2e", "warm_schedule", "roofline", "clocks", "config"):
        assert k in line
    if scaling == "weak":
        jobs = [j for r in range(2) for j in bench.sweep_jobs("weak", r, 2, dry=True)[0]]
        assert line["config"]["total_instances"] == 2 * 4096
    else:
        parts = [bench.sweep_jobs("strong", r, 2, dry=True)[0] for r in range(2)]
        jobs = parts[0] + parts[1]
        whole = C.c4_jobs(duration_s=60.0)[::16]
        assert sorted(j[3] for j in jobs) == sorted(j[3] for j in whole)  # a partition of the sweep
        assert abs(len(parts[0]) - len(parts[1])) <= len(whole) // 4
        assert line["config"]["total_instances"] == 4096
    assert line["request_steps_total_per_step"] == _oracle_rsteps(jobs)
