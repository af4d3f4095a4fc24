"""C3 at its stated size (BASELINE configs[2]: 1 replica, pool 1,536 blocks, long-tail
outputs, ~1M requests) through the CPU oracle -> tests/golden/c3_full.json.

The oracle (oracle/ssb_oracle.c) is the restatement of the reference that
tests/test_oracle_golden.py pins to 7,500+ fixtures the reference itself produced; at
this size the Python reference would need days, so the oracle is the golden's author. Its
literal trail_plus (a full re-sort of the waiting list and a visit of every candidate per
step) did not finish the 1M-request backlog in 4.5 hours, so trail_plus runs in the oracle's
fast mode (an indexed waiting set with the same decisions, checked against the literal path
by tests/test_oracle_golden.py::test_oracle_fast_trail_plus_equals_literal).
Stored per instance: every ssb_stats counter, the decision digest, and a sha256 of each
record column (f64 bit patterns / i32), plus the trace's sha256 so a changed synthesiser
is caught before a mismatch is blamed on the kernel.

usage: python tools/make_c3_golden.py [duration_s]
"""
import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2410_17840_b200 import configs as C  # noqa: E402
from paper_2410_17840_b200 import instances as I  # noqa: E402

KEYS = ("iterations", "request_steps", "batch_tokens", "dispatches", "preempts", "parks", "finished",
        "peak_batch_tokens", "digest", "status")
COLS = ("first_token", "finish", "first_dispatch", "preempt_count", "server")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def trace_sha(tr) -> str:
    h = hashlib.sha256()
    for a in (tr.arrival, tr.prompt, tr.output):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    dur = float(sys.argv[1]) if len(sys.argv) > 1 else 833_334.0
    out = ROOT / "tests" / "golden" / ("c3_full.json" if len(sys.argv) < 3 else sys.argv[2])
    O.build()
    O.set_trail_fast(True)
    batch = I.make_batch(C.c3_jobs(dur))
    t0 = time.perf_counter()
    rec, st = O.run_batch(batch, mode=1, threads=len(batch.instances))  # Engine.run (one replica each)
    dt = time.perf_counter() - t0
    inst = []
    for i, row in enumerate(batch.instances):
        o, n = int(row["record_offset"]), int(row["n_requests"])
        d = {k: int(st[i][k]) for k in KEYS}
        d["label"] = batch.labels[i]
        d["n_requests"] = n
        d["records_sha256"] = {c: sha(getattr(rec, c)[o:o + n]) for c in COLS}
        inst.append(d)
    doc = {"config": "C3", "duration_s": dur, "trace_sha256": trace_sha(batch.trace),
           "oracle_seconds": dt, "oracle_threads": len(batch.instances), "oracle_trail_plus": "fast mode",
           "instances": inst}
    out.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps({k: v for k, v in doc.items() if k != "instances"}), flush=True)


if __name__ == "__main__":
    main()
