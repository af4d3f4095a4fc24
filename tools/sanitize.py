"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): every policy on
single engines, a 4-replica SAL cluster (one CTA) and a 16-replica SAL cluster (a 2-CTA
thread-block cluster, DSMEM), a 24-replica trail_plus cluster and a 6-engine cluster of differing
prebuilt engines (pipelined kernel), with the event ring on; compared with the oracle.
usage: compute-sanitizer --tool memcheck python tools/sanitize.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from oracle import oracle as O
import paper_2410_17840_b200 as P
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate

tr = P.synthesize(P.SynthSpec(duration_s=6.0, mean_qps=20.0, burstiness=2.0, seed=3))
jobs = [(P.ClusterSettings(1, P.EngineSettings(policy=p, c=0.5, pool_blocks=1000, max_output=2048, block_size=bs), P.BalancerSettings("rr"), 0),
         tr, 1.0) for p in ("fcfs", "nopreempt", "trail_plus", "larry") for bs in (16, 10)]
jobs += [(P.ClusterSettings(n, P.EngineSettings(policy="larry", pool_blocks=1000), P.BalancerSettings(b, poll_interval_s=0.05), 1),
          tr, 1.0) for n in (4, 16) for b in ("sal", "p2c")]
jobs += [(P.ClusterSettings(24, P.EngineSettings(policy="trail_plus", c=0.5, pool_blocks=1000), P.BalancerSettings("sal", poll_interval_s=0.05), 2),
          tr, 1.0)]
batch = I.make_batch(jobs)
# a cluster of prebuilt engines that differ (pool, block size, cap, costs): per-server parameters
srv = np.zeros(6, dtype=I._abi.ENGINE_PARAMS)
srv[:] = batch.instances[len(jobs) - 1]["engine"]
srv["pool_blocks"] = [1000, 1400, 1100, 2000, 1000, 1200]
srv["block_size"] = [16, 16, 8, 16, 32, 16]
srv["max_tokens_per_batch"] = [1024, 512, 1024, 2048, 256, 1024]
hb = I.make_batch([(P.ClusterSettings(6, P.EngineSettings(policy="trail_plus", c=0.5, pool_blocks=1000), P.BalancerSettings("sal", poll_interval_s=0.05), 4), tr, 1.0)])
batch = I.Batch(P.Trace(np.concatenate([batch.trace.arrival, hb.trace.arrival]),
                        np.concatenate([batch.trace.prompt, hb.trace.prompt]),
                        np.concatenate([batch.trace.output, hb.trace.output])),
                np.concatenate([batch.instances, hb.instances]), batch.n_records + hb.n_records, [], {len(jobs): srv})
batch.instances[-1]["trace_offset"] = len(batch.trace.arrival) - len(hb.trace.arrival)
batch.instances[-1]["record_offset"] = batch.n_records - hb.n_records
rec, st, ev = simulate.run_batch(batch, events=True)
orec, ost = O.run_batch(batch)
assert np.array_equal(st["digest"], ost["digest"]) and (st["status"] == 0).all()
print("sanitize workload ok:", len(jobs), "instances,", int(st["request_steps"].sum()), "request-steps")
