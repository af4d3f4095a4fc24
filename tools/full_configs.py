"""All five BASELINE configs at FULL size: the CUDA path vs the CPU oracle (bit-exact
check of every per-instance counter, the decision digest and every record), with
timings of both. Writes a markdown table (stdout) and a JSON file.

usage: python tools/full_configs.py [c1 c2 c3 c4 c5 | cN:duration_s ...] [--json out.json] [--no-oracle]

The oracle is test infrastructure (oracle/ssb_oracle.c, a serial restatement of the
reference pinned to the reference's own outputs); here it is the checker and the
CPU timing beside the GPU's. Oracle threads = one per instance (capped at the host's
cores); the GPU runs every instance of a config in one ssb_simulate launch."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2410_17840_b200 import configs as C  # noqa: E402
from paper_2410_17840_b200 import instances as I  # noqa: E402
from paper_2410_17840_b200 import simulate  # noqa: E402

KEYS = ("iterations", "request_steps", "batch_tokens", "dispatches", "preempts", "parks", "finished",
        "peak_batch_tokens", "digest", "status")


def gpu_run(batch):
    db = simulate.upload(batch)
    simulate.launch(db)  # first pass: also the device-cycle estimates for the schedule
    torch.cuda.synchronize()
    st0 = simulate.download(db)[1]
    simulate.retry_overflows(db, st0)
    torch.cuda.synchronize()
    st0 = simulate.download(db)[1]
    c = simulate.measured_cost(db.h_inst, st0)
    if c is not None:
        db.h_inst["est_cost"] = c
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    simulate.launch(db)
    e1.record()
    torch.cuda.synchronize()
    rec, st = simulate.download(db)
    return e0.elapsed_time(e1) / 1e3, rec, st


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out_json = None
    if "--json" in sys.argv:
        out_json = sys.argv[sys.argv.index("--json") + 1]
        args = [a for a in args if a != out_json]
    which = args or ["c1", "c2", "c3", "c4", "c5"]
    no_oracle = "--no-oracle" in sys.argv
    O.build()
    cores = os.cpu_count() or 1
    rows = []
    print(f"host cores: {cores}; GPU: {torch.cuda.get_device_name(0)}", flush=True)
    for w in which:
        t0 = time.perf_counter()
        name, _, dur = w.partition(":")  # "c3:83334" = config 3 on its first 83,334 s of trace
        fn = {"c1": C.c1_jobs, "c2": C.c2_jobs, "c3": C.c3_jobs, "c4": C.c4_jobs, "c5": C.c5_jobs}[name]
        jobs = fn(float(dur)) if dur else fn()
        batch = I.make_batch(jobs)
        t_synth = time.perf_counter() - t0
        g_s, grec, gst = gpu_run(batch)
        print(f"{w}: GPU {g_s:.3f} s, {int(gst['request_steps'].sum()):,} request-steps, status "
              f"{np.unique(gst['status']).tolist()}, synth {t_synth:.1f} s", flush=True)
        if no_oracle:
            continue
        threads = min(cores, len(batch.instances))
        t1 = time.perf_counter()
        orec, ost = O.run_batch(batch, threads=threads)
        o_s = time.perf_counter() - t1
        bad = [k for k in KEYS if not np.array_equal(gst[k], ost[k])]
        for col in ("first_token", "finish", "first_dispatch", "preempt_count", "server"):
            a, b = getattr(grec, col), getattr(orec, col)
            same = np.array_equal(a.view(np.int64) if a.dtype == np.float64 else a,
                                  b.view(np.int64) if b.dtype == np.float64 else b)
            if not same:
                bad.append(col)
        rs = int(gst["request_steps"].sum())
        row = {"config": w, "instances": len(batch.instances), "requests": int(batch.n_records),
               "servers": int(batch.instances["n_servers"].max()), "request_steps": rs,
               "iterations": int(gst["iterations"].sum()), "preempts": int(gst["preempts"].sum()),
               "gpu_s": g_s, "gpu_rsteps_per_s": rs / g_s, "oracle_s": o_s, "oracle_threads": threads,
               "oracle_rsteps_per_s": rs / o_s, "bit_exact": not bad, "mismatch": bad, "synth_s": t_synth}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del grec, orec
        torch.cuda.empty_cache()
    print()
    print("| config | instances x servers | requests | request-steps | GPU s | GPU rsteps/s | oracle s (threads) | "
          "oracle rsteps/s | GPU/oracle | bit-exact |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['config'].upper()} | {r['instances']} x {r['servers']} | {r['requests']:,} | {r['request_steps']:,} | "
              f"{r['gpu_s']:.3f} | {r['gpu_rsteps_per_s']:.3e} | {r['oracle_s']:.2f} ({r['oracle_threads']}) | "
              f"{r['oracle_rsteps_per_s']:.3e} | {r['gpu_rsteps_per_s'] / r['oracle_rsteps_per_s']:.1f}x | "
              f"{'yes' if r['bit_exact'] else 'NO: ' + ','.join(r['mismatch'])} |")
    if out_json:
        Path(out_json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
