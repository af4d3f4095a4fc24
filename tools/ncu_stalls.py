"""Headline metrics + warp-stall breakdown of one kernel in an ncu report.
usage: python tools/ncu_stalls.py report.ncu-rep [kernel_regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
k = sys.argv[2] if len(sys.argv) > 2 else "k_engines"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{k}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_issued.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:60s} {v[i]} {u[i]}")
st = {}
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
        try:
            st[n[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v[i].replace(",", ""))
        except ValueError:
            pass
tot = sum(st.values()) or 1
print("stall samples:", ", ".join(f"{k} {100 * x / tot:.1f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1]) if x / tot > 0.005))
