"""Stall-reason breakdown of the SASS lines that belong to one device function (by the
nvdisasm line table): python tools/ncu_func_stalls.py report.ncu-rep kernel_regex func_name [lib]"""
import collections, csv, io, os, re, subprocess, sys, tempfile
rep, kname, fname = sys.argv[1], sys.argv[2], sys.argv[3]
lib = sys.argv[4] if len(sys.argv) > 4 else "paper_2410_17840_b200/libssb.so"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kname}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
isrc = hdr.index("Source")
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "summary" not in f][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
sec = line = None
off2line = {}
for ln in dis.splitlines():
    m = re.match(r'\s*\.section\s+\.text\.(\S+),', ln)
    if m:
        sec = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and sec and kname.split(":")[-1] in sec:
        off2line[int(m.group(1), 16)] = line
srcs = {}
def func_of(key):
    if not key: return "?"
    f, n = key
    pth = next((q for q in ["paper_2410_17840_b200/csrc/" + f, "include/" + f] if os.path.exists(q)), None)
    if not pth: return f
    L = srcs.setdefault(pth, open(pth).read().splitlines())
    for i in range(n - 1, -1, -1):
        m = re.search(r'(?:__device__|__global__)[^(]*?\b(\w+)\s*\(', L[i])
        if m: return m.group(1)
    return f
base = None
tot = collections.Counter(); ex = 0; per_line = collections.Counter(); per_line_x = collections.Counter()
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except Exception:
        continue
    if base is None: base = a
    key = off2line.get(a - base)
    if func_of(key) != fname: continue
    x = int(r[iex] or 0); ex += x
    s = 0
    for i in stall_cols:
        v = int(float(r[i] or 0)); tot[hdr[i]] += v; s += v
    per_line[key] += s; per_line_x[key] += x
print(f"{fname}: executed warp-instructions {ex}, samples {sum(tot.values())}")
for k, v in tot.most_common(12): print(f"  {k:24s} {v}")
for key, v in per_line.most_common(25):
    f, n = key
    pth = next((q for q in ["paper_2410_17840_b200/csrc/" + f, "include/" + f] if os.path.exists(q)), None)
    text = open(pth).read().splitlines()[n - 1].strip()[:80] if pth else ""
    print(f"{v:6d} ex {per_line_x[key]:8d} {f}:{n} {text}")
