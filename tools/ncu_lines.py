"""Aggregate ncu SASS-level samples per CUDA source line (nvdisasm -g line info).
usage: python tools/ncu_lines.py report.ncu-rep kernel_substring [lib.so] [top]"""
import csv, io, re, subprocess, sys, tempfile, os, collections
rep, kname = sys.argv[1], sys.argv[2]
lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2410_17840_b200/libssb.so"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kname}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isamp, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ia], 16), int(r[isamp] or 0), int(r[iex] or 0)))
    except Exception:
        pass
base = recs[0][0]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "summary" not in f][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
sec = None
line = None
off2line = {}
for ln in dis.splitlines():
    m = re.match(r'\s*\.section\s+\.text\.(\S+),', ln)
    if m:
        sec = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and sec and kname in sec:
        off2line[int(m.group(1), 16)] = line
agg = collections.Counter(); aggx = collections.Counter()
for a, s, x in recs:
    l = off2line.get(a - base)
    agg[l] += s; aggx[l] += x
tot = sum(agg.values()); totx = sum(aggx.values())
print(f"samples {tot}, warp-instructions {totx}")
src = {}
for (f, n), c in agg.most_common(top):
    pass
# per enclosing function (nearest preceding __device__/__global__ definition)
import re as _re
srcs = {}
def func_of(f, n):
    pth = next((q for q in ["paper_2410_17840_b200/csrc/" + f, "include/" + f] if os.path.exists(q)), None)
    if not pth:
        return f
    L = srcs.setdefault(pth, open(pth).read().splitlines())
    for i in range(n - 1, -1, -1):
        m = _re.search(r'(?:__device__|__global__)[^(]*?\b(\w+)\s*\(', L[i])
        if m:
            return f"{f}:{m.group(1)}"
    return f
fs, fx = collections.Counter(), collections.Counter()
for key in set(agg) | set(aggx):
    fn = func_of(*key) if key else "?"
    fs[fn] += agg[key]; fx[fn] += aggx[key]
print("-- per function: stall samples, executed warp-instructions")
for fn, c in fs.most_common(25):
    print(f"{c:7d} {100*c/tot:5.1f}%  ex {fx[fn]:10d} {100*fx[fn]/max(totx,1):5.1f}%  {fn}")
print("-- per line")
for key, c in agg.most_common(top):
    if key is None:
        print(f"{c:7d} {100*c/tot:5.1f}%  ?"); continue
    f, n = key
    path = next((p for p in ["paper_2410_17840_b200/csrc/" + f, "include/" + f] if os.path.exists(p)), None)
    text = open(path).read().splitlines()[n - 1].strip()[:90] if path else ""
    print(f"{c:7d} {100*c/tot:5.1f}% ex {aggx[key]:9d} {f}:{n}  {text}")
