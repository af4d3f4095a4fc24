"""Instruction-cache footprint of a kernel from an ncu report: distinct executed SASS
instructions (and their 128 B lines) per enclosing CUDA function, weighted by execution.
usage: python tools/ncu_footprint.py report.ncu-rep kernel_substring [lib.so]"""
import collections, csv, io, os, re, subprocess, sys, tempfile
rep, kname = sys.argv[1], sys.argv[2]
lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2410_17840_b200/libssb.so"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kname}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0] if "Source" in rows[0] else rows[1]
st = 1 if h is rows[0] else 2
ia, iex = h.index("Address"), h.index("Instructions Executed")
recs = []
for r in rows[st:]:
    try:
        recs.append((int(r[ia], 16), int(r[iex] or 0)))
    except Exception:
        pass
base = recs[0][0]
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
    if m and sec and kname in sec:
        off2line[int(m.group(1), 16)] = line
srcs = {}
def func_of(key):
    if not key:
        return "?"
    f, n = key
    pth = next((q for q in ["paper_2410_17840_b200/csrc/" + f, "include/" + f] if os.path.exists(q)), None)
    if not pth:
        return f
    L = srcs.setdefault(pth, open(pth).read().splitlines())
    for i in range(n - 1, -1, -1):
        m = re.search(r'(?:__device__|__global__)[^(]*?\b(\w+)\s*\(', L[i])
        if m:
            return f"{f}:{m.group(1)}"
    return f
S = sum(x for _, x in recs)
fp, ex = collections.Counter(), collections.Counter()
for a, x in recs:
    if x > 0:
        fn = func_of(off2line.get(a - base))
        fp[fn] += 1
        ex[fn] += x
print(f"executed instructions: {sum(fp.values())} distinct ({sum(fp.values()) * 16 / 1024:.0f} KB), {S} total")
for fn, c in fp.most_common(40):
    print(f"{c:6d} instrs {c * 16 / 1024:5.1f} KB   exec share {100 * ex[fn] / S:5.1f}%   {fn}")
