"""Count SASS instructions per source line / enclosing function of a kernel in libssb.so."""
import collections, os, re, subprocess, sys, tempfile
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2410_17840_b200/libssb.so"
kname = sys.argv[2] if len(sys.argv) > 2 else "k_engines"
import fnmatch
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "summary" not in f][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
sec = None; line = None; cnt = collections.Counter(); total = 0
for ln in dis.splitlines():
    m = re.match(r'\s*\.section\s+\.text\.(\S+),', ln)
    if m: sec = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m: line = (os.path.basename(m.group(1)), int(m.group(2))); continue
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', ln) and sec and kname in sec:
        cnt[line] += 1; total += 1
# map lines to enclosing function (crude: nearest preceding '__device__' def line)
src = {}
for f in ("ssb_engine.cuh", "ssb_kernels.cu"):
    p = "paper_2410_17840_b200/csrc/" + f
    if os.path.exists(p): src[f] = open(p).read().splitlines()
def func_of(f, n):
    L = src.get(f)
    if not L: return f
    for i in range(n - 1, -1, -1):
        m = re.search(r'(?:__device__|__global__)[^(]*?\b(\w+)\s*\(', L[i])
        if m: return f"{f}:{m.group(1)}"
    return f
fc = collections.Counter()
for k, c in cnt.items():
    fc[func_of(*k) if k else "?"] += c
print("total", total)
for k, c in fc.most_common(30): print(f"{c:6d} {k}")
