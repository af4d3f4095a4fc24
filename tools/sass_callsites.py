"""Static SASS instructions per outermost engine call site (nvdisasm -gi inline chains):
which source lines of ssb_engine.cuh / ssb_kernels.cu pull in the most inlined code.
usage: python tools/sass_callsites.py [lib] [kernel] [top]"""
import collections, os, re, subprocess, sys, tempfile
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2410_17840_b200/libssb.so"
kname = sys.argv[2] if len(sys.argv) > 2 else "k_engines"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "summary" not in f][0]
dis = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout
sec = None
chain = []
fresh = True
inner = collections.Counter()   # (innermost engine-file line) -> instrs
outer = collections.Counter()   # (outermost engine-file line that is a call into another engine function)
for ln in dis.splitlines():
    m = re.match(r'\s*\.section\s+\.text\.(\S+),', ln)
    if m:
        sec = m.group(1); continue
    if ln.strip().startswith("//## File"):
        locs = [(os.path.basename(f), int(n)) for f, n in re.findall(r'"([^"]+)", line (\d+)', ln)]
        if fresh:
            chain, fresh = [], False
        for c in locs:
            if c not in chain:
                chain.append(c)
        continue
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', ln):
        fresh = True
    if re.match(r'\s*/\*[0-9a-f]{4,}\*/', ln) and sec and kname in sec and chain:
        own = [c for c in chain if c[0] in ("ssb_engine.cuh", "ssb_kernels.cu")]
        if own:
            inner[own[0]] += 1
            # call sites: every engine-file location in the chain except the innermost
            for c in own[1:]:
                outer[c] += 1
srcs = {f: open(p).read().splitlines() for f, p in [("ssb_engine.cuh", "paper_2410_17840_b200/csrc/ssb_engine.cuh"),
                                                     ("ssb_kernels.cu", "paper_2410_17840_b200/csrc/ssb_kernels.cu")]}
print(f"-- call sites by inlined instructions (top {top})")
for (f, n), c in outer.most_common(top):
    print(f"{c:6d}  {f}:{n}  {srcs[f][n - 1].strip()[:100]}")
