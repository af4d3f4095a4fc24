"""Sync timeline of k_cluster_pipe (timeline build: tools/build_variant.sh timeline -DSSB_PIPE_TIMELINE;
run with SSB_LIB=tools/variants/libssb_timeline.so): per sync of the first instance, how long the
router waited, each engine's wake latency after the publish, its work and iterations in that
wake, and which engine finished last. usage: python tools/probe_sync.py [c5|c2] [duration_s]"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_17840_b200 import _abi, configs as C, instances as I, simulate  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
dur = float(sys.argv[2]) if len(sys.argv) > 2 else 600.0
job = (C.c5_jobs(dur)[0] if which == "c5" else C.c2_jobs()[2])
lib = _abi.load_library()
lib.ssb_debug_sync_timeline.restype = ctypes.c_int32
lib.ssb_debug_sync_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
db = simulate.upload(I.make_batch([job]))
simulate.launch(db)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); simulate.launch(db); e1.record(); torch.cuda.synchronize()
n = int(db.h_inst[0]["n_servers"])
W = 2 + 3 * 128
S = 4096
tl = np.zeros(S * W, dtype=np.uint64)
got = lib.ssb_debug_sync_timeline(tl.ctypes.data, S)
tl = tl.reshape(S, W).astype(np.int64)
valid = tl[:, 0] > 0
tl = tl[valid]
pub, done = tl[:, 0], tl[:, 1]
eng = tl[:, 2:2 + 3 * n].reshape(len(tl), n, 3)
wake, edone, its = eng[:, :, 0] - pub[:, None], eng[:, :, 1] - pub[:, None], eng[:, :, 2]
wait = done - pub
gap = np.diff(pub)
print(f"{job[3]}: kernel {e0.elapsed_time(e1):.1f} ms, syncs recorded {len(tl)}")
pc = lambda a: " / ".join(f"{v:8.0f}" for v in np.percentile(a, [10, 50, 90, 99]))  # noqa: E731
print("ns p10/p50/p90/p99")
print("router wait (publish -> all done)  ", pc(wait))
print("sync-to-sync                        ", pc(gap))
print("routing between syncs (gap - wait)  ", pc(gap - wait[:-1]))
print("engine wake latency (all engines)   ", pc(wake.ravel()))
print("engine done after publish (max/sync)", pc(edone.max(1)))
print("last engine's wake latency          ", pc(wake[np.arange(len(tl)), edone.argmax(1)]))
print("last engine's work (done - wake)    ", pc((edone - wake)[np.arange(len(tl)), edone.argmax(1)]))
print("last engine's iterations in the wake", pc(its[np.arange(len(tl)), edone.argmax(1)]))
print("iterations in the sync wake (all)   ", pc(its.ravel()))
print("router all-done seen after last done", pc(wait - edone.max(1)))
print("last engine histogram:", np.bincount(edone.argmax(1), minlength=n))
