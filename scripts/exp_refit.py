"""Device time of refit alone (rings 2500 x 1500): N back-to-back refits of
A between two CUDA events (host runs ahead, so this is device time), plus
the per-call host cost of the public refit()."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import _lib  # noqa: E402

nu = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
tz, tb = md.ring_pair_base(nu, nv)
A = md.build_f12(tz)
meshes = [md.apply_transform(tz, md.ring_frame_transforms(f)[0]) for f in range(8)]
for m in meshes:
    md.refit(A, m)
torch.cuda.synchronize()
L = _lib.lib()
views = [(m.device_view(), A.device_view()) for m in meshes]
s = _lib.stream_ptr()
N = 64
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    torch.cuda.synchronize()
    e0.record()
    for i in range(N):
        g, v = views[i % 8]
        L.gd_refit(C.byref(g), C.byref(v), s)
    e1.record()
    torch.cuda.synchronize()
    print(f"device refit (raw ctypes, back to back): {e0.elapsed_time(e1) / N * 1e3:.1f} us")
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(N):
    md.refit(A, meshes[i % 8])
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"public refit(): host {((t1 - t0) / N) * 1e6:.1f} us/call, wall incl. drain {((t2 - t0) / N) * 1e6:.1f} us/call")
