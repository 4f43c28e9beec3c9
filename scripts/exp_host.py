"""Host-side cost of one public-API frame (rings): where the e2e time goes."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import query as Q  # noqa: E402

nu = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
tz, tb = md.ring_pair_base(nu, nv)
A, B = md.build_f12(tz), md.build_f12(tb)
cfg = md.EngineConfig(front_hard_cap=1 << 27)
T = {}


def tick(name, t0):
    t = time.perf_counter()
    T.setdefault(name, []).append((t - t0) * 1e6)
    return t


for f in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    xa, xb = md.ring_frame_transforms(f)
    t0 = tick("ring_frame_transforms", t0)
    a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
    t0 = tick("apply_transform x2", t0)
    md.refit(A, a)
    md.refit(B, b)
    t0 = tick("refit x2 (host)", t0)
    pq = Q.PreparedQuery(a, b, A, B, cfg, "min")
    t0 = tick("PreparedQuery()", t0)
    pq.launch()
    t0 = tick("launch", t0)
    torch.cuda.synchronize()
    t0 = tick("device wait", t0)
    r = pq.collect()
    t0 = tick("collect (D2H + result)", t0)
for k, v in T.items():
    v = sorted(v[5:])
    print(f"{k:28s} median {v[len(v) // 2]:8.1f} us")
