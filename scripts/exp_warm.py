"""Temporal warm start on the rings sequence: per-frame query time and work,
cold vs seeded with the previous frame's witness (PreparedQuery.seed_from),
and run_sequence wall time both ways.  python scripts/exp_warm.py [frames]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import query as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nu, nv = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (2500, 1500)
tz, tb = md.ring_pair_base(nu, nv)
A, B = md.build_f12(tz), md.build_f12(tb)
cfg = md.EngineConfig(front_hard_cap=1 << 27)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def frame(f):
    xa, xb = md.ring_frame_transforms(f)
    return md.apply_transform(tz, xa), md.apply_transform(tb, xb)


a, b = frame(0)
plans = [Q.PreparedQuery(a, b, A, B, cfg, "min", private_workspace=True) for _ in range(2)]
cold = Q.PreparedQuery(a, b, A, B, cfg, "min", private_workspace=True)
plans[1].bind(a, b).run()
rows = []
for f in range(1, n + 1):
    a, b = frame(f)
    md.refit(A, a)
    md.refit(B, b)
    rc = cold.bind(a, b).run()
    torch.cuda.synchronize()
    ev[0].record()
    cold.launch()
    ev[1].record()
    torch.cuda.synchronize()
    ms_cold = ev[0].elapsed_time(ev[1])
    prev, cur = plans[(f - 1) % 2], plans[f % 2]
    cur.bind(a, b).seed_from(prev)
    ev[0].record()
    cur.launch()
    ev[1].record()
    rw = cur.collect()
    ms_warm = ev[0].elapsed_time(ev[1])
    assert rw.distance == rc.distance and rw.witness.tri_a == rc.witness.tri_a, f
    rows.append((ms_cold, ms_warm, rc.expanded_pairs, rw.expanded_pairs, rc.peak_front, rw.peak_front))
r = np.array(rows)
print(json.dumps({"frames": n, "tris": tz.n_triangles, "cold_ms": round(float(r[:, 0].mean()), 4),
                  "warm_ms": round(float(r[:, 1].mean()), 4), "cold_expanded": int(r[:, 2].mean()),
                  "warm_expanded": int(r[:, 3].mean()), "cold_peak": int(r[:, 4].mean()),
                  "warm_peak": int(r[:, 5].mean())}))
xfs = [md.ring_frame_transforms(f) for f in range(4 * n)]
for warm in (False, True, False, True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = md.run_sequence(tz, tb, A, B, xfs, cfg=cfg, warm=warm)
    torch.cuda.synchronize()
    print(json.dumps({"run_sequence_warm": warm, "ms_per_frame": round((time.perf_counter() - t0) * 1e3 / len(xfs), 4),
                      "first": out[0].tolist()}))
