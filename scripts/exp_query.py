"""Per-iteration anatomy of one rings query (real-time CUDA events, not ncu):
fronts, bound after each iteration, per-launch expand ms; then the same query
seeded with its own witness (warm_pair) to show how much a tight initial
bound shrinks the fronts.  Usage: python scripts/exp_query.py [nu nv frame kind]"""

import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import _lib  # noqa: E402

nu = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
frame = int(sys.argv[3]) if len(sys.argv) > 3 else 7
kind = sys.argv[4] if len(sys.argv) > 4 else "min"
tz, tb = md.ring_pair_base(nu, nv)
A, B = md.build_f12(tz), md.build_f12(tb)
cfg = md.EngineConfig(front_hard_cap=1 << 27)
xa, xb = md.ring_frame_transforms(frame)
a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
md.refit(A, a)
md.refit(B, b)
L = _lib.lib()


def once(warm=None, reps=5):
    pq = md.PreparedQuery(a, b, A, B, cfg, kind, warm)
    for _ in range(2):
        pq.run()
    L.gd_set_profiling(1)
    best = None
    for _ in range(reps):
        r = pq.run()
        ph = (C.c_float * 256)()
        n = L.gd_query_phase_ms(ph, 256)
        vals = list(ph[:n])
        if best is None or sum(vals[:5]) < sum(best[:5]):
            best = vals
    L.gd_set_profiling(0)
    return r, best


for warm in (None, "self"):
    r0 = once()[0] if warm else None
    r, ph = once(None if warm is None else (r0.witness.tri_a, r0.witness.tri_b))
    out = {"warm": warm, "distance": r.distance, "witness": [r.witness.tri_a, r.witness.tri_b],
           "phases_ms": dict(zip(["init", "expand", "narrow", "exact", "final"], [round(x, 4) for x in ph[:5]])),
           "expanded": r.expanded_pairs, "narrow_pairs": r.narrow_pairs, "band": r.band_pairs,
           "edges_ms": {"prologue": round(ph[5 + 3 * len(r.iterations)], 4),
                        "first_plan": round(ph[6 + 3 * len(r.iterations)], 4),
                        "epilogue": round(ph[7 + 3 * len(r.iterations)], 4)}
           if 7 + 3 * len(r.iterations) < len(ph) else None,
           "iters": [{"k": s.k, "in": s.front_in, "out": s.front_out, "culled": s.culled,
                      "bound": round(s.bound_after, 6), "ms": round(ph[5 + i], 4) if 5 + i < len(ph) else None,
                      "sweep_ms": round(ph[5 + len(r.iterations) + i], 4)
                      if 5 + len(r.iterations) + i < len(ph) else None,
                      "plan_ms": round(ph[5 + 2 * len(r.iterations) + i], 4)
                      if 5 + 2 * len(r.iterations) + i < len(ph) else None}
                     for i, s in enumerate(r.iterations)],
           }
    print(json.dumps(out))
torch.cuda.synchronize()
