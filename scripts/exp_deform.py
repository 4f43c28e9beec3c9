"""Deformable sequence on the rings: every frame A's
vertices are displaced on the GPU (a travelling wave, torch ops), handed over
in place with TriangleMesh.deformed, then refit + min query.  Device ms per
frame, split into restage+refit and query.  python scripts/exp_deform.py [frames]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
tz, tb = md.ring_pair_base(2500, 1500)
xa, xb = md.ring_frame_transforms(0)
A, B = md.build_f12(tz), md.build_f12(tb)
b = md.apply_transform(tb, xb)
md.refit(B, b)
V0 = torch.tensor(tz.vertices, device="cuda")
cfg = md.EngineConfig(front_hard_cap=1 << 27)
rows = []
for f in range(n + 2):
    E = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    E[3].record()
    V = V0 + 0.002 * torch.sin(V0 * 7.0 + 0.3 * f)          # the simulation's new positions (device)
    torch.cuda.synchronize()
    E[0].record()
    a = md.apply_transform(tz.deformed(V), xa)
    md.refit(A, a)                                          # restage (f64 -> f32, leaf sets) + refit
    E[1].record()
    r = md.run_min_query(a, b, A, B, cfg)
    E[2].record()
    torch.cuda.synchronize()
    if f >= 2:
        rows.append((E[0].elapsed_time(E[1]), E[1].elapsed_time(E[2]), E[3].elapsed_time(E[0])))
print(json.dumps({"frames": n, "tris": tz.n_triangles, "deform_restage_refit_ms": round(sum(x[0] for x in rows) / n, 4),
                  "query_ms_incl_host": round(sum(x[1] for x in rows) / n, 4),
                  "wave_generation_ms (torch, not ours)": round(sum(x[2] for x in rows) / n, 4),
                  "last_distance": r.distance}))
