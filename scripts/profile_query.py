"""One warm-up + N profiled frames of the rings workload (for ncu):
refit A, refit B, query.  Usage: python scripts/profile_query.py [nu nv frames kind]"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402

nu = int(sys.argv[1]) if len(sys.argv) > 1 else 2500
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
frames = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kind = sys.argv[4] if len(sys.argv) > 4 else "min"
tz, tb = md.ring_pair_base(nu, nv)
A, B = md.build_f12(tz), md.build_f12(tb)
cfg = md.EngineConfig(front_hard_cap=1 << 27)
run = md.run_min_query if kind == "min" else md.run_max_query
for f in range(frames + 1):
    xa, xb = md.ring_frame_transforms(f * 7)
    a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
    md.refit(A, a)
    md.refit(B, b)
    torch.cuda.nvtx.range_push(f"frame{f}")
    r = run(a, b, A, B, cfg)
    torch.cuda.nvtx.range_pop()
    print(f, r.distance, r.witness.tri_a, r.witness.tri_b, len(r.iterations), r.expanded_pairs, r.narrow_pairs,
          r.band_pairs, [(s.k, s.front_in, s.front_out) for s in r.iterations])
torch.cuda.synchronize()
