"""Per-frame device time of the rings min query (CUDA events around each
launch, refits outside the region) over the bench's frames:
python scripts/exp_frames_query.py [f0 f1 [kind]]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402

f0, f1 = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (3, 23)
kind = sys.argv[3] if len(sys.argv) > 3 else "min"
tz, tb = md.ring_pair_base(2500, 1500)
A, B = md.build_f12(tz), md.build_f12(tb)
cfg = md.EngineConfig(front_hard_cap=1 << 27)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ms = []
for f in range(f0, f1):
    xa, xb = md.ring_frame_transforms(f)
    a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
    md.refit(A, a)
    md.refit(B, b)
    pq = md.PreparedQuery(a, b, A, B, cfg, kind)
    pq.run()
    torch.cuda.synchronize()
    t = []
    for _ in range(5):
        ev[0].record()
        pq.launch()
        ev[1].record()
        torch.cuda.synchronize()
        t.append(ev[0].elapsed_time(ev[1]))
    ms.append(float(np.median(t)))
print(kind, "per-frame query ms", np.round(ms, 4).tolist())
print(kind, "mean", round(float(np.mean(ms)), 4), "min", round(float(np.min(ms)), 4))
