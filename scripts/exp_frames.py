"""Query time of the rings sequence in the world frame vs B's local frame
(GdConfig.frame), same frames: python scripts/exp_frames.py [frames]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import query as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
tz, tb = md.ring_pair_base(2500, 1500)
A, B = md.build_f12(tz), md.build_f12(tb)
cfg = md.EngineConfig(front_hard_cap=1 << 27)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for frame in ("world", "b-local"):
    ms, peak, exp = [], [], []
    for f in range(0, n * 37, 37):
        xa, xb = md.ring_frame_transforms(f)
        a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
        pq = Q.PreparedQuery(a, b, A, B, cfg, "min", frame=frame)
        r = pq.run()
        torch.cuda.synchronize()
        ev[0].record()
        pq.launch()
        ev[1].record()
        torch.cuda.synchronize()
        ms.append(ev[0].elapsed_time(ev[1]))
        peak.append(r.peak_front)
        exp.append(r.expanded_pairs)
    print(frame, "query ms", np.round(ms, 3).tolist(), "mean", round(float(np.mean(ms)), 3),
          "peak front mean", int(np.mean(peak)), "expanded mean", int(np.mean(exp)))
