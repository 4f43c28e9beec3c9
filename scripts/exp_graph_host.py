"""Host-side anatomy of run_sequence_minmax (config 3 as one CUDA graph per
frame): wall clock of each part of the per-frame host loop -- apply_transform,
FrameGraph.launch (node-parameter patch + cudaGraphLaunch), results() (wait +
record decode) -- beside the graph's device time.
python scripts/exp_graph_host.py [frames]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
tz, tb = md.ring_pair_base(2500, 1500)
A, B = md.build_f12(tz), md.build_f12(tb)
xfs = [md.ring_frame_transforms(f) for f in range(n + 2)]
cfg = md.EngineConfig(front_hard_cap=1 << 27)
md.run_sequence_minmax(tz, tb, A, B, xfs[:2], ("min", "max"), cfg)  # captures the two graphs
torch.cuda.synchronize()

for rep in range(2):
    t0 = time.perf_counter()
    out = md.run_sequence_minmax(tz, tb, A, B, xfs[2:n + 2], ("min", "max"), cfg)
    print("run_sequence_minmax ms/frame", round((time.perf_counter() - t0) * 1e3 / n, 4))

fg = md.FrameGraph(tz, tb, A, B, ("min", "max"), cfg)
t_xf, t_launch, t_res, t_wait = [], [], [], []
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for f in range(n):
    xa, xb = xfs[f]
    t0 = time.perf_counter()
    a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
    t1 = time.perf_counter()
    fg.launch(a, b)
    t2 = time.perf_counter()
    fg._ready.synchronize()
    t3 = time.perf_counter()
    fg.results()
    t4 = time.perf_counter()
    t_xf.append(t1 - t0)
    t_launch.append(t2 - t1)
    t_wait.append(t3 - t2)
    t_res.append(t4 - t3)
ev[0].record()
for f in range(n):
    xa, xb = xfs[f]
    fg.launch(md.apply_transform(tz, xa), md.apply_transform(tb, xb))
ev[1].record()
torch.cuda.synchronize()
fg.close()
med = lambda x: round(float(np.median(x)) * 1e3, 4)  # noqa: E731
print("per frame ms: apply_transform x2", med(t_xf), "launch", med(t_launch), "wait", med(t_wait),
      "results", med(t_res), "| back-to-back device ms/frame", round(ev[0].elapsed_time(ev[1]) / n, 4))
