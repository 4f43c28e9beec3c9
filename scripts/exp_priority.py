"""Frame pipelining (refit of frame f+1 on a second stream, overlapping frame
f's narrow / exact phases) with and without a high-priority query stream:
device ms per frame over K frames (CUDA events), rings 2 x 7.5M, min query.
python scripts/exp_priority.py [K]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
tz, tb = md.ring_pair_base(2500, 1500)
A, B = md.build_f12(tz), md.build_f12(tb)
cfg = md.EngineConfig(front_hard_cap=1 << 27)
frames = []
for f in range(K + 3):
    xa, xb = md.ring_frame_transforms(f * 7)
    a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
    frames.append((a, b, md.PreparedQuery(a, b, A, B, cfg, "min", private_workspace=True)))


def run(qprio, rprio):
    qs = torch.cuda.Stream(priority=qprio)
    rs = torch.cuda.Stream(priority=rprio)
    trav = [torch.cuda.Event() for _ in frames]
    refd = [torch.cuda.Event() for _ in frames]
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    for i, (a, b, pq) in enumerate(frames):
        if i == 3:
            s.record(qs)
        with torch.cuda.stream(rs):
            rs.wait_stream(qs) if i == 0 else rs.wait_event(trav[i - 1])
            A._device_refit(a)
            B._device_refit(b)
            refd[i].record(rs)
        qs.wait_event(refd[i])
        with torch.cuda.stream(qs):
            pq.launch(stream=None, traversal_done=trav[i])
    e.record(qs)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (len(frames) - 3)


lo, hi = torch.cuda.Stream.priority_range()
for rep in range(2):
    for name, qp, rp in (("equal", 0, 0), ("query high", hi, 0), ("refit low / query high", hi, lo)):
        print(rep, name, round(run(qp, rp), 4), "ms/frame", flush=True)
