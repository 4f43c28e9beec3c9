"""Traversal schedule sweep: the device schedule threshold (k = 2 sweeps,
EngineConfig.device_schedule) and the reference rule's C (front_cap) vs the rings query's phases (CUDA events, best of 5) and its
per-iteration times.  Usage: python scripts/exp_sched.py [nu nv frame kind]"""

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
kinds = sys.argv[4].split(",") if len(sys.argv) > 4 else ["min", "max"]
tz, tb = md.ring_pair_base(nu, nv)
A, B = md.build_f12(tz), md.build_f12(tb)
xa, xb = md.ring_frame_transforms(frame)
a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
md.refit(A, a)
md.refit(B, b)
L = _lib.lib()


def once(cfg, kind, reps=7):
    pq = md.PreparedQuery(a, b, A, B, cfg, kind)
    for _ in range(2):
        pq.run()
    L.gd_set_profiling(1)
    best = None
    for _ in range(reps):
        r = pq.run()
        ph = (C.c_float * 64)()
        n = L.gd_query_phase_ms(ph, 64)
        vals = list(ph[:n])
        if best is None or sum(vals[:5]) < sum(best[:5]):
            best = vals
    L.gd_set_profiling(0)
    # plain timing (no phase events between the kernels)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        pq.launch()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    pq.collect()
    return r, best, min(ts), sorted(ts)[len(ts) // 2]


VARIANTS = [(-1, 1 << 18, 5), (-1, 1 << 20, 5), (-1, 1 << 22, 5)] + [
    (sched, 1 << 18, 5) for sched in (1 << 12, 1 << 14, 1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 20, 1 << 22, 1 << 26)]
for kind in kinds:
    for sched, fc, dc in VARIANTS:
        cfg = md.EngineConfig(front_cap=fc, depth_cap=dc, front_hard_cap=1 << 28, device_schedule=sched)
        r, ph, tmin, tmed = once(cfg, kind)
        its = r.iterations
        print(json.dumps({
            "kind": kind, "schedule": sched, "front_cap": fc, "depth_cap": dc, "query_ms_min": round(tmin, 4),
            "query_ms_med": round(tmed, 4), "distance": r.distance,
            "witness": [r.witness.tri_a, r.witness.tri_b],
            "phases_ms": [round(x, 4) for x in ph[:5]], "expanded": r.expanded_pairs,
            "iters": [(s.k, s.front_in, round(ph[5 + i], 4) if 5 + i < len(ph) else None)
                      for i, s in enumerate(its)]}), flush=True)
