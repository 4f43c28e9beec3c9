"""Front engine vs the per-triangle DFS comparator (query.py:622-708) on the
interlocked rings at several sizes: device time per query and node counts.
usage: python scripts/exp_dfs.py [nu nv ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2411_11244_b200 as md


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record()
        r = fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best, r


sizes = [int(x) for x in sys.argv[1:]] or [100, 50, 500, 250, 2500, 1500]
for nu, nv in zip(sizes[::2], sizes[1::2]):
    tz, tb = md.ring_pair_base(nu, nv)
    xa, xb = md.ring_frame_transforms(137)
    a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
    ta, tbv = md.build_f12(a), md.build_f12(b)
    for q in ("min", "max"):
        run = md.run_min_query if q == "min" else md.run_max_query
        ms_f, rf = timed(lambda: run(a, b, ta, tbv))
        ms_d, rd = timed(lambda: md.run_dfs_baseline(a, b, tbv, q), reps=3)
        print(json.dumps({"tris": a.n_triangles, "kind": q, "front_ms": round(ms_f, 4), "dfs_ms": round(ms_d, 4),
                          "equal": rf.distance == rd.distance and rf.witness.tri_a == rd.witness.tri_a
                          and rf.witness.tri_b == rd.witness.tri_b,
                          "front_expanded": rf.expanded_pairs, "dfs_visited": rd.visited_nodes,
                          "front_narrow": rf.narrow_pairs, "dfs_narrow": rd.narrow_pairs}), flush=True)
