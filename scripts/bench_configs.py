"""All BASELINE.json configs on one B200 (device time via CUDA events,
after a warm-up query), one JSON line per measurement:

  1  tori 2 x 10K, min + max (+ the unmodified reference on the host)
  2  rings 2 x 7.5M, min single frame
  3  rings 2 x 7.5M, min + max over a rotation sequence (frames/s)
  4  nested shells 2 x 2M (lat 1001 x lon 1000, r 0.8 / 0.81), min + max
  5  rings size sweep 100K -> 30M total triangles, min + max

usage: python scripts/bench_configs.py [configs ...] [--frames N] [--out file]
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import query as Q  # noqa: E402

CFG = md.EngineConfig(front_hard_cap=1 << 28)
OUT = None


def emit(rec):
    line = json.dumps(rec)
    print(line, flush=True)
    if OUT:
        with open(OUT, "a") as fh:
            fh.write(line + "\n")


def timed_query(a, b, ta, tb, kind, cfg=CFG, reps=5):
    """Median device time of the query: CUDA events around the launch; a
    query whose front outgrew the arena (several rounds, DESIGN.md "Front
    arena") is timed through collect(), which runs the remaining rounds --
    host gaps between rounds included."""
    pq = Q.PreparedQuery(a, b, ta, tb, cfg, kind)
    r = pq.run()  # warm-up (and the answer)
    rounds = int(pq.res.rounds)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        torch.cuda.synchronize()
        s.record()
        pq.launch()
        if rounds > 1:
            pq.collect()
        e.record()
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    if rounds == 1:
        pq.collect()
    t0 = time.perf_counter()
    r2 = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb, cfg)
    e2e = (time.perf_counter() - t0) * 1e3
    assert r2.distance == r.distance
    return r, float(np.median(ms)), e2e


def result_fields(r):
    return {"rounds": _rounds(r), "distance": r.distance, "witness": [r.witness.tri_a, r.witness.tri_b] if r.witness else None,
            "iterations": len(r.iterations), "peak_front": r.peak_front, "expanded_pairs": r.expanded_pairs,
            "narrow_pairs": r.narrow_pairs, "band_pairs": r.band_pairs}


def _rounds(r):
    return getattr(r, "rounds", None)


def build_pair(a, b):
    t0 = time.perf_counter()
    ta, tb = md.build_f12(a), md.build_f12(b)
    torch.cuda.synchronize()
    return ta, tb, time.perf_counter() - t0


def config1():
    a, b = md.gen_scene("interlocked-rings", {"nu": 100, "nv": 50})
    ta, tb, bs = build_pair(a, b)
    for kind in ("min", "max"):
        r, ms, e2e = timed_query(a, b, ta, tb, kind, md.EngineConfig())
        rec = {"config": 1, "scene": "tori 2 x 10K", "kind": kind, "tris_per_mesh": a.n_triangles, "build_s": bs,
               "query_ms": ms, "e2e_ms": e2e, **result_fields(r)}
        ref = _reference()
        if ref is not None:
            A, B = ref.TriangleMesh(a.vertices, a.triangles), ref.TriangleMesh(b.vertices, b.triangles)
            RA, RB = ref.build_f12(A), ref.build_f12(B)
            run = ref.run_min_query if kind == "min" else ref.run_max_query
            t0 = time.perf_counter()
            rr = run(A, B, RA, RB, ref.EngineConfig(threads=os.cpu_count() or 1))
            rec["reference_ms"] = (time.perf_counter() - t0) * 1e3
            rec["reference_threads"] = os.cpu_count()
            rec["reference_distance_equal"] = rr.distance == r.distance
            rec["reference_witness_equal"] = (rr.witness.tri_a, rr.witness.tri_b) == (r.witness.tri_a, r.witness.tri_b)
        emit(rec)


def _reference():
    src = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
    if not (src / "meshdist").exists():
        return None
    sys.path.insert(0, str(src))
    import meshdist

    return meshdist


def config2():
    tz, tb = md.ring_pair_base(2500, 1500)
    A, B, bs = build_pair(tz, tb)
    xa, xb = md.ring_frame_transforms(0)
    a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
    md.refit(A, a)
    md.refit(B, b)
    r, ms, e2e = timed_query(a, b, A, B, "min")
    emit({"config": 2, "scene": "rings 2 x 7.5M, frame 0", "kind": "min", "tris_per_mesh": tz.n_triangles,
          "build_s": bs, "query_ms": ms, "e2e_ms": e2e, **result_fields(r)})


def config3(n_frames):
    tz, tb = md.ring_pair_base(2500, 1500)
    A, B, _ = build_pair(tz, tb)
    xfs = [md.ring_frame_transforms(f) for f in range(n_frames)]
    pm = pM = None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    dmin, dmax = [], []
    for f in range(min(3, n_frames)):  # warm-up
        a, b = md.apply_transform(tz, xfs[f][0]), md.apply_transform(tb, xfs[f][1])
        md.refit(A, a)
        md.refit(B, b)
        md.run_min_query(a, b, A, B, CFG)
        md.run_max_query(a, b, A, B, CFG)
    torch.cuda.synchronize()
    ev[0].record()
    t0 = time.perf_counter()
    for f in range(n_frames):
        a, b = md.apply_transform(tz, xfs[f][0]), md.apply_transform(tb, xfs[f][1])
        md.refit(A, a)
        md.refit(B, b)
        if pm is None:
            pm = Q.PreparedQuery(a, b, A, B, CFG, "min")
            pM = Q.PreparedQuery(a, b, A, B, CFG, "max")
        pm.bind(a, b).launch()
        rmin = pm.collect()
        pM.bind(a, b).launch()
        rmax = pM.collect()
        dmin.append(rmin.distance)
        dmax.append(rmax.distance)
    ev[1].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    # the same frames through the public API run_sequence_minmax (one CUDA
    # graph per frame with the min / max query group, two graphs alternating
    # on two streams), after one call that captures its graphs
    md.run_sequence_minmax(tz, tb, A, B, xfs[:2], ("min", "max"), CFG)
    torch.cuda.synchronize()
    ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev2[0].record()
    t1 = time.perf_counter()
    seq = md.run_sequence_minmax(tz, tb, A, B, xfs, ("min", "max"), CFG)
    ev2[1].record()
    torch.cuda.synchronize()
    wall_seq = time.perf_counter() - t1
    assert [float(x) for x in seq["min"][:, 0]] == dmin and [float(x) for x in seq["max"][:, 0]] == dmax
    emit({"config": 3, "scene": f"rings 2 x 7.5M, {n_frames}-frame rotation sequence (refit A + B + min + max)",
          "frames": n_frames,
          "run_sequence_minmax": {"frames_per_s_wall": n_frames / wall_seq,
                                  "ms_per_frame_device": ev2[0].elapsed_time(ev2[1]) / n_frames},
          "per_query_sync": {"frames_per_s_wall": n_frames / wall,
                             "ms_per_frame_device": ev[0].elapsed_time(ev[1]) / n_frames},
          "answers_equal": True,
          "d_min_range": [min(dmin), max(dmin)], "d_max_range": [min(dmax), max(dmax)], "gpus": 1})


def config4():
    """Nested shells 2 x 2M: the reference needs front_hard_cap raised for
    this scene; here it is unlimited (2^40) and the fronts
    that outgrow the arena are expanded in chunks."""
    a, b = md.gen_scene("nested-shells", {"lat": 1001, "lon": 1000, "r_inner": 0.8, "r_outer": 0.81})
    ta, tb, bs = build_pair(a, b)
    cfg = md.EngineConfig(front_hard_cap=1 << 40)
    for kind in ("min", "max"):
        t0 = time.perf_counter()
        r, ms, e2e = timed_query(a, b, ta, tb, kind, cfg, reps=3)
        emit({"config": 4, "scene": "nested shells 2 x 2M (r 0.8 / 0.81)", "kind": kind,
              "tris_per_mesh": a.n_triangles, "build_s": bs, "query_ms": ms, "e2e_ms": e2e,
              "wall_s_incl_warmup": time.perf_counter() - t0, "arena_entries": Q._auto_arena(),
              "iters": [(s.k, s.front_in, s.front_out) for s in r.iterations], **result_fields(r)})


def config5():
    for nu, nv in [(250, 100), (500, 150), (1000, 250), (1500, 500), (2500, 1000), (5000, 1500)]:
        tz, tb = md.ring_pair_base(nu, nv)
        A, B, bs = build_pair(tz, tb)
        xa, xb = md.ring_frame_transforms(0)
        a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
        md.refit(A, a)
        md.refit(B, b)
        for kind in ("min", "max"):
            r, ms, e2e = timed_query(a, b, A, B, kind)
            emit({"config": 5, "scene": f"rings {nu} x {nv}", "kind": kind, "tris_total": 2 * tz.n_triangles,
                  "build_s": bs, "query_ms": ms, "e2e_ms": e2e, **result_fields(r)})
        del A, B
        torch.cuda.empty_cache()


def main():
    global OUT
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[1, 2, 3, 4, 5])
    ap.add_argument("--frames", type=int, default=1000)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    OUT = args.out
    for c in args.configs:
        {1: config1, 2: config2, 3: lambda: config3(args.frames), 4: config4, 5: config5}[c]()


if __name__ == "__main__":
    main()
