"""Second set of golden vectors, made FROM THE REFERENCE ITSELF (the live
package under /root/reference/pkg/src, pure Python + numpy):

* config-4 geometry (nested shells, r 0.8 / 0.81 -- the near-contact stress
  case of BASELINE.json) at the largest sizes the reference builds in
  seconds-to-minutes, min and max, float64 and float32: distance, witness,
  witness points, counters;
* rings (the config 2/3 torus pair) at 50K triangles per mesh, three frames
  of the rotation sequence, min and max;
* tree topology (the greedy power-of-two pairing, bvh.py:98-181) of 60K and
  120K-triangle tori.

    python tests/golden/make_golden_r2.py [/root/reference/pkg/src]

Writes tests/golden/golden_r2.json and golden_r2.npz.  The GPU box has no
/root/reference: tests read only these files.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

from make_golden import load_reference, sha  # noqa: E402


def main(src: str = "/root/reference/pkg/src"):
    md = load_reference(src)
    from meshdist import bvh as rt, query as rq

    from paper_2411_11244_b200 import scenes as ps

    meta: dict = {"reference": src, "generated_by": "tests/golden/make_golden_r2.py"}
    out: dict = {}

    # 1. nested shells (config 4 geometry), min / max, float64 / float32
    meta["shells"] = []
    for lat, lon in ((31, 30), (61, 60), (91, 90), (121, 120)):
        params = {"lat": lat, "lon": lon, "r_inner": 0.8, "r_outer": 0.81}
        a, b = md.gen_scene("nested-shells", params)
        rec = {"params": params, "hash_a": sha(a), "hash_b": sha(b), "tris": int(len(a.triangles))}
        for prec in (64, 32):
            dt = np.float64 if prec == 64 else np.float32
            t0 = time.time()
            ta, tb = rt.build_f12(a, dtype=dt), rt.build_f12(b, dtype=dt)
            rec[f"build{prec}_s"] = time.time() - t0
            cfg = rq.EngineConfig(precision=prec, threads="auto", front_hard_cap=1 << 30)
            for q in ("min", "max"):
                t0 = time.time()
                r = (rq.run_min_query if q == "min" else rq.run_max_query)(a, b, ta, tb, cfg)
                rec[f"{q}{prec}"] = {"distance": r.distance, "tri_a": r.witness.tri_a, "tri_b": r.witness.tri_b,
                                     "point_a": r.witness.point_a.tolist(), "point_b": r.witness.point_b.tolist(),
                                     "witness_exact": r.witness_exact, "iterations": len(r.iterations),
                                     "expanded_pairs": r.expanded_pairs, "narrow_pairs": r.narrow_pairs,
                                     "seconds": time.time() - t0}
                print("shells", lat, lon, prec, q, r.distance, r.witness.tri_a, r.witness.tri_b, flush=True)
        meta["shells"].append(rec)

    # 2. rings 50K triangles per mesh, frames of the rotation sequence
    tz, tbase = ps.ring_pair_base(250, 100)
    meta["rings50k"] = []
    for f in (7, 333, 901):
        xa, xb = ps.ring_frame_transforms(f)
        va = tz.vertices @ xa.rotation.T + xa.translation
        vb = tbase.vertices @ xb.rotation.T + xb.translation
        fa, fb = md.TriangleMesh(va, tz.triangles), md.TriangleMesh(vb, tbase.triangles)
        ta, tb = rt.build_f12(fa), rt.build_f12(fb)
        rec = {"frame": f, "hash_a": sha(fa), "hash_b": sha(fb)}
        for q in ("min", "max"):
            r = (rq.run_min_query if q == "min" else rq.run_max_query)(
                fa, fb, ta, tb, rq.EngineConfig(threads="auto", front_hard_cap=1 << 30))
            rec[q] = {"distance": r.distance, "tri_a": r.witness.tri_a, "tri_b": r.witness.tri_b,
                      "point_a": r.witness.point_a.tolist(), "point_b": r.witness.point_b.tolist()}
            print("rings50k", f, q, r.distance, r.witness.tri_a, r.witness.tri_b, flush=True)
        meta["rings50k"].append(rec)

    # 3. pairing topology of larger tori (many surface-area ties)
    meta["pairings"] = []
    for nu, nv in ((300, 100), (400, 150)):
        t, _ = ps.ring_pair_base(nu, nv)
        mesh = md.TriangleMesh(t.vertices, t.triangles)
        t0 = time.time()
        tr = rt.build_f12(mesh)
        name = f"torus{nu}x{nv}"
        out[f"pair_{name}_leaf"] = tr.leaf_tris.astype(np.int32)
        out[f"pair_{name}_order"] = tr.prim_order.astype(np.int32)
        meta["pairings"].append({"name": name, "nu": nu, "nv": nv, "tris": int(len(t.triangles)),
                                 "seconds": time.time() - t0})
        print("pairing", name, time.time() - t0, flush=True)

    np.savez_compressed(HERE / "golden_r2.npz", **out)
    with open(HERE / "golden_r2.json", "w") as fh:
        json.dump(meta, fh, indent=1, default=float)
    print("wrote", HERE / "golden_r2.npz", HERE / "golden_r2.json")


if __name__ == "__main__":
    main(*sys.argv[1:])
