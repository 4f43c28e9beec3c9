"""Generate the golden vectors in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container, where the read-only reference is importable:

    python tests/golden/make_golden.py [/root/reference/pkg/src]

It imports the reference package `meshdist` by path (pure Python + numpy)
and records its outputs on deterministic inputs.  The GPU box has no
/root/reference; tests there read only the committed .npz / .json files.
Inputs that need the product's new scene kinds (tori) are generated with
`paper_2411_11244_b200.scenes` (host numpy code) and stored verbatim.
"""

from __future__ import annotations

import hashlib
import importlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))


def load_reference(src: str):
    sys.path.insert(0, src)
    md = importlib.import_module("meshdist")
    assert Path(md.__file__).resolve().is_relative_to(Path(src).resolve()), md.__file__
    return md


def tri_battery(rng: np.random.Generator) -> tuple[np.ndarray, np.ndarray, list]:
    """(N, 3, 3) pairs covering generic, near-parallel, coplanar, piercing,
    degenerate, shared-feature, tie-heavy and offset configurations."""
    t1, t2, tags = [], [], []

    def add(a, b, tag):
        t1.append(np.asarray(a, dtype=np.float64))
        t2.append(np.asarray(b, dtype=np.float64))
        tags.append(tag)

    for _ in range(800):
        add(rng.normal(size=(3, 3)), rng.normal(size=(3, 3)), "random")
    for _ in range(300):
        add(rng.normal(size=(3, 3)), rng.normal(size=(3, 3)) + rng.normal(size=3) * 5.0, "far")
    for _ in range(200):  # near-parallel planes
        a = np.c_[rng.uniform(-1, 1, (3, 2)), np.zeros(3)]
        b = np.c_[rng.uniform(-1, 1, (3, 2)), np.full(3, 10.0 ** rng.uniform(-9, 0))]
        b[:, 2] += rng.normal(size=3) * 10.0 ** rng.uniform(-12, -4)
        add(a, b, "parallel")
    for _ in range(200):  # coplanar (z = 0), overlapping or not
        add(np.c_[rng.uniform(-1, 1, (3, 2)), np.zeros(3)], np.c_[rng.uniform(-1, 1, (3, 2)), np.zeros(3)], "coplanar")
    for _ in range(200):  # piercing: a segment through B's interior
        b = rng.normal(size=(3, 3))
        w = rng.dirichlet(np.ones(3))
        x = w @ b
        n = np.cross(b[1] - b[0], b[2] - b[0])
        n /= np.linalg.norm(n)
        s = rng.uniform(0.05, 1.0)
        a = np.stack([x + s * n, x - s * n * rng.uniform(0.1, 1.0), x + rng.normal(size=3)])
        add(a, b, "pierce")
    for _ in range(150):  # degenerate: collinear / repeated / point triangles
        p = rng.normal(size=3)
        d = rng.normal(size=3)
        kind = rng.integers(3)
        if kind == 0:
            a = np.stack([p, p + d, p + 2.5 * d])
        elif kind == 1:
            a = np.stack([p, p, p + d])
        else:
            a = np.stack([p, p, p])
        b = rng.normal(size=(3, 3)) if rng.random() < 0.5 else np.stack([p + d, p + d, p - d]) + rng.normal(size=3)
        add(a, b, "degenerate")
    for _ in range(150):  # shared vertex / shared edge
        a = rng.normal(size=(3, 3))
        b = rng.normal(size=(3, 3))
        b[0] = a[1]
        if rng.random() < 0.5:
            b[1] = a[2]
        add(a, b, "shared")
    for _ in range(150):  # integer grid: exact ties and zeros
        add(rng.integers(-2, 3, (3, 3)).astype(np.float64), rng.integers(-2, 3, (3, 3)).astype(np.float64), "grid")
    for _ in range(100):  # far from the origin
        off = rng.normal(size=3) * 1000.0
        add(rng.normal(size=(3, 3)) + off, rng.normal(size=(3, 3)) + off + rng.normal(size=3), "offset")
    # SPEC bounds.py examples
    add([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 0, 1], [1, 0, 1], [0, 1, 1]], "spec-parallel")
    add([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0.2, 0.2, 0], [1.2, 0.2, 0], [0.2, 1.2, 0]], "spec-coplanar")
    add([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 0, 0], [1, 0, 0], [0, 1, 0]], "spec-identical")
    return np.stack(t1), np.stack(t2), tags


def box_battery(rng: np.random.Generator):
    lo_a, hi_a, lo_b, hi_b = [], [], [], []
    for i in range(2000):
        c = rng.normal(size=(2, 3)) * (0.2 if i % 3 == 0 else 2.0)
        e = np.abs(rng.normal(size=(2, 3)))
        if i % 7 == 0:
            e[0] = 0.0  # point box
        if i % 11 == 0:
            e[1, rng.integers(3)] = 0.0  # flat box
        if i % 13 == 0:
            c[1] = c[0]
            e[1] = e[0]  # identical boxes
        if i % 17 == 0:
            c = np.round(c)
            e = np.round(e + 0.5)
        lo_a.append(c[0] - e[0])
        hi_a.append(c[0] + e[0])
        lo_b.append(c[1] - e[1])
        hi_b.append(c[1] + e[1])
    return [np.asarray(x) for x in (lo_a, hi_a, lo_b, hi_b)]


def sha(mesh) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(mesh.vertices, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(mesh.triangles, dtype=np.int64).tobytes())
    return h.hexdigest()


def main(src: str = "/root/reference/pkg/src"):
    md = load_reference(src)
    from meshdist import bounds as rb, bvh as rt, query as rq

    from paper_2411_11244_b200 import scenes as ps

    rng = np.random.default_rng(20241117)
    out: dict = {}
    meta: dict = {"reference": src, "generated_by": "tests/golden/make_golden.py"}

    # 1. narrow phase battery, float64 and float32
    t1, t2, tags = tri_battery(rng)
    out["tri_t1"], out["tri_t2"] = t1, t2
    meta["tri_tags"] = tags
    for prec, dt in ((64, np.float64), (32, np.float32)):
        a, b = t1.astype(dt), t2.astype(dt)
        d, p, q = rb.batch_tri_tri_min(a, b)
        out[f"tri_min{prec}_d"], out[f"tri_min{prec}_p"], out[f"tri_min{prec}_q"] = d, p, q
        d, p, q = rb.batch_tri_tri_max(a, b)
        out[f"tri_max{prec}_d"], out[f"tri_max{prec}_p"], out[f"tri_max{prec}_q"] = d, p, q

    # 2. box bounds battery
    boxes = box_battery(rng)
    for i, name in enumerate(("box_amin", "box_amax", "box_bmin", "box_bmax")):
        out[name] = boxes[i]
    for prec, dt in ((64, np.float64), (32, np.float32)):
        bx = [x.astype(dt) for x in boxes]
        out[f"box_min_lower{prec}"] = rb.batch_min_lower(*bx)
        out[f"box_max_upper{prec}"] = rb.batch_max_upper(*bx)
        out[f"box_enh_min_upper{prec}"] = rb.batch_enhanced_min_upper(*bx)
        out[f"box_enh_max_lower{prec}"] = rb.batch_enhanced_max_lower(*bx)

    # 3. trees: structure + boxes (SPEC acceptance 7 sizes and more)
    tree_cases = []
    for n in (1, 2, 3, 4, 5, 7, 8, 13, 100, 1000, 1500, 3333):
        ma, _ = md.gen_scene("random-blobs", {"n": n, "seed": n})
        tree_cases.append((f"blobs{n}", ma))
    tz, tb = ps.ring_pair_base(40, 25)  # 2000 tris, indexed, not a power of two
    tree_cases.append(("torus2000", md.TriangleMesh(tz.vertices, tz.triangles)))
    meta["trees"] = []
    for name, mesh in tree_cases:
        out[f"tree_{name}_V"] = mesh.vertices
        out[f"tree_{name}_T"] = mesh.triangles
        for prec, dt in ((64, np.float64), (32, np.float32)):
            t = rt.build_f12(mesh, dtype=dt)
            out[f"tree_{name}_min{prec}"] = t.node_min
            out[f"tree_{name}_max{prec}"] = t.node_max
        out[f"tree_{name}_leaf"] = t.leaf_tris
        out[f"tree_{name}_order"] = t.prim_order
        out[f"tree_{name}_depth"] = np.asarray(t.depth)
        meta["trees"].append(name)
    # pairing-only cases at larger n (tori and blobs, many SA ties in tori)
    meta["pairings"] = []
    for nu, nv in ((60, 41), (97, 53), (120, 70)):
        tz, _ = ps.ring_pair_base(nu, nv)
        mesh = md.TriangleMesh(tz.vertices, tz.triangles)
        t0 = time.time()
        t = rt.build_f12(mesh)
        name = f"torus{nu}x{nv}"
        out[f"pair_{name}_leaf"] = t.leaf_tris.astype(np.int32)
        out[f"pair_{name}_order"] = t.prim_order.astype(np.int32)
        meta["pairings"].append({"name": name, "nu": nu, "nv": nv, "seconds": time.time() - t0})

    # 4. engine battery vs brute force, 64 and 32 bit
    battery = []
    for seed in range(8):
        battery.append(("random-blobs", {"n": 60 + 40 * seed, "seed": seed, "gap": 0.1 * seed}))
    for res in (6, 9, 12, 15):
        battery.append(("offset-grids", {"res": res, "seed": res, "gap": 0.25 + 0.05 * res}))
    for lat, lon in ((6, 8), (8, 12), (10, 14)):
        battery.append(("nested-shells", {"lat": lat, "lon": lon, "r_inner": 0.8, "r_outer": 0.9}))
    for seed in range(3):
        battery.append(("intersecting-clusters", {"n": 150 + 100 * seed, "seed": seed}))
    meta["engine"] = []
    for kind, params in battery:
        ma, mb = md.gen_scene(kind, params)
        rec = {"kind": kind, "params": params, "hash_a": sha(ma), "hash_b": sha(mb)}
        for prec in (64, 32):
            dt = np.float64 if prec == 64 else np.float32
            ta, tb = rt.build_f12(ma, dtype=dt), rt.build_f12(mb, dtype=dt)
            cfg = rq.EngineConfig(precision=prec)
            for q in ("min", "max"):
                r = (rq.run_min_query if q == "min" else rq.run_max_query)(ma, mb, ta, tb, cfg)
                bf = (rq.brute_force_min if q == "min" else rq.brute_force_max)(ma, mb, dtype=dt)
                rec[f"{q}{prec}"] = {
                    "distance": r.distance,
                    "tri_a": r.witness.tri_a,
                    "tri_b": r.witness.tri_b,
                    "point_a": r.witness.point_a.tolist(),
                    "point_b": r.witness.point_b.tolist(),
                    "witness_exact": r.witness_exact,
                    "iterations": [[s.k, s.front_in, s.front_out, s.culled, s.bound_after] for s in r.iterations],
                    "expanded_pairs": r.expanded_pairs,
                    "narrow_pairs": r.narrow_pairs,
                    "brute_distance": bf[0],
                    "brute_tri_a": bf[1].tri_a,
                    "brute_tri_b": bf[1].tri_b,
                }
        meta["engine"].append(rec)

    # 5. config 1: two ~10K tori, generic interlock (BASELINE.json configs[0])
    ma, mb = ps.gen_scene("interlocked-rings", {"nu": 100, "nv": 50})
    ra, rbm = md.TriangleMesh(ma.vertices, ma.triangles), md.TriangleMesh(mb.vertices, mb.triangles)
    ta, tb = rt.build_f12(ra), rt.build_f12(rbm)
    cfg1 = {"hash_a": sha(ra), "hash_b": sha(rbm)}
    for q in ("min", "max"):
        t0 = time.time()
        r = (rq.run_min_query if q == "min" else rq.run_max_query)(ra, rbm, ta, tb)
        cfg1[q] = {"distance": r.distance, "tri_a": r.witness.tri_a, "tri_b": r.witness.tri_b,
                   "point_a": r.witness.point_a.tolist(), "point_b": r.witness.point_b.tolist(),
                   "seconds": time.time() - t0, "narrow_pairs": r.narrow_pairs,
                   "expanded_pairs": r.expanded_pairs}
    meta["config1"] = cfg1
    # a few rotation-sequence frames of config 1 (config 3 definition)
    tz, tbase = ps.ring_pair_base(100, 50)
    meta["frames"] = []
    for f in (1, 137, 500, 999):
        xa, xb = ps.ring_frame_transforms(f)
        va = tz.vertices @ xa.rotation.T + xa.translation
        vb = tbase.vertices @ xb.rotation.T + xb.translation
        fa, fb = md.TriangleMesh(va, tz.triangles), md.TriangleMesh(vb, tbase.triangles)
        ta, tb = rt.build_f12(fa), rt.build_f12(fb)
        rec = {"frame": f, "hash_a": sha(fa), "hash_b": sha(fb)}
        for q in ("min", "max"):
            r = (rq.run_min_query if q == "min" else rq.run_max_query)(fa, fb, ta, tb)
            rec[q] = {"distance": r.distance, "tri_a": r.witness.tri_a, "tri_b": r.witness.tri_b}
        meta["frames"].append(rec)

    # 6. scene hashes (bitwise generator parity)
    meta["scenes"] = []
    for kind, params in [("random-blobs", {}), ("random-blobs", {"n": 77, "seed": 5, "gap": 0.0}),
                         ("intersecting-clusters", {}), ("intersecting-clusters", {"n": 1, "seed": 3}),
                         ("nested-shells", {}), ("nested-shells", {"lat": 31, "lon": 17, "r_outer": 0.81}),
                         ("offset-grids", {}), ("offset-grids", {"res": 7, "gap": 0.1, "seed": 9})]:
        ma, mb = md.gen_scene(kind, params)
        meta["scenes"].append({"kind": kind, "params": params, "hash_a": sha(ma), "hash_b": sha(mb)})

    # 7. SPEC known-answer examples, as the reference computes them
    A = md.Aabb
    unit = A([0, 0, 0], [1, 1, 1], tight=True)
    kat = {
        "min_lower_gap_x": md.aabb_min_lower(A([0, 0, 0], [1, 1, 1]), A([2, 0, 0], [3, 1, 1])),
        "min_lower_overlap": md.aabb_min_lower(A([0, 0, 0], [1, 1, 1]), A([0.5, 0.5, 0.5], [2, 2, 2])),
        "min_lower_diag": md.aabb_min_lower(A([0, 0, 0], [1, 1, 1]), A([2, 2, 2], [3, 3, 3])),
        "max_upper_unit": md.aabb_max_upper(unit, unit),
        "max_upper_point": md.aabb_max_upper(A([0, 0, 0], [0, 0, 0]), A([1, 1, 1], [2, 2, 2])),
        "enh_min_upper_unit": md.enhanced_min_upper(unit, unit),
        "enh_max_lower_unit": md.enhanced_max_lower(unit, unit),
        "descendant_0_1_0": md.descendant(0, 1, 0),
        "descendant_0_2_3": md.descendant(0, 2, 3),
        "descendant_2_2_0": md.descendant(2, 2, 0),
    }
    cfg = rq.EngineConfig()
    kat["adaptive_1"] = rq.adaptive_depth(1, cfg, 10)
    kat["adaptive_100000"] = rq.adaptive_depth(100000, cfg, 10)
    kat["adaptive_1000_rem2"] = rq.adaptive_depth(1000, cfg, 2)
    meta["kat"] = kat

    np.savez_compressed(HERE / "golden.npz", **out)
    with open(HERE / "golden.json", "w") as fh:
        json.dump(meta, fh, indent=1, default=float)
    print("wrote", HERE / "golden.npz", HERE / "golden.json")


if __name__ == "__main__":
    main(*sys.argv[1:])
