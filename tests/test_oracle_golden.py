"""The oracle restatement reproduces the reference's own outputs (golden
vectors from tests/golden/make_golden.py) bit for bit.  CPU only."""

from pathlib import Path

import numpy as np
import pytest


def _eq(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape and a.dtype == b.dtype, (a.shape, b.shape, a.dtype, b.dtype)
    bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
    assert not bad.any(), f"{bad.sum()} mismatches, first at {np.argwhere(bad)[:3].tolist()}"


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("kind", ["min", "max"])
def test_tri_tri_battery(golden, oracle, prec, kind):
    dt = np.float64 if prec == 64 else np.float32
    t1, t2 = golden["tri_t1"].astype(dt), golden["tri_t2"].astype(dt)
    fn = oracle.tri_tri_min if kind == "min" else oracle.tri_tri_max
    d, p, q = fn(t1, t2)
    _eq(d, golden[f"tri_{kind}{prec}_d"])
    _eq(p, golden[f"tri_{kind}{prec}_p"])
    _eq(q, golden[f"tri_{kind}{prec}_q"])


@pytest.mark.parametrize("prec", [64, 32])
def test_box_bounds_battery(golden, oracle, prec):
    dt = np.float64 if prec == 64 else np.float32
    bx = [golden[k].astype(dt) for k in ("box_amin", "box_amax", "box_bmin", "box_bmax")]
    _eq(oracle.box_min_lower(*bx), golden[f"box_min_lower{prec}"])
    _eq(oracle.box_max_upper(*bx), golden[f"box_max_upper{prec}"])
    _eq(oracle.enhanced_min_upper(*bx), golden[f"box_enh_min_upper{prec}"])
    _eq(oracle.enhanced_max_lower(*bx), golden[f"box_enh_max_lower{prec}"])


def test_bound_sandwich(golden, oracle):
    """SPEC acceptance 4 on the golden boxes: lower <= enhanced <= upper."""
    bx = [golden[k] for k in ("box_amin", "box_amax", "box_bmin", "box_bmax")]
    lo, hi = oracle.box_min_lower(*bx), oracle.box_max_upper(*bx)
    emu, eml = oracle.enhanced_min_upper(*bx), oracle.enhanced_max_lower(*bx)
    assert (lo <= emu).all() and (emu <= hi).all()
    assert (lo <= eml).all() and (eml <= hi).all()


def test_trees(golden, golden_meta, oracle):
    for name in golden_meta["trees"]:
        V, T = golden[f"tree_{name}_V"], golden[f"tree_{name}_T"]
        for prec, dt in ((64, np.float64), (32, np.float32)):
            t = oracle.build_tree(V, T, dtype=dt)
            _eq(t.node_min, golden[f"tree_{name}_min{prec}"])
            _eq(t.node_max, golden[f"tree_{name}_max{prec}"])
        _eq(t.leaf_tris, golden[f"tree_{name}_leaf"])
        _eq(t.prim_order, golden[f"tree_{name}_order"])
        assert t.depth == int(golden[f"tree_{name}_depth"])


def test_pairings(golden, golden_meta, oracle):
    from paper_2411_11244_b200.scenes import ring_pair_base

    for rec in golden_meta["pairings"]:
        tz, _ = ring_pair_base(rec["nu"], rec["nv"])
        t = oracle.build_tree(tz.vertices, tz.triangles)
        _eq(t.leaf_tris.astype(np.int32), golden[f"pair_{rec['name']}_leaf"])
        _eq(t.prim_order.astype(np.int32), golden[f"pair_{rec['name']}_order"])


def _scene(md, rec):
    return md.gen_scene(rec["kind"], rec["params"])


def test_engine_battery(golden_meta, oracle, md):
    for rec in golden_meta["engine"]:
        ma, mb = _scene(md, rec)
        for prec in (64, 32):
            dt = np.float64 if prec == 64 else np.float32
            ta = oracle.build_tree(ma.vertices, ma.triangles, dtype=dt)
            tb = oracle.build_tree(mb.vertices, mb.triangles, dtype=dt)
            pa, pb = ma.triangle_points(dt), mb.triangle_points(dt)
            for q in ("min", "max"):
                r = oracle.run_query(ta, tb, pa, pb, q, oracle.Config(precision=prec))
                g = rec[f"{q}{prec}"]
                assert r.distance == g["distance"], (rec["kind"], rec["params"], q, prec)
                assert (r.tri_a, r.tri_b) == (g["tri_a"], g["tri_b"])
                assert r.point_a.tolist() == g["point_a"] and r.point_b.tolist() == g["point_b"]
                assert [list(s) for s in r.iterations] == g["iterations"]
                assert (r.expanded_pairs, r.narrow_pairs) == (g["expanded_pairs"], g["narrow_pairs"])


def test_brute_force_small(golden_meta, oracle, md):
    for rec in golden_meta["engine"][:6]:
        ma, mb = _scene(md, rec)
        for q in ("min", "max"):
            d, ta, tb, _, _ = oracle.brute_force(ma.triangle_points(), mb.triangle_points(), q)
            g = rec[f"{q}64"]
            assert (d, ta, tb) == (g["brute_distance"], g["brute_tri_a"], g["brute_tri_b"])


def test_config1_tori(golden_meta, oracle, md):
    g = golden_meta["config1"]
    ma, mb = md.gen_scene("interlocked-rings", {"nu": 100, "nv": 50})
    ta = oracle.build_tree(ma.vertices, ma.triangles)
    tb = oracle.build_tree(mb.vertices, mb.triangles)
    for q in ("min", "max"):
        r = oracle.run_query(ta, tb, ma.triangle_points(), mb.triangle_points(), q)
        assert r.distance == g[q]["distance"]
        assert (r.tri_a, r.tri_b) == (g[q]["tri_a"], g[q]["tri_b"])


def test_kat(golden_meta, oracle):
    k = golden_meta["kat"]
    box = lambda lo, hi: (np.array([lo], float), np.array([hi], float))  # noqa: E731
    a, b = box([0, 0, 0], [1, 1, 1]), box([2, 0, 0], [3, 1, 1])
    assert oracle.box_min_lower(*a, *b)[0] == k["min_lower_gap_x"] == 1.0
    u = box([0, 0, 0], [1, 1, 1])
    assert oracle.enhanced_min_upper(*u, *u)[0] == k["enh_min_upper_unit"]
    assert oracle.enhanced_max_lower(*u, *u)[0] == k["enh_max_lower_unit"] == 1.0
    assert oracle.box_max_upper(*u, *u)[0] == k["max_upper_unit"]
    cfg = oracle.Config()
    assert oracle.adaptive_k(1, cfg, 10) == k["adaptive_1"] == 5
    assert oracle.adaptive_k(100000, cfg, 10) == k["adaptive_100000"] == 1
    assert oracle.adaptive_k(1000, cfg, 2) == k["adaptive_1000_rem2"] == 2


@pytest.mark.parametrize("seed", range(4))
def test_fast_pairing_matches_literal_greedy(oracle, seed):
    """oracle/pairing.c (the O(n log n) restatement) == the reference's
    literal greedy loop (bvh.py:122-166) on random and tie-heavy keys."""
    rng = np.random.default_rng(100 + seed)
    for n in list(range(2, 80)) + [127, 255, 257, 511, 513, 1023, 2049, 3001]:
        sa = np.round(rng.random(n - 1) * 8) / 8 if seed % 2 else rng.random(n - 1)
        assert oracle.greedy_pairs_fast(sa, n).tolist() == oracle.greedy_pairs(sa, n), (seed, n)


def test_fast_pairing_large_tori_golden(oracle):
    """The reference's own pairing of 60K / 120K-triangle tori
    (tests/golden/golden_r2.npz, make_golden_r2.py)."""
    import json

    from paper_2411_11244_b200.scenes import ring_pair_base

    here = Path(__file__).resolve().parent / "golden"
    meta = json.loads((here / "golden_r2.json").read_text())
    arr = np.load(here / "golden_r2.npz")
    for rec in meta["pairings"]:
        tz, _ = ring_pair_base(rec["nu"], rec["nv"])
        V, T = tz.vertices, tz.triangles
        _, order = oracle.morton_order(V, T)
        P = V[T]
        sa = oracle.pair_surface_areas(order, P.min(axis=1), P.max(axis=1))
        leaf = oracle.leaves_from_pairs(order, oracle.greedy_pairs_fast(sa, len(T)), len(T))
        _eq(leaf.astype(np.int32), arr[f"pair_{rec['name']}_leaf"])
        _eq(order.astype(np.int32), arr[f"pair_{rec['name']}_order"])


def test_oracle_nested_shells_config4_geometry(oracle, md):
    """The oracle's engine reproduces the reference's config-4 geometry
    answers (nested shells r 0.8 / 0.81, golden_r2.json) at the smallest
    recorded size: distance and witness, float64 and float32."""
    import json

    meta = json.loads((Path(__file__).resolve().parent / "golden" / "golden_r2.json").read_text())
    rec = meta["shells"][0]
    a, b = md.gen_scene("nested-shells", rec["params"])
    for prec, dt in ((64, np.float64), (32, np.float32)):
        ta = oracle.build_tree(a.vertices, a.triangles, dtype=dt)
        tb = oracle.build_tree(b.vertices, b.triangles, dtype=dt)
        cfg = oracle.Config(precision=prec, front_hard_cap=1 << 30)
        for kind in ("min", "max"):
            r = oracle.run_query(ta, tb, a.triangle_points(dt), b.triangle_points(dt), kind, cfg)
            want = rec[f"{kind}{prec}"]
            assert r.distance == want["distance"], (prec, kind)
            assert (r.tri_a, r.tri_b) == (want["tri_a"], want["tri_b"]), (prec, kind)
