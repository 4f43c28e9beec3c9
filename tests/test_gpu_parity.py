"""Parity of the CUDA path with the reference (golden vectors made by the
reference itself) and with the CPU oracle.  Bar: bitwise for the exact
kernels, trees and query distances; witness = the brute-force witness
(lexicographically smallest tied pair)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _eq(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
    assert not bad.any(), f"{what}: {bad.sum()} mismatches, first {np.argwhere(bad)[:3].tolist()}"


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("kind", ["min", "max"])
def test_tri_tri_exact_bitwise(md, gpu, golden, prec, kind):
    dt = np.float64 if prec == 64 else np.float32
    t1, t2 = golden["tri_t1"].astype(dt), golden["tri_t2"].astype(dt)
    d, p, q = (md.batch_tri_tri_min if kind == "min" else md.batch_tri_tri_max)(t1, t2)
    assert d.dtype == dt
    _eq(d, golden[f"tri_{kind}{prec}_d"], "d")
    _eq(p, golden[f"tri_{kind}{prec}_p"], "p")
    _eq(q, golden[f"tri_{kind}{prec}_q"], "q")


@pytest.mark.parametrize("kind", ["min", "max"])
def test_tri_tri_fast_within_slack(md, gpu, golden, kind):
    """The traversal's float32 filter stays within E/2 = 2^-16 * max|coord|
    of the float64 reference distance."""
    from paper_2411_11244_b200.bounds import tri_tri_fast

    t1, t2 = golden["tri_t1"], golden["tri_t2"]
    ref = golden[f"tri_{kind}64_d"]
    fast = tri_tri_fast(kind, t1, t2).astype(np.float64)
    M = np.maximum(np.abs(t1).reshape(len(t1), -1).max(1), np.abs(t2).reshape(len(t2), -1).max(1))
    M = np.maximum(M, np.abs(t1.astype(np.float32)).reshape(len(t1), -1).max(1))
    err = np.abs(fast - ref) / (M * 2.0**-16)
    assert err.max() <= 1.0, f"max error {err.max():.3g} x (E/2) at {int(err.argmax())}"


def _adversarial_pairs(rng, n):
    """Near-parallel, near-touching, sliver and coplanar triangle pairs --
    where the float32 closest points are ill-conditioned
    (scripts/exp_narrow_error.py has the full families)."""
    a = rng.normal(size=(n, 3, 3))
    out = []
    b = a + rng.normal(size=(n, 1, 3)) * 1e-3 + rng.normal(size=(n, 3, 3)) * 10.0 ** rng.uniform(-9, -2, (n, 1, 1))
    out.append((a, b))  # near-parallel (nearly translated copies)
    mid = 0.5 * (a[:, 0] + a[:, 1])
    b = rng.normal(size=(n, 3, 3))
    b += (mid - b[:, 0])[:, None, :] + rng.normal(size=(n, 1, 3)) * 10.0 ** rng.uniform(-8, -2, (n, 1, 1))
    out.append((a, b))  # near-touching
    s = a.copy()
    t = rng.uniform(size=(n, 1))
    s[:, 2] = s[:, 0] * t + s[:, 1] * (1 - t) + rng.normal(size=(n, 3)) * 10.0 ** rng.uniform(-8, -3, (n, 1))
    out.append((s, rng.normal(size=(n, 3, 3)) * 0.5 + rng.normal(size=(n, 1, 3))))  # slivers
    c = rng.normal(size=(n, 3, 3))
    c[:, :, 2] = 0.0
    d = rng.normal(size=(n, 3, 3))
    d[:, :, 2] = 10.0 ** rng.uniform(-9, -1, size=(n, 1))
    out.append((c, d))  # coplanar / nearly
    return out


def test_tri_tri_min_lower_bound(md, gpu):
    """The exact band windows on a conditioning-aware float32 lower bound
    of the min distance (geometry.cuh tri_tri_min_fast_lb): it never exceeds
    the reference's float64 distance by more than rounding (4 ulps of the
    coordinate scale), although the raw float32 estimate overshoots it by up
    to ~290 ulps on such pairs (beyond the band's E / 2 = 128)."""
    from paper_2411_11244_b200.bounds import tri_tri_fast

    rng = np.random.default_rng(11)
    for fam, (a, b) in enumerate(_adversarial_pairs(rng, 1 << 17)):
        a32, b32 = a.astype(np.float32), b.astype(np.float32)
        lb = tri_tri_fast("min-lb", a32, b32).astype(np.float64)
        fast = tri_tri_fast("min", a32, b32).astype(np.float64)
        ref = md.batch_tri_tri_min(a, b)[0]
        M = np.maximum(np.abs(a).reshape(len(a), -1).max(1), np.abs(b).reshape(len(b), -1).max(1))
        ulp = M * 2.0 ** -23
        assert ((lb - ref) / ulp).max() <= 4.0, fam
        assert np.all(lb <= fast + 4.0 * ulp)  # the estimate of another code path: rounding apart


def test_near_contact_overestimate_scene(md, gpu):
    """A scene built so that the round-1 band (windowing on the raw float32
    distance with slack E) returned the wrong pair: triangle pair (a, b) is
    the optimum, but its float32 distance overshoots the reference's by far
    more than E (a near-touching, ill-conditioned configuration, ~1700 float32
    ulps), while (a, b2) -- b2 a copy of a moved along a's normal, a few ulps
    farther -- is estimated exactly.  With the conditioning-aware lower bound
    the engine returns the brute-force answer."""
    from paper_2411_11244_b200.bounds import tri_tri_fast

    rng = np.random.default_rng(1)
    n = 1 << 20
    a = rng.normal(size=(n, 3, 3))
    b = rng.normal(size=(n, 3, 3))
    mid = 0.5 * (a[:, 0] + a[:, 1])
    b += (mid - b[:, 0])[:, None, :] + rng.normal(size=(n, 1, 3)) * 10.0 ** rng.uniform(-8, -2, (n, 1, 1))
    i = 515104
    ta = a[i].astype(np.float32).astype(np.float64)
    tb = b[i].astype(np.float32).astype(np.float64)
    d1 = float(md.batch_tri_tri_min(ta[None], tb[None])[0][0])
    nrm = np.cross(ta[1] - ta[0], ta[2] - ta[0])
    nrm /= np.linalg.norm(nrm)
    M = max(np.abs(ta).max(), np.abs(tb).max())
    ulp = M * 2.0 ** -23
    chosen = None
    for k in range(1, 400):
        for sgn in (1.0, -1.0):
            tb2 = (ta + sgn * (d1 + k * ulp) * nrm).astype(np.float32).astype(np.float64)
            d2 = float(md.batch_tri_tri_min(ta[None], tb2[None])[0][0])
            if d1 < d2 < d1 + 30 * ulp:
                chosen = tb2
                break
        if chosen is not None:
            break
    assert chosen is not None
    f_opt = float(tri_tri_fast("min", ta[None].astype(np.float32), tb[None].astype(np.float32))[0])
    f_alt = float(tri_tri_fast("min", ta[None].astype(np.float32), chosen[None].astype(np.float32))[0])
    E = 2.0 ** -15 * max(M, np.abs(chosen).max())
    assert f_opt > f_alt + E  # the raw float32 window would have dropped the optimum
    A = md.TriangleMesh(ta, np.array([[0, 1, 2]]))
    B = md.TriangleMesh(np.concatenate([tb, chosen]), np.array([[0, 1, 2], [3, 4, 5]]))
    for prec, dt in ((64, np.float64), (32, np.float32)):
        tA, tB = md.build_f12(A, dtype=dt), md.build_f12(B, dtype=dt)
        r = md.run_min_query(A, B, tA, tB, md.EngineConfig(precision=prec))
        d, w = md.brute_force_min(A, B, dtype=dt)
        assert r.distance == d and (r.witness.tri_a, r.witness.tri_b) == (w.tri_a, w.tri_b), prec
        if prec == 64:
            assert (w.tri_a, w.tri_b) == (0, 0)  # the ill-conditioned pair is the float64 optimum


@pytest.mark.parametrize("prec", [64, 32])
def test_box_bounds_bitwise(md, gpu, golden, prec):
    dt = np.float64 if prec == 64 else np.float32
    bx = [golden[k].astype(dt) for k in ("box_amin", "box_amax", "box_bmin", "box_bmax")]
    _eq(md.batch_min_lower(*bx), golden[f"box_min_lower{prec}"], "min_lower")
    _eq(md.batch_max_upper(*bx), golden[f"box_max_upper{prec}"], "max_upper")
    _eq(md.batch_enhanced_min_upper(*bx), golden[f"box_enh_min_upper{prec}"], "enh_min_upper")
    _eq(md.batch_enhanced_max_lower(*bx), golden[f"box_enh_max_lower{prec}"], "enh_max_lower")


def test_scalar_kat(md, gpu, golden_meta):
    k = golden_meta["kat"]
    A = md.Aabb
    unit = A([0, 0, 0], [1, 1, 1], tight=True)
    assert md.aabb_min_lower(A([0, 0, 0], [1, 1, 1]), A([2, 0, 0], [3, 1, 1])) == k["min_lower_gap_x"]
    assert md.aabb_min_lower(A([0, 0, 0], [1, 1, 1]), A([2, 2, 2], [3, 3, 3])) == k["min_lower_diag"]
    assert md.aabb_max_upper(A([0, 0, 0], [0, 0, 0]), A([1, 1, 1], [2, 2, 2])) == k["max_upper_point"]
    assert md.enhanced_min_upper(unit, unit) == k["enh_min_upper_unit"]
    assert md.enhanced_max_lower(unit, unit) == k["enh_max_lower_unit"]
    with pytest.raises(md.TightnessError):
        md.enhanced_min_upper(A([0, 0, 0], [1, 1, 1]), unit)
    d, p, q = md.tri_tri_min([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 0, 1], [1, 0, 1], [0, 1, 1]])
    assert d == 1.0
    d, _, _ = md.tri_tri_max([[0, 0, 0], [3, 0, 0], [0, 1, 0]], [[0, 0, 0], [3, 0, 0], [0, 1, 0]])
    assert d == np.sqrt(10.0)


def test_build_trees_bitwise(md, gpu, golden, golden_meta):
    for name in golden_meta["trees"]:
        mesh = md.TriangleMesh(golden[f"tree_{name}_V"], golden[f"tree_{name}_T"])
        for prec, dt in ((64, np.float64), (32, np.float32)):
            t = md.build_f12(mesh, dtype=dt)
            _eq(t.prim_order, golden[f"tree_{name}_order"], f"{name} order")
            _eq(t.leaf_tris, golden[f"tree_{name}_leaf"], f"{name} leaves")
            assert t.depth == int(golden[f"tree_{name}_depth"])
            assert t.node_min.dtype == dt
            _eq(t.node_min, golden[f"tree_{name}_min{prec}"], f"{name} min{prec}")
            _eq(t.node_max, golden[f"tree_{name}_max{prec}"], f"{name} max{prec}")


def test_build_pairing_tori(md, gpu, golden, golden_meta):
    for rec in golden_meta["pairings"]:
        tz, _ = md.ring_pair_base(rec["nu"], rec["nv"])
        t = md.build_f12(tz)
        _eq(t.leaf_tris.astype(np.int32), golden[f"pair_{rec['name']}_leaf"], rec["name"])
        _eq(t.prim_order.astype(np.int32), golden[f"pair_{rec['name']}_order"], rec["name"])


def test_build_structure_suite(md, gpu, oracle):
    """SPEC acceptance 7: fullness, 1-2 triangle leaves, tight containment,
    build -> refit fixed point, at sizes 1, 2, 3, 4, 5, 7, 1000."""
    for n in (1, 2, 3, 4, 5, 7, 1000):
        a, _ = md.gen_scene("random-blobs", {"n": n, "seed": 3})
        t = md.build_f12(a)
        L = t.leaf_count
        assert L & (L - 1) == 0 and L <= n < 2 * L and t.n_nodes == 2 * L - 1
        ids = t.leaf_tris[t.leaf_tris >= 0]
        assert sorted(ids.tolist()) == list(range(n))
        before = (t.node_min.copy(), t.node_max.copy())
        md.refit(t, a)
        _eq(t.node_min, before[0])
        _eq(t.node_max, before[1])
        P = a.triangle_points()
        for node in range(t.n_nodes):
            lo_d = t.depth - md.remaining_depth(t, node)
            first = ((node + 1) << (t.depth - lo_d)) - 1 - (L - 1)
            ranks = range(first, first + (1 << (t.depth - lo_d)))
            tris = [x for r in ranks for x in t.leaf_prims(r)]
            pts = P[tris].reshape(-1, 3)
            assert np.array_equal(pts.min(0), t.node_min[node]) and np.array_equal(pts.max(0), t.node_max[node])


def test_refit_moved_mesh(md, gpu, oracle):
    a, _ = md.gen_scene("interlocked-rings", {"nu": 60, "nv": 30})
    t = md.build_f12(a)
    xf = md.RigidTransform.from_axis_angle((0.3, -1, 2), 1.3, (0.5, -0.25, 2.0))
    moved = md.apply_transform(a, xf)
    md.refit(t, moved)
    # same topology, boxes recomputed from the reference's moved vertices
    ref = oracle.Tree(np.empty((t.n_nodes, 3)), np.empty((t.n_nodes, 3)), t.leaf_tris, t.prim_order, t.depth)
    oracle.fill_boxes(ref, moved.vertices, moved.triangles)
    # the lazy device transform reproduces numpy's dgemm vertices bit for bit
    assert np.array_equal(t.node_min, ref.node_min) and np.array_equal(t.node_max, ref.node_max)
    # so does a refit with an explicitly materialised mesh
    md.refit(t, md.TriangleMesh(moved.vertices, moved.triangles))
    assert np.array_equal(t.node_min, ref.node_min) and np.array_equal(t.node_max, ref.node_max)
    with pytest.raises(md.TopologyMismatchError):
        md.refit(t, md.gen_scene("random-blobs", {"n": 7})[0])
    # translation commutes with min/max (SPEC refit example)
    t2 = md.build_f12(a)
    md.refit(t2, md.apply_transform(a, md.RigidTransform(np.eye(3), (1.0, 2.0, 3.0))))
    assert np.array_equal(t2.node_min, md.build_f12(a).node_min + [1.0, 2.0, 3.0])


def _check_query(md, ma, mb, prec, rec_q, tag):
    dt = np.float64 if prec == 64 else np.float32
    ta, tb = md.build_f12(ma, dtype=dt), md.build_f12(mb, dtype=dt)
    cfg = md.EngineConfig(precision=prec)
    for q in ("min", "max"):
        g = rec_q(q)
        r = (md.run_min_query if q == "min" else md.run_max_query)(ma, mb, ta, tb, cfg)
        assert r.distance == g["distance"], (tag, q, prec, r.distance, g["distance"])
        assert r.distance == g["brute_distance"]
        assert (r.witness.tri_a, r.witness.tri_b) == (g["brute_tri_a"], g["brute_tri_b"]), (tag, q, prec)
        assert r.witness_exact
        if (r.witness.tri_a, r.witness.tri_b) == (g["tri_a"], g["tri_b"]):
            assert r.witness.point_a.tolist() == g["point_a"] and r.witness.point_b.tolist() == g["point_b"]


@pytest.mark.parametrize("prec", [64, 32])
def test_engine_battery(md, gpu, golden_meta, prec):
    for rec in golden_meta["engine"]:
        ma, mb = md.gen_scene(rec["kind"], rec["params"])
        _check_query(md, ma, mb, prec, lambda q: rec[f"{q}{prec}"], (rec["kind"], rec["params"]))


def test_config1_tori_golden(md, gpu, golden_meta):
    g = golden_meta["config1"]
    a, b = md.gen_scene("interlocked-rings", {"nu": 100, "nv": 50})
    ta, tb = md.build_f12(a), md.build_f12(b)
    for q in ("min", "max"):
        r = (md.run_min_query if q == "min" else md.run_max_query)(a, b, ta, tb)
        assert r.distance == g[q]["distance"]
        assert (r.witness.tri_a, r.witness.tri_b) == (g[q]["tri_a"], g[q]["tri_b"])
        assert r.witness.point_a.tolist() == g[q]["point_a"]
        assert r.witness.point_b.tolist() == g[q]["point_b"]
    d, pair = md.min_distance(a, b)
    assert d == g["min"]["distance"] and pair == (g["min"]["tri_a"], g["min"]["tri_b"])
    d, pair = md.max_distance(a, b)
    assert d == g["max"]["distance"] and pair == (g["max"]["tri_a"], g["max"]["tri_b"])


def test_rotation_frames_golden(md, gpu, golden_meta):
    """Config-3 frames through the lazy device transform + refit: the
    reference's distances and witnesses bit for bit (the device transform
    follows numpy's dgemm arithmetic, engine.cuh mesh_vertex)."""
    tz, tb = md.ring_pair_base(100, 50)
    bvh_a, bvh_b = md.build_f12(tz), md.build_f12(tb)
    for rec in golden_meta["frames"]:
        xa, xb = md.ring_frame_transforms(rec["frame"])
        a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
        md.refit(bvh_a, a)
        md.refit(bvh_b, b)
        for q in ("min", "max"):
            r = (md.run_min_query if q == "min" else md.run_max_query)(a, b, bvh_a, bvh_b)
            assert r.distance == rec[q]["distance"], (rec["frame"], q)
            assert (r.witness.tri_a, r.witness.tri_b) == (rec[q]["tri_a"], rec[q]["tri_b"])
        d, pair = md.min_distance(tz, b, xa)
        assert d == rec["min"]["distance"] and pair == (rec["min"]["tri_a"], rec["min"]["tri_b"])


def test_rotation_frames_golden_sequence_paths(md, gpu, golden_meta):
    """The same golden config-3 frames through the sequence drivers: the
    temporal warm start (run_sequence(warm=True): each frame seeded on the
    device with the previous frame's witness), the pipelined and plain
    loops, and the per-frame CUDA graph (run_sequence_minmax: refit A + refit B + min
    + max replayed as one graph) -- all the reference's distances and
    witnesses bit for bit."""
    tz, tb = md.ring_pair_base(100, 50)
    bvh_a, bvh_b = md.build_f12(tz), md.build_f12(tb)
    recs = golden_meta["frames"]
    xfs = [md.ring_frame_transforms(rec["frame"]) for rec in recs]
    want = {q: np.array([[r[q]["distance"], r[q]["tri_a"], r[q]["tri_b"]] for r in recs]) for q in ("min", "max")}
    for q in ("min", "max"):
        for opts in ({"warm": True}, {"warm": True, "pipelined": False}, {}, {"graph": True}):
            got = md.run_sequence(tz, tb, bvh_a, bvh_b, xfs, q, **opts)
            np.testing.assert_array_equal(got, want[q], err_msg=f"{q} {opts}")
    both = md.run_sequence_minmax(tz, tb, bvh_a, bvh_b, xfs)
    for q in ("min", "max"):
        np.testing.assert_array_equal(both[q], want[q], err_msg=q)
    # a FrameGraph replayed frame by frame, then the plain API on the same trees
    a0, b0 = md.apply_transform(tz, xfs[0][0]), md.apply_transform(tb, xfs[0][1])
    fg = md.FrameGraph(a0, b0, bvh_a, bvh_b, ("max", "min"))
    for rec, (xa, xb) in zip(recs, xfs):
        a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
        out = fg.run(a, b)
        for q in ("min", "max"):
            assert (out[q].distance, out[q].witness.tri_a, out[q].witness.tri_b) == (
                rec[q]["distance"], rec[q]["tri_a"], rec[q]["tri_b"]), (rec["frame"], q)
        assert out["min"].witness.point_a.shape == (3,)
        # the trees now hold this frame's boxes: the plain query agrees
        r = md.run_min_query(a, b, bvh_a, bvh_b)
        assert r.distance == rec["min"]["distance"]
    fg.close()
    with pytest.raises(ValueError):
        md.FrameGraph(a0, b0, bvh_a, bvh_b, ("median",))
    # a chunked traversal (an arena far too small for the fronts): the graph's
    # record says `pending` and the remaining rounds run after the replay
    cfg = md.EngineConfig(arena_entries=1 << 11, front_hard_cap=1 << 30)
    fg = md.FrameGraph(a0, b0, bvh_a, bvh_b, ("min", "max"), cfg)
    for rec, (xa, xb) in list(zip(recs, xfs))[:3]:
        a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
        out = fg.run(a, b)
        for q in ("min", "max"):
            assert (out[q].distance, out[q].witness.tri_a, out[q].witness.tri_b) == (
                rec[q]["distance"], rec[q]["tri_a"], rec[q]["tri_b"]), (rec["frame"], q, "chunked")
    fg.close()


def test_brute_force_device(md, gpu, golden_meta):
    for rec in golden_meta["engine"][:10]:
        ma, mb = md.gen_scene(rec["kind"], rec["params"])
        for prec, dt in ((64, np.float64), (32, np.float32)):
            for q in ("min", "max"):
                g = rec[f"{q}{prec}"]
                d, w = (md.brute_force_min if q == "min" else md.brute_force_max)(ma, mb, dtype=dt)
                assert (d, w.tri_a, w.tri_b) == (g["brute_distance"], g["brute_tri_a"], g["brute_tri_b"])
    a, b = md.gen_scene("random-blobs", {"n": 4000})
    with pytest.raises(md.SizeGuardError):
        md.brute_force_min(a, b)


def test_variants_agree(md, gpu):
    """SPEC acceptance 5/9 analogues: culling off, enhanced bounds off, k = 1,
    warm start and guarantee_witness all give the same distance + witness."""
    for kind, params in [("random-blobs", {"n": 300, "seed": 4}), ("offset-grids", {"res": 14}),
                         ("nested-shells", {"lat": 12, "lon": 16, "r_outer": 0.85}),
                         ("intersecting-clusters", {"n": 400, "seed": 9})]:
        a, b = md.gen_scene(kind, params)
        ta, tb = md.build_f12(a), md.build_f12(b)
        for q in ("min", "max"):
            run = md.run_min_query if q == "min" else md.run_max_query
            base = run(a, b, ta, tb)
            for cfg in (md.EngineConfig(culling=False, front_hard_cap=1 << 26), md.EngineConfig(enhanced_bounds=False),
                        md.EngineConfig(depth_cap=1), md.EngineConfig(guarantee_witness=True)):
                r = run(a, b, ta, tb, cfg)
                assert r.distance == base.distance and (r.witness.tri_a, r.witness.tri_b) == (
                    base.witness.tri_a, base.witness.tri_b), (kind, q, cfg)
            warm = run(a, b, ta, tb, warm_pair=(base.witness.tri_a, base.witness.tri_b))
            assert warm.distance == base.distance
            assert warm.expanded_pairs <= base.expanded_pairs
        if kind == "intersecting-clusters":
            assert base.distance == 0.0 or q == "max"


def test_degenerate_depths(md, gpu, oracle):
    """depth-0 trees and mixed depths (query.py:368-377, 510-518)."""
    a1 = md.TriangleMesh([[0, 0, 0.0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    a3, _ = md.gen_scene("random-blobs", {"n": 3, "seed": 1})
    big, _ = md.gen_scene("interlocked-rings", {"nu": 60, "nv": 40})
    for ma, mb in ((a1, a1), (a1, big), (big, a1), (a3, big), (big, a3)):
        ta, tb = md.build_f12(ma), md.build_f12(mb)
        for q in ("min", "max"):
            r = (md.run_min_query if q == "min" else md.run_max_query)(ma, mb, ta, tb)
            d, ia, ib, _, _ = oracle.brute_force(ma.triangle_points(), mb.triangle_points(), q, force=True)
            assert r.distance == d and (r.witness.tri_a, r.witness.tri_b) == (ia, ib)


def test_errors(md, gpu):
    a, b = md.gen_scene("nested-shells", {"lat": 40, "lon": 40, "r_outer": 0.82})
    ta, tb = md.build_f12(a), md.build_f12(b)
    with pytest.raises(md.FrontOverflowError) as ei:
        md.run_max_query(a, b, ta, tb, md.EngineConfig(front_hard_cap=64))
    assert ei.value.cap == 64 and ei.value.candidates > 64
    with pytest.raises(md.ConfigError):
        md.run_min_query(a, b, ta, tb, md.EngineConfig(precision=32))
    # the workspace is healthy after an overflow
    assert md.run_min_query(a, b, ta, tb).distance > 0


def test_expand_front_step_api(md, gpu, oracle):
    """The single-step API reproduces the reference loop bit for bit."""
    a, b = md.gen_scene("random-blobs", {"n": 200, "seed": 2})
    ta, tb = md.build_f12(a), md.build_f12(b)
    cfg = md.EngineConfig()
    pa, pb = a.triangle_points(), b.triangle_points()
    r = md.batch_min_lower(ta.node_min[:1], ta.node_max[:1], tb.node_min[:1], tb.node_max[:1])[0]
    st = md.QueryState("min", md.batch_enhanced_min_upper(ta.node_min[:1], ta.node_max[:1], tb.node_min[:1],
                                                          tb.node_max[:1])[0])
    front = md.Front(np.zeros(1, np.int64), np.zeros(1, np.int64), np.asarray([r]), 0, 0)
    while len(front):
        k = md.adaptive_depth(len(front), cfg, max(ta.depth - front.depth_a, tb.depth - front.depth_b))
        front = md.expand_front(front, k, st, ta, tb, pa, pb, cfg)
    want = oracle.run_query(oracle.build_tree(a.vertices, a.triangles), oracle.build_tree(b.vertices, b.triangles),
                            pa, pb, "min")
    assert st.bound == want.distance
    assert [(s.k, s.front_in, s.front_out, s.culled, s.bound_after) for s in st.iterations] == [
        tuple(x) for x in want.iterations]


def test_dfs_comparator(md, gpu, golden_meta, oracle):
    """run_dfs_baseline (query.py:622-708): the per-triangle descent returns
    the reference's exact float64 distance and the brute-force witness, and
    counts its node examinations."""
    for rec in golden_meta["engine"][:12]:
        ma, mb = md.gen_scene(rec["kind"], rec["params"])
        tb = md.build_f12(mb)
        for q in ("min", "max"):
            g = rec[f"{q}64"]
            r = md.run_dfs_baseline(ma, mb, tb, q)
            assert r.distance == g["brute_distance"], (rec["kind"], q)
            assert (r.witness.tri_a, r.witness.tri_b) == (g["brute_tri_a"], g["brute_tri_b"])
            assert r.witness_exact and r.iterations == () and r.expanded_pairs == 0
            assert r.visited_nodes >= ma.n_triangles and r.narrow_pairs > 0
    # depth-0 trees, moved meshes, float32-built trees
    a1 = md.TriangleMesh([[0, 0, 0.0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    big, _ = md.gen_scene("interlocked-rings", {"nu": 60, "nv": 40})
    ring, other = md.gen_scene("interlocked-rings", {"nu": 30, "nv": 20})
    xf = md.RigidTransform.from_axis_angle((0.2, 1, 0.3), 0.7, (0.3, -0.1, 0.2))
    for ma, mb, dt in ((a1, a1, np.float64), (a1, big, np.float64), (big, a1, np.float64),
                       (md.apply_transform(ring, xf), other, np.float32)):
        tb = md.build_f12(mb, dtype=dt)
        for q in ("min", "max"):
            r = md.run_dfs_baseline(ma, mb, tb, q)
            d, ia, ib, _, _ = oracle.brute_force(ma.triangle_points(), mb.triangle_points(), q, force=True)
            assert r.distance == d and (r.witness.tri_a, r.witness.tri_b) == (ia, ib), (q, ma.n_triangles)
    with pytest.raises(ValueError):
        md.run_dfs_baseline(a1, a1, md.build_f12(a1), "mean")


def test_deformed_meshes(md, gpu, oracle):
    """Deformable refit: TriangleMesh.deformed with host
    arrays or a float64 CUDA tensor (used in place) refits the same tree and
    answers exactly like a mesh built from the same vertices."""
    import torch

    a, b = md.gen_scene("interlocked-rings", {"nu": 30, "nv": 20})
    ta, tb = md.build_f12(a), md.build_f12(b)
    md.run_min_query(a, b, ta, tb)
    rng = np.random.default_rng(3)
    for step in range(3):
        V = a.vertices + 0.01 * rng.normal(size=a.vertices.shape)
        for src in (V, torch.tensor(V, device="cuda")):
            d = a.deformed(src)
            assert d.n_vertices == a.n_vertices and d.triangles is a.triangles
            md.refit(ta, d)
            fresh = md.TriangleMesh(V, a.triangles)
            for q in ("min", "max"):
                r = (md.run_min_query if q == "min" else md.run_max_query)(d, b, ta, tb)
                dd, ia, ib, _, _ = oracle.brute_force(fresh.triangle_points(), b.triangle_points(), q, force=True)
                assert r.distance == dd and (r.witness.tri_a, r.witness.tri_b) == (ia, ib), (step, q)
            assert np.array_equal(d.vertices, V)
    # transformed deformed mesh, boxes equal the reference's on the moved vertices
    xf = md.RigidTransform.from_axis_angle((0, 1, 1), 0.4, (0.1, 0.2, 0.3))
    moved = md.apply_transform(a.deformed(torch.tensor(V, device="cuda")), xf)
    md.refit(ta, moved)
    ref = oracle.Tree(np.empty((ta.n_nodes, 3)), np.empty((ta.n_nodes, 3)), ta.leaf_tris, ta.prim_order, ta.depth)
    oracle.fill_boxes(ref, moved.vertices, moved.triangles)
    assert np.array_equal(ta.node_min, ref.node_min) and np.array_equal(ta.node_max, ref.node_max)
    with pytest.raises(ValueError):
        a.deformed(torch.zeros((3, 3), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        a.deformed(np.zeros((a.n_vertices + 1, 3)))


@pytest.mark.parametrize("prec", [64, 32])
def test_nonfinite_vertices(md, gpu, oracle, prec):
    """Non-finite coordinates behave as in the reference (its np.minimum /
    np.maximum boxes propagate NaN to the root; `key < nan` culls every
    candidate): a NaN vertex gives distance NaN, no witness, one iteration
    that culls the root's whole expansion; +-inf coordinates give the
    brute-force minimum and an infinite maximum without a witness (the
    reference's values on this scene, checked here in CPU tests' terms)."""
    import warnings

    warnings.simplefilter("ignore")
    dt = np.float64 if prec == 64 else np.float32
    cfg = md.EngineConfig(precision=prec)
    a, b = md.gen_scene("random-blobs", {"n": 50, "seed": 1})
    for side in ("a", "b"):
        V = (a if side == "a" else b).vertices.copy()
        V[5] = np.nan
        bad = md.TriangleMesh(V, (a if side == "a" else b).triangles)
        ma, mb = (bad, b) if side == "a" else (a, bad)
        ta, tb = md.build_f12(ma, dtype=dt), md.build_f12(mb, dtype=dt)
        assert np.isnan((ta if side == "a" else tb).node_min[0]).all()
        for run in (md.run_min_query, md.run_max_query):
            r = run(ma, mb, ta, tb, cfg)
            assert np.isnan(r.distance) and r.witness is None, (side, run.__name__)
            assert len(r.iterations) == 1 and r.iterations[0].front_out == 0
            assert r.iterations[0].culled == 4 ** r.iterations[0].k == r.expanded_pairs and r.narrow_pairs == 0
    for val in (np.inf, -np.inf):
        V = a.vertices.copy()
        V[5, 1] = val
        a2 = md.TriangleMesh(V, a.triangles)
        ta, tb = md.build_f12(a2, dtype=dt), md.build_f12(b, dtype=dt)
        r = md.run_min_query(a2, b, ta, tb, cfg)
        d, ia, ib, _, _ = oracle.brute_force(a2.triangle_points(dt), b.triangle_points(dt), "min")
        assert r.distance == d and (r.witness.tri_a, r.witness.tri_b) == (ia, ib)
        r = md.run_max_query(a2, b, ta, tb, cfg)
        assert r.distance == np.inf and r.witness is None


@pytest.mark.parametrize("scene", ["interlocked-rings", "nested-shells"])
def test_query_group_matches_separate(md, gpu, scene):
    """launch_group (gd_query_group_async: the min and max traversals back to
    back, then both narrow / exact chains side by side on forked streams)
    gives each query's separate answer -- distance, witness, points --
    including when the group is replayed with the other order
    and when one plan appears alone."""
    params = {"nu": 60, "nv": 30} if scene == "interlocked-rings" else {}
    a, b = md.gen_scene(scene, params)
    xa = md.RigidTransform.from_axis_angle([0.3, 1.0, 0.2], 0.7, [0.05, -0.02, 0.01])
    a = md.apply_transform(a, xa)
    ta, tb = md.build_f12(a), md.build_f12(b)
    cfg = md.EngineConfig(front_hard_cap=1 << 30)
    want = {k: (md.run_min_query if k == "min" else md.run_max_query)(a, b, ta, tb, cfg) for k in ("min", "max")}
    plans = {k: md.PreparedQuery(a, b, ta, tb, cfg, k, private_workspace=True) for k in ("min", "max")}
    for order in (("min", "max"), ("max", "min"), ("min",), ("max",)):
        md.launch_group([plans[k] for k in order])
        for k in order:
            got = plans[k].collect()
            w = want[k]
            assert got.distance == w.distance, (order, k)
            assert (got.witness.tri_a, got.witness.tri_b) == (w.witness.tri_a, w.witness.tri_b), (order, k)
            np.testing.assert_array_equal(got.witness.point_a, w.witness.point_a)
            np.testing.assert_array_equal(got.witness.point_b, w.witness.point_b)
            assert got.iterations and got.iterations[-1].front_out == 0, (order, k)
    with pytest.raises(ValueError, match="share"):
        other = md.PreparedQuery(b, a, tb, ta, cfg, "min", private_workspace=True)
        md.launch_group([plans["min"], other])


@pytest.mark.parametrize("lat_lon, long_list", [((16, 20), False), ((260, 300), True)])
def test_narrow_paths_short_and_long_lists(md, gpu, lat_lon, long_list):
    """Min queries evaluate a short candidate list (<= 2^18 triangle pairs)
    exactly right away and a long one through the float32 band
    (narrow.cuh direct_exact); nested shells are near contact everywhere, so
    both sizes are reached -- both equal the device brute force (distance and
    lexicographic witness), in float64 and float32."""
    lat, lon = lat_lon
    a, b = md.gen_scene("nested-shells", {"lat": lat, "lon": lon, "r_inner": 0.8, "r_outer": 0.81})
    for prec in (64, 32):
        dt = np.float64 if prec == 64 else np.float32
        ta, tb = md.build_f12(a, dtype=dt), md.build_f12(b, dtype=dt)
        r = md.run_min_query(a, b, ta, tb, md.EngineConfig(precision=prec, front_hard_cap=1 << 30))
        assert (r.narrow_pairs > 1 << 18) == long_list, r.narrow_pairs
        d, w = md.brute_force_min(a, b, force=True, dtype=dt)
        assert r.distance == d and (r.witness.tri_a, r.witness.tri_b) == (w.tri_a, w.tri_b), prec


def test_min_rescan_after_band_overflow_long_list(md, gpu):
    """A long candidate list (> 2^18, the float32 stage runs) with a 2-entry
    band: the band overflows, the record says pending bit 1, and the rescan
    pass (host-driven through gd_query_round) still returns the brute-force
    answer."""
    from paper_2411_11244_b200 import query as Q

    a, b = md.gen_scene("nested-shells", {"lat": 260, "lon": 300, "r_inner": 0.8, "r_outer": 0.81})
    ta, tb = md.build_f12(a), md.build_f12(b)
    pq = Q.PreparedQuery(a, b, ta, tb, md.EngineConfig(front_hard_cap=1 << 30), "min")
    pq.g_cfg.band_cap = 2
    pq.launch()
    r = pq.collect()  # collect sees pending bit 1 and runs the rescan itself
    assert r.narrow_pairs > 1 << 18
    d, w = md.brute_force_min(a, b, force=True)
    assert r.distance == d and (r.witness.tri_a, r.witness.tri_b) == (w.tri_a, w.tri_b)
