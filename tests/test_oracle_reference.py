"""The oracle restatement against the LIVE reference package (CPU only).

Runs wherever the reference is importable: `/root/reference/pkg/src` in the build
container, or the unmodified copy installed into `baseline/_ref` (git-ignored,
shipped to the GPU box by gpurun).  Skips otherwise -- the committed golden vectors
(test_oracle_golden.py) pin the oracle on every machine.  Fresh seeded inputs here,
so the oracle is checked beyond the goldens it was written against.
"""

import numpy as np
import pytest


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    bad = ~((a == b) | (np.isnan(a) & np.isnan(b)))
    assert not bad.any(), f"{bad.sum()} mismatches, first at {np.argwhere(bad)[:3].tolist()}"


def _tris(rng, n, scale=1.0):
    base = rng.normal(size=(n, 1, 3))
    return base + scale * rng.normal(size=(n, 3, 3)) * rng.uniform(0.01, 1.0, size=(n, 1, 1))


@pytest.mark.parametrize("prec", [64, 32])
def test_tri_tri_random(reference, oracle, prec):
    """bounds.py:245-330 vs oracle.tri_tri_min/max on fresh random pairs,
    including exact copies (distance 0) and shared vertices."""
    from importlib import import_module

    rb = import_module(reference.__name__ + ".bounds")
    rng = np.random.default_rng(1234 + prec)
    dt = np.float64 if prec == 64 else np.float32
    t1 = _tris(rng, 3000).astype(dt)
    t2 = _tris(rng, 3000).astype(dt) * 0.3 + t1 * 0.7
    t2[:100] = t1[:100]                       # identical triangles
    t2[100:200, 0] = t1[100:200, 1]           # shared vertex
    for fr, fo in ((rb.batch_tri_tri_min, oracle.tri_tri_min), (rb.batch_tri_tri_max, oracle.tri_tri_max)):
        dr, pr, qr = fr(t1, t2)
        do, po, qo = fo(t1, t2)
        _eq(do, dr)
        _eq(po, pr)
        _eq(qo, qr)


def test_box_bounds_random(reference, oracle):
    """bounds.py:47-101 (Eqs. 5-10) vs the oracle, f64 and f32."""
    from importlib import import_module

    rb = import_module(reference.__name__ + ".bounds")
    rng = np.random.default_rng(77)
    for dt in (np.float64, np.float32):
        c = rng.normal(size=(4, 5000, 3))
        amin = (c[0] - np.abs(c[1])).astype(dt)
        amax = (c[0] + np.abs(c[1])).astype(dt)
        bmin = (c[2] - np.abs(c[3])).astype(dt)
        bmax = (c[2] + np.abs(c[3])).astype(dt)
        for name, fo in (("batch_min_lower", oracle.box_min_lower), ("batch_max_upper", oracle.box_max_upper),
                         ("batch_enhanced_min_upper", oracle.enhanced_min_upper),
                         ("batch_enhanced_max_lower", oracle.enhanced_max_lower)):
            _eq(fo(amin, amax, bmin, bmax), getattr(rb, name)(amin, amax, bmin, bmax))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 300, 1000, 2049])
def test_build_random_soup(reference, oracle, n):
    """build_f12 (bvh.py:267-289) vs oracle.build_tree: prim_order, leaf_tris
    and every node box, both dtypes (exercises the pairing deferrals)."""
    rng = np.random.default_rng(n)
    V = np.round(rng.normal(size=(3 * n, 3)), 2)  # rounded: surface-area ties
    T = np.arange(3 * n).reshape(n, 3)
    mesh = reference.TriangleMesh(V, T)
    for dt in (np.float64, np.float32):
        r = reference.build_f12(mesh, dtype=dt)
        o = oracle.build_tree(V, T, dtype=dt)
        _eq(o.prim_order, r.prim_order)
        _eq(o.leaf_tris, r.leaf_tris)
        _eq(o.node_min, r.node_min)
        _eq(o.node_max, r.node_max)
        assert o.depth == r.depth


@pytest.mark.parametrize("kind", ["min", "max"])
@pytest.mark.parametrize("prec", [64, 32])
def test_engine_small_tori(reference, oracle, md, kind, prec):
    """run_min_query / run_max_query (query.py:540-568) vs oracle.run_query on a
    small interlocked-rings scene at a rotation-sequence frame: distance,
    witness and every IterationStat."""
    tz, tb = md.ring_pair_base(30, 20)
    xa, xb = md.ring_frame_transforms(137)
    A = reference.TriangleMesh(tz.vertices, tz.triangles)
    B = reference.TriangleMesh(tb.vertices, tb.triangles)
    A = reference.apply_transform(A, reference.RigidTransform(xa.rotation, xa.translation))
    B = reference.apply_transform(B, reference.RigidTransform(xb.rotation, xb.translation))
    dt = np.float64 if prec == 64 else np.float32
    ra, rbv = reference.build_f12(A, dtype=dt), reference.build_f12(B, dtype=dt)
    cfg = reference.EngineConfig(precision=prec)
    run = reference.run_min_query if kind == "min" else reference.run_max_query
    want = run(A, B, ra, rbv, cfg)
    oa = oracle.build_tree(A.vertices, A.triangles, dtype=dt)
    ob = oracle.build_tree(B.vertices, B.triangles, dtype=dt)
    got = oracle.run_query(oa, ob, oracle.triangle_points(A.vertices, A.triangles, dt),
                           oracle.triangle_points(B.vertices, B.triangles, dt), kind, oracle.Config(precision=prec))
    assert got.distance == want.distance
    assert (got.tri_a, got.tri_b) == (want.witness.tri_a, want.witness.tri_b)
    assert [tuple(s[:4]) for s in got.iterations] == [(s.k, s.front_in, s.front_out, s.culled)
                                                      for s in want.iterations]
    assert got.expanded_pairs == want.expanded_pairs and got.narrow_pairs == want.narrow_pairs


OBJ_CASES = [
    "# comment\nv 0 0 0\nv 1 0 0 # trailing\nv 1 1 0\nv 0 1 0\nvn 0 0 1\nvt 0 0\nf 1/1/1 2/2/1 3//1 4\nf -4 -3 -2\n",
    "v 1e-3 .5 5.\r\nv +1_0.5 -0 2E+2\r\nv inf 0 -NaN\r\nv 0 0 1\rf 1 2 3\r\ng grp\no obj\ns off\nf 2 3 4 1\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n\n\n   \n\tf -1 -2 -3\nusemtl x\nf 0003 +2 1_0\n",
    "v 0 0\n",
    "v 0 0 zero\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 0\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 4\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 -4\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 x/1\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 /3\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 99999999999999999999999\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 1 2\n",
    "v 0 0 0\nv 1 0 0\rv 0 1 0\r\nf 1 2 3 'q\n",
    "",
]


@pytest.mark.parametrize("case", range(len(OBJ_CASES)))
def test_load_obj_matches_reference(reference, md, tmp_path, case):
    """The native OBJ parser (csrc/obj.cpp) against the reference's load_obj
    (mesh.py:112-163): same arrays, or the same exception type, line and
    message."""
    p = tmp_path / f"c{case}.obj"
    p.write_bytes(OBJ_CASES[case].encode())
    try:
        want = reference.load_obj(p)
    except Exception as exc:  # noqa: BLE001 - compare the failure itself
        with pytest.raises(Exception) as got:
            md.load_obj(p)
        assert type(got.value).__name__ == type(exc).__name__
        assert str(got.value) == str(exc)
        assert getattr(got.value, "line_no", None) == getattr(exc, "line_no", None)
        return
    got = md.load_obj(p)
    assert np.array_equal(got.vertices, want.vertices, equal_nan=True)
    assert np.array_equal(got.triangles, want.triangles)


def test_load_obj_large_matches_reference(reference, md, tmp_path):
    """A 20K-triangle OBJ written from a torus: identical arrays."""
    tz, _ = md.ring_pair_base(100, 100)
    p = tmp_path / "torus.obj"
    with open(p, "w") as fh:
        for v in tz.vertices:
            fh.write(f"v {float(v[0])!r} {float(v[1])!r} {float(v[2])!r}\n")
        for t in tz.triangles:
            fh.write(f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}\n")
    got, want = md.load_obj(p), reference.load_obj(p)
    assert np.array_equal(got.vertices, want.vertices) and np.array_equal(got.triangles, want.triangles)


def test_reference_nonfinite_semantics(reference):
    """Pins the behaviour tests/test_gpu_parity.py::test_nonfinite_vertices
    asserts for the device engine: a NaN vertex makes the reference's root box
    NaN (np.minimum), every candidate is culled and the distance is NaN with
    no witness after one iteration; +-inf gives a finite minimum and an
    infinite, witness-less maximum."""
    import warnings

    warnings.simplefilter("ignore")
    a, b = reference.gen_scene("random-blobs", {"n": 50, "seed": 1})
    V = a.vertices.copy()
    V[5] = np.nan
    a2 = reference.TriangleMesh(V, a.triangles)
    ta, tb = reference.build_f12(a2), reference.build_f12(b)
    assert np.isnan(ta.node_min[0]).all()
    for run in (reference.run_min_query, reference.run_max_query):
        r = run(a2, b, ta, tb)
        assert np.isnan(r.distance) and r.witness is None and len(r.iterations) == 1
        s = r.iterations[0]
        assert s.front_out == 0 and s.culled == 4 ** s.k == r.expanded_pairs and r.narrow_pairs == 0
    V = a.vertices.copy()
    V[5, 1] = np.inf
    a3 = reference.TriangleMesh(V, a.triangles)
    ta = reference.build_f12(a3)
    rmin = reference.run_min_query(a3, b, ta, tb)
    assert rmin.distance == reference.brute_force_min(a3, b)[0] and rmin.witness is not None
    rmax = reference.run_max_query(a3, b, ta, tb)
    assert rmax.distance == np.inf and rmax.witness is None
