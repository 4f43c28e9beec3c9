"""Parity against the second golden set (tests/golden/make_golden_r2.py, made
by the reference itself): the config-4 geometry (nested shells r 0.8 / 0.81,
the near-contact stress case) at up to 29K triangles per mesh, rings at 50K
triangles over three rotation frames, and the pairing topology of 60K / 120K
triangle tori.

Witness rule: the device returns the lexicographically
smallest (tri_a, tri_b) attaining the exact distance -- the brute-force
witness (query.py:589-597).  The reference returns the smallest among the
pairs IT evaluated, so the two agree except on exact ties its strict culling
skipped (query.py:16-24).  A differing witness is accepted only as a
documented tie: the reference arithmetic on the device's pair gives exactly
the reference's distance, and the device's pair is lexicographically smaller.
"""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def g2():
    with open(GOLDEN / "golden_r2.json") as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def g2arr():
    return np.load(GOLDEN / "golden_r2.npz")


def _sha(mesh):
    import hashlib

    h = hashlib.sha256()
    h.update(np.ascontiguousarray(mesh.vertices, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(mesh.triangles, dtype=np.int64).tobytes())
    return h.hexdigest()


def _classify(md, a, b, kind, prec, got, want):
    """'equal' or 'tie' (asserts it is a documented tie)."""
    pair = (got.witness.tri_a, got.witness.tri_b)
    ref_pair = (want["tri_a"], want["tri_b"])
    if pair == ref_pair:
        np.testing.assert_array_equal(got.witness.point_a, want["point_a"])
        np.testing.assert_array_equal(got.witness.point_b, want["point_b"])
        return "equal"
    dt = np.float64 if prec == 64 else np.float32
    pa = a.triangle_points(dt)[[pair[0]]]
    pb = b.triangle_points(dt)[[pair[1]]]
    d = (md.batch_tri_tri_min if kind == "min" else md.batch_tri_tri_max)(pa, pb)[0][0]
    assert float(d) == want["distance"], (kind, prec, pair, float(d), want["distance"])
    assert pair < ref_pair, (pair, ref_pair)
    return "tie"


@pytest.mark.parametrize("prec", [64, 32])
def test_nested_shells_config4_geometry(md, gpu, g2, prec):
    dt = np.float64 if prec == 64 else np.float32
    ties = {}
    for rec in g2["shells"]:
        a, b = md.gen_scene("nested-shells", rec["params"])
        assert (_sha(a), _sha(b)) == (rec["hash_a"], rec["hash_b"])
        ta, tb = md.build_f12(a, dtype=dt), md.build_f12(b, dtype=dt)
        cfg = md.EngineConfig(precision=prec, front_hard_cap=1 << 40)
        for kind in ("min", "max"):
            want = rec[f"{kind}{prec}"]
            got = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb, cfg)
            assert want["witness_exact"]
            assert got.distance == want["distance"], (rec["params"], kind, got.distance, want["distance"])
            assert got.witness_exact
            ties[(rec["tris"], kind)] = _classify(md, a, b, kind, prec, got, want)
    print("nested shells witness classification:", ties)


def test_rings_50k_frames(md, gpu, g2):
    from paper_2411_11244_b200 import scenes

    tz, tbase = scenes.ring_pair_base(250, 100)
    ta, tb = md.build_f12(tz), md.build_f12(tbase)
    for rec in g2["rings50k"]:
        xa, xb = scenes.ring_frame_transforms(rec["frame"])
        a, b = md.apply_transform(tz, xa), md.apply_transform(tbase, xb)
        assert (_sha(a), _sha(b)) == (rec["hash_a"], rec["hash_b"])
        md.refit(ta, a)
        md.refit(tb, b)
        for kind in ("min", "max"):
            got = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb)
            assert got.distance == rec[kind]["distance"], (rec["frame"], kind)
            _classify(md, a, b, kind, 64, got, rec[kind])


def test_pairing_topology_large_tori(md, gpu, g2, g2arr):
    from paper_2411_11244_b200 import scenes

    for rec in g2["pairings"]:
        t, _ = scenes.ring_pair_base(rec["nu"], rec["nv"])
        tree = md.build_f12(t)
        np.testing.assert_array_equal(tree.prim_order, g2arr[f"pair_{rec['name']}_order"])
        np.testing.assert_array_equal(tree.leaf_tris, g2arr[f"pair_{rec['name']}_leaf"])
