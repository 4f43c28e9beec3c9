"""Randomised exactness sweep on the GPU: the engine against the device brute
force (the reference's all-pairs rule, query.py:571-619) on scenes of varied
size, scale, offset and shape -- distances and witnesses identical, min and
max, both precisions.  Exercises the float32 slack argument (DESIGN.md
"Exactness") far from the golden scenes: coordinates up to 1e5, tiny and
sliver triangles, touching / interpenetrating soups, near-duplicates."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scene(md, rng, case):
    kind = case % 5
    n = int(rng.integers(5, 700))
    scale = float(10.0 ** rng.uniform(-3, 5))
    off = rng.normal(size=3) * scale * float(rng.choice([0.0, 1.0, 100.0]))
    if kind == 0:    # two gaussian soups with a gap
        a = rng.normal(size=(n, 1, 3)) + 0.05 * rng.normal(size=(n, 3, 3))
        b = rng.normal(size=(n, 1, 3)) + 0.05 * rng.normal(size=(n, 3, 3)) + [3.0, 0, 0]
    elif kind == 1:  # interpenetrating soups (distance 0 likely)
        a = rng.normal(size=(n, 1, 3)) + 0.2 * rng.normal(size=(n, 3, 3))
        b = rng.normal(size=(n, 1, 3)) + 0.2 * rng.normal(size=(n, 3, 3))
    elif kind == 2:  # slivers and tiny triangles
        base = rng.normal(size=(n, 1, 3))
        d = rng.normal(size=(n, 1, 3))
        a = np.concatenate([base, base + d, base + d * (1 + 1e-6) + 1e-7 * rng.normal(size=(n, 1, 3))], axis=1)
        b = rng.normal(size=(n, 1, 3)) * 0.5 + 1e-3 * rng.normal(size=(n, 3, 3)) + [0, 2.0, 0]
    elif kind == 3:  # near-duplicate copy shifted by a hair
        a = rng.normal(size=(n, 1, 3)) + 0.1 * rng.normal(size=(n, 3, 3))
        b = a + 1e-4 * rng.normal(size=(1, 1, 3))
    else:            # planar grids facing each other (many ties)
        g = int(np.sqrt(n)) + 2
        xs, ys = np.meshgrid(np.arange(g, dtype=float), np.arange(g, dtype=float))
        quads = np.stack([xs[:-1, :-1], ys[:-1, :-1]], -1).reshape(-1, 2)
        tri = []
        for x, y in quads:
            tri.append([[x, y, 0], [x + 1, y, 0], [x + 1, y + 1, 0]])
            tri.append([[x, y, 0], [x + 1, y + 1, 0], [x, y + 1, 0]])
        a = np.asarray(tri)
        b = a + [0.25, 0.5, 0.75]
    a = a * scale + off
    b = b * scale + off
    mk = lambda p: md.TriangleMesh(p.reshape(-1, 3), np.arange(p.shape[0] * 3).reshape(-1, 3))  # noqa: E731
    return mk(a), mk(b)


@pytest.mark.parametrize("block", range(4))
def test_engine_matches_brute_force(md, gpu, block):
    rng = np.random.default_rng(9000 + block)
    for case in range(block * 100, block * 100 + 100):
        a, b = _scene(md, rng, case)
        for prec in (64, 32):
            dt = np.float64 if prec == 64 else np.float32
            ta, tb = md.build_f12(a, dtype=dt), md.build_f12(b, dtype=dt)
            cfg = md.EngineConfig(precision=prec, front_hard_cap=1 << 26)
            for kind in ("min", "max"):
                r = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb, cfg)
                d, w = (md.brute_force_min if kind == "min" else md.brute_force_max)(a, b, force=True, dtype=dt)
                assert r.distance == d, (case, prec, kind, r.distance, d)
                assert (r.witness.tri_a, r.witness.tri_b) == (w.tri_a, w.tri_b), (case, prec, kind)


def test_moved_meshes_and_dfs(md, gpu):
    """Rigidly moved ring pairs (the lazy device transform against numpy's
    dgemm vertices of the brute force) and the DFS comparator."""
    rng = np.random.default_rng(77)
    for case in range(40):
        nu, nv = int(rng.integers(8, 40)), int(rng.integers(6, 20))
        tz, tb = md.ring_pair_base(nu, nv)
        axis = rng.normal(size=3)
        xa = md.RigidTransform.from_axis_angle(axis, float(rng.uniform(0, 6.3)), rng.normal(size=3) * 0.3)
        xb = md.RigidTransform.from_axis_angle(rng.normal(size=3), float(rng.uniform(0, 6.3)), rng.normal(size=3) * 0.3)
        a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
        ta, tbt = md.build_f12(tz), md.build_f12(tb)
        md.refit(ta, a)
        md.refit(tbt, b)
        for kind in ("min", "max"):
            r = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tbt)
            d, w = (md.brute_force_min if kind == "min" else md.brute_force_max)(a, b, force=True)
            assert r.distance == d and (r.witness.tri_a, r.witness.tri_b) == (w.tri_a, w.tri_b), (case, kind)
            if case % 4 == 0:
                rd = md.run_dfs_baseline(a, b, tbt, kind)
                assert rd.distance == d and (rd.witness.tri_a, rd.witness.tri_b) == (w.tri_a, w.tri_b), (case, kind)
