"""Exactness corner cases of the float32 traversal + reference-arithmetic
exact pass, each checked against the CPU oracle's
brute force (the reference's own arithmetic, query.py:571-619):

* meshes authored far from the origin and moved back by their transform
  (the float32 transform's rounding scales with the base coordinates);
* transforms applied to already-moved meshes (the reference applies them one
  by one);
* traversal in B's local frame at precision 32 with the scene far from the
  world origin (the exact pass rounds at world-coordinate scale);
* several host threads querying at once (per-thread workspaces).
"""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _brute(oracle, a, b, kind, prec=64):
    dt = np.float64 if prec == 64 else np.float32
    d, ia, ib, _, _ = oracle.brute_force(a.triangle_points(dt), b.triangle_points(dt), kind, force=True)
    return d, (ia, ib)


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("offset", [1e3, 1e4])
def test_far_base_cancelled_by_transform(md, gpu, oracle, offset, prec):
    """Base vertices ~offset from the origin, the transform brings the pair
    back to unit scale: the slack must follow the float32 transform's
    rounding (|R||v| + |t|), not the small world coordinates."""
    a0, b0 = md.gen_scene("interlocked-rings", {"nu": 40, "nv": 20})
    shift = np.array([offset, -0.7 * offset, 0.4 * offset])
    a_far = md.TriangleMesh(a0.vertices + shift, a0.triangles)
    b_far = md.TriangleMesh(b0.vertices - 0.5 * shift, b0.triangles)
    ra = md.RigidTransform.from_axis_angle((0.3, 1.0, 0.2), 0.7)
    rb = md.RigidTransform.from_axis_angle((1.0, -0.2, 0.5), -0.4)
    xa = md.RigidTransform(ra.rotation, -ra.rotation @ shift)
    xb = md.RigidTransform(rb.rotation, rb.rotation @ (0.5 * shift) + np.array([0.02, 0.01, -0.03]))
    dt = np.float64 if prec == 64 else np.float32
    ta, tb = md.build_f12(a_far, dtype=dt), md.build_f12(b_far, dtype=dt)
    a, b = md.apply_transform(a_far, xa), md.apply_transform(b_far, xb)
    md.refit(ta, a)
    md.refit(tb, b)
    cfg = md.EngineConfig(precision=prec)
    for kind in ("min", "max"):
        got = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb, cfg)
        d, w = _brute(oracle, a, b, kind, prec)
        assert got.distance == d, (kind, got.distance, d)
        assert (got.witness.tri_a, got.witness.tri_b) == w, kind


def test_chained_transforms_bitwise(md, gpu, oracle):
    """apply_transform of a moved mesh: the device answer is the reference's
    on its transform-by-transform vertices, bit for bit."""
    a0, b0 = md.gen_scene("interlocked-rings", {"nu": 40, "nv": 20})
    ta, tb = md.build_f12(a0), md.build_f12(b0)
    a = a0
    for i in range(4):  # incremental per-frame transforms (animation pattern)
        a = md.apply_transform(a, md.RigidTransform.from_axis_angle((1.0, 0.3 * i, 0.1), 0.05, (0.003, -0.002, 0.001)))
    md.refit(ta, a)
    md.refit(tb, b0)
    for kind in ("min", "max"):
        got = (md.run_min_query if kind == "min" else md.run_max_query)(a, b0, ta, tb)
        d, w = _brute(oracle, a, b0, kind)
        assert got.distance == d and (got.witness.tri_a, got.witness.tri_b) == w, kind
    # the refit boxes are the reference's boxes of those vertices (fill_boxes
    # on the same topology, bvh.py:242-264)
    n = ta.n_nodes
    ref = oracle.Tree(np.empty((n, 3)), np.empty((n, 3)), np.asarray(ta.leaf_tris), np.asarray(ta.prim_order),
                      ta.depth)
    oracle.fill_boxes(ref, a.vertices, a.triangles)
    np.testing.assert_array_equal(ta.node_min, ref.node_min)
    np.testing.assert_array_equal(ta.node_max, ref.node_max)


def test_blocal_precision32_far_from_world_origin(md, gpu, oracle):
    """frame='b-local' at precision 32 with the pair 1e3 away from the world
    origin: same answer as the world frame and the brute force."""
    from paper_2411_11244_b200 import query as Q

    a0, b0 = md.gen_scene("interlocked-rings", {"nu": 40, "nv": 20})
    xa = md.RigidTransform.from_axis_angle((0.2, 0.9, 0.1), 0.3, (1000.0, 800.0, -600.0))
    xb = md.RigidTransform.from_axis_angle((1.0, 0.1, -0.4), -0.2, (1000.05, 800.02, -599.97))
    ta, tb = md.build_f12(a0, dtype=np.float32), md.build_f12(b0, dtype=np.float32)
    a, b = md.apply_transform(a0, xa), md.apply_transform(b0, xb)
    cfg = md.EngineConfig(precision=32)
    for kind in ("min", "max"):
        d, w = _brute(oracle, a, b, kind, 32)
        for frame in ("world", "b-local"):
            got = Q.PreparedQuery(a, b, ta, tb, cfg, kind, frame=frame).run()
            assert got.distance == d and (got.witness.tri_a, got.witness.tri_b) == w, (kind, frame)


def test_concurrent_host_threads(md, gpu):
    """Queries from several host threads at once use per-thread workspaces:
    every thread gets its own scene's answer."""
    scenes = []
    for seed in range(4):
        a, b = md.gen_scene("random-blobs", {"n": 300, "seed": seed, "gap": 0.05})
        ta, tb = md.build_f12(a), md.build_f12(b)
        want = {k: (md.run_min_query if k == "min" else md.run_max_query)(a, b, ta, tb) for k in ("min", "max")}
        scenes.append((a, b, ta, tb, want))
    errors = []

    def work(i):
        import torch

        torch.cuda.set_device(0)
        a, b, ta, tb, want = scenes[i]
        try:
            for rep in range(20):
                for k in ("min", "max"):
                    r = (md.run_min_query if k == "min" else md.run_max_query)(a, b, ta, tb)
                    if r.distance != want[k].distance or r.witness.tri_a != want[k].witness.tri_a:
                        errors.append((i, rep, k, r.distance, want[k].distance))
        except Exception as exc:  # report, never hide
            errors.append((i, repr(exc)))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(scenes))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:5]


def test_concurrent_query_groups(md, gpu):
    """Query groups (gd_query_group_async: forked narrow chains) launched from
    several host threads at once on their own streams: each thread's fork /
    join events are its own, every group returns its scene's answers."""
    import torch

    scenes = []
    for seed in range(4):
        a, b = md.gen_scene("random-blobs", {"n": 300, "seed": 10 + seed, "gap": 0.05})
        ta, tb = md.build_f12(a), md.build_f12(b)
        want = {k: (md.run_min_query if k == "min" else md.run_max_query)(a, b, ta, tb) for k in ("min", "max")}
        scenes.append((a, b, ta, tb, want))
    errors = []

    def work(i):
        torch.cuda.set_device(0)
        a, b, ta, tb, want = scenes[i]
        try:
            plans = [md.PreparedQuery(a, b, ta, tb, md.EngineConfig(), k, private_workspace=True)
                     for k in ("min", "max")]
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                for rep in range(20):
                    md.launch_group(plans)
                    for k, p in zip(("min", "max"), plans):
                        r = p.collect()
                        if r.distance != want[k].distance or r.witness.tri_a != want[k].witness.tri_a:
                            errors.append((i, rep, k, r.distance, want[k].distance))
        except Exception as exc:  # report, never hide
            errors.append((i, repr(exc)))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(scenes))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:5]
