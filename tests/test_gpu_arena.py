"""Front arena: the traversal's level stack in an
arena sized independently of front_hard_cap, chunked depth-first expansion
when a level does not fit, and the reference's iteration statistics and
FrontOverflowError semantics on top of it."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scene(md, name):
    if name == "rings":
        a, b = md.ring_pair_base(250, 100)  # 50K triangles each
        xa, xb = md.ring_frame_transforms(11)
        return md.apply_transform(a, xa), md.apply_transform(b, xb)
    if name == "shells":
        return md.gen_scene("nested-shells", {"lat": 40, "lon": 48, "r_inner": 0.8, "r_outer": 0.81})
    return md.gen_scene(name, {"n": 400, "seed": 3})


def _trees(md, a, b):
    return md.build_f12(a), md.build_f12(b)


def _device_k(md, n, cfg, rem_a, rem_b, threshold):
    """The device schedule (GdConfig.schedule >= 0): the reference rule, but
    k = 2 where it gives 1 for fronts up to the threshold with >= 2 levels
    left on each tree (traverse.cu plan_sweep)."""
    k = md.adaptive_depth(n, cfg, max(rem_a, rem_b))
    if (k == 1 and cfg.depth_cap >= 2 and min(rem_a, rem_b) >= 2 and n <= threshold
            and 16 * n <= cfg.front_hard_cap):
        k = 2
    return k


@pytest.mark.parametrize("kind", ["min", "max"])
@pytest.mark.parametrize("scene", ["rings", "shells"])
@pytest.mark.parametrize("schedule", [-1, 0, 1 << 14])
def test_iteration_stats_follow_schedule(md, gpu, kind, scene, schedule):
    """schedule -1: k of every iteration is the reference's adaptive_depth of
    its front (query.py:266-284); >= 0: the device schedule's.  Fronts chain
    (front_out[i] == front_in[i+1]); every candidate is either culled or
    survives (the last iteration's survivors are the leaf pairs, not a front:
    front_out 0); the bound is monotone; the answer does not depend on the
    schedule."""
    a, b = _scene(md, scene)
    ta, tb = _trees(md, a, b)
    cfg = md.EngineConfig(front_hard_cap=1 << 30, device_schedule=schedule)
    run = md.run_min_query if kind == "min" else md.run_max_query
    r = run(a, b, ta, tb, cfg)
    ref = run(a, b, ta, tb, md.EngineConfig(front_hard_cap=1 << 30, device_schedule=-1))
    assert r.distance == ref.distance
    assert (r.witness.tri_a, r.witness.tri_b) == (ref.witness.tri_a, ref.witness.tri_b)
    threshold = {-1: 0, 0: 1 << 17}.get(schedule, schedule)
    its = r.iterations
    assert its and its[-1].front_out == 0
    da = db = 0
    total = 0
    for i, s in enumerate(its):
        rem_a, rem_b = ta.depth - da, tb.depth - db
        assert s.k == _device_k(md, s.front_in, cfg, rem_a, rem_b, threshold), (i, s)
        ka, kb = min(s.k, rem_a), min(s.k, rem_b)
        cand = s.front_in << (ka + kb)
        total += cand
        if i + 1 < len(its):
            assert s.front_out == its[i + 1].front_in, i
            assert s.culled + s.front_out == cand, (i, s)
        else:
            assert s.culled <= cand
        da, db = da + ka, db + kb
        if i:
            prev = its[i - 1].bound_after
            assert (s.bound_after <= prev) if kind == "min" else (s.bound_after >= prev), i
    assert (da, db) == (ta.depth, tb.depth)
    assert r.expanded_pairs == total


@pytest.mark.parametrize("kind", ["min", "max"])
@pytest.mark.parametrize("scene", ["rings", "shells", "random-blobs"])
def test_chunked_expansion_identical(md, gpu, kind, scene):
    """Arenas far too small for the fronts force chunked, depth-first
    expansion over many rounds (one per leaf chunk): the answer is bitwise
    the breadth-first one, the expanded candidates are accounted per
    iteration across chunks."""
    a, b = _scene(md, scene)
    ta, tb = _trees(md, a, b)
    run = md.run_min_query if kind == "min" else md.run_max_query
    want = run(a, b, ta, tb, md.EngineConfig(front_hard_cap=1 << 30))
    for arena in (1 << 16, 1 << 13, 1 << 10):
        cfg = md.EngineConfig(front_hard_cap=1 << 30, arena_entries=arena)
        pq = md.PreparedQuery(a, b, ta, tb, cfg, kind)
        got = pq.run()
        assert got.distance == want.distance, (arena, got.distance, want.distance)
        assert (got.witness.tri_a, got.witness.tri_b) == (want.witness.tri_a, want.witness.tri_b), arena
        np.testing.assert_array_equal(got.witness.point_a, want.witness.point_a)
        if arena == 1 << 10 and scene != "random-blobs":  # the blobs' fronts are tiny
            assert pq.res.rounds > 1, "the small arena must chunk"
        # per iteration (depth pair) the chunks' fronts add up
        assert got.iterations[-1].front_out == 0
        assert all(s.front_in > 0 for s in got.iterations)
        # synchronous C entry point loops the rounds itself
        assert run(a, b, ta, tb, cfg).distance == want.distance


def test_front_hard_cap_semantics_independent_of_arena(md, gpu):
    """FrontOverflowError (query.py:373-376, 448-449) depends on
    front_hard_cap only: the same query overflows with a roomy arena
    (breadth first) and with a tiny one (chunked, iteration totals)."""
    a, b = _scene(md, "rings")
    ta, tb = _trees(md, a, b)
    ok = md.run_min_query(a, b, ta, tb, md.EngineConfig(front_hard_cap=1 << 30, device_schedule=-1))
    cand, da, db = [], 0, 0
    for s in ok.iterations:
        ka, kb = min(s.k, ta.depth - da), min(s.k, tb.depth - db)
        cand.append(s.front_in << (ka + kb))
        da, db = da + ka, db + kb
    cap = max(cand) // 2
    # the reference schedule and the device schedule (whose k = 2 sweeps
    # only run while their candidates fit the cap) raise alike
    for arena in (0, 1 << 13):
        for sched in (-1, 0):
            with pytest.raises(md.FrontOverflowError) as ei:
                md.run_min_query(a, b, ta, tb, md.EngineConfig(front_hard_cap=cap, arena_entries=arena,
                                                               device_schedule=sched))
            assert ei.value.cap == cap and ei.value.candidates > cap
    # a cap well above every iteration's candidates passes in both layouts
    cap_ok = 4 * max(cand)
    for arena in (0, 1 << 13):
        for sched in (-1, 0):
            r = md.run_min_query(a, b, ta, tb, md.EngineConfig(front_hard_cap=cap_ok, arena_entries=arena,
                                                               device_schedule=sched))
            assert r.distance == ok.distance


def test_arena_too_small_fails_loudly(md, gpu):
    a, b = _scene(md, "rings")
    ta, tb = _trees(md, a, b)
    with pytest.raises(RuntimeError, match="arena"):
        md.run_min_query(a, b, ta, tb, md.EngineConfig(front_hard_cap=1 << 30, arena_entries=64))


def test_arena_config_validation(md):
    with pytest.raises(md.ConfigError):
        md.EngineConfig(arena_entries=-1)


def test_sequence_minmax_chunked_frames(md, gpu):
    """run_sequence_minmax overlaps frame f + 1's refits with frame f's narrow
    phases; a frame whose traversal is chunked (the arena far too small)
    cannot resume its later rounds after the next frame's refit, so it is
    recomputed through the plain API -- every frame equals the plain API's
    min and max, with a roomy arena and with a tiny one."""
    from paper_2411_11244_b200.parallel import release_frame_graphs

    a0, b0 = md.ring_pair_base(120, 60)
    ta, tb = md.build_f12(a0), md.build_f12(b0)
    xfs = [md.ring_frame_transforms(f) for f in range(0, 70, 7)]
    want = []
    for xa, xb in xfs:
        a, b = md.apply_transform(a0, xa), md.apply_transform(b0, xb)
        cfg = md.EngineConfig(front_hard_cap=1 << 30)
        want.append((md.run_min_query(a, b, ta, tb, cfg), md.run_max_query(a, b, ta, tb, cfg)))
    for arena in (0, 1 << 10):
        cfg = md.EngineConfig(front_hard_cap=1 << 30, arena_entries=arena)
        out = md.run_sequence_minmax(a0, b0, ta, tb, xfs, ("min", "max"), cfg)
        release_frame_graphs()
        for f, (wmin, wmax) in enumerate(want):
            for k, w in (("min", wmin), ("max", wmax)):
                d, t1, t2 = out[k][f]
                assert d == w.distance and (int(t1), int(t2)) == (w.witness.tri_a, w.witness.tri_b), (arena, f, k)


def test_back_to_back_launches_one_workspace(md, gpu):
    """Many queries enqueued back to back on one workspace without a host
    sync: every k_traverse launch meets on its own launch epoch (no memset,
    traverse.cu prologue_barrier), so a launch never starts from the previous
    one's state -- all answers equal the first (a duplicated epoch would
    deadlock or, with the spin watchdog, fail loudly)."""
    a, b = _scene(md, "rings")
    ta, tb = _trees(md, a, b)
    cfg = md.EngineConfig(front_hard_cap=1 << 30)
    for kind in ("min", "max"):
        pq = md.PreparedQuery(a, b, ta, tb, cfg, kind)
        want = pq.run()
        for _ in range(64):
            pq.launch()
        got = pq.collect()
        assert got.distance == want.distance and got.witness.tri_a == want.witness.tri_a, kind
        assert got.witness.tri_b == want.witness.tri_b, kind
