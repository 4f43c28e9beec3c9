"""Multi-GPU paths on one GPU (gpurun provides one): the split query's parts
run one after another and combine to the single-GPU answer; two processes
sharing cuda:0 over a gloo group run the distributed split query (bound cells
linked over CUDA IPC, all-reduced between budgeted traversal rounds, and not
exchanged) and the sharded frame sequence end to end."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SCENES = [("interlocked-rings", {"nu": 100, "nv": 50}), ("interlocked-rings", {"nu": 250, "nv": 100}),
          ("nested-shells", {"lat": 24, "lon": 30, "r_outer": 0.83}), ("random-blobs", {"n": 3000, "seed": 5}),
          ("offset-grids", {"res": 30})]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("scene", range(len(SCENES)))
def test_split_parts_combine(md, gpu, scene, world):
    from paper_2411_11244_b200 import parallel

    kind_, params = SCENES[scene]
    a, b = md.gen_scene(kind_, params)
    ta, tb = md.build_f12(a), md.build_f12(b)
    cfg = md.EngineConfig(front_hard_cap=1 << 26)
    for kind in ("min", "max"):
        full = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb, cfg)
        parts = [parallel.split_part(a, b, ta, tb, kind, cfg, r, world) for r in range(world)]
        rows = [(p.distance, p.witness.tri_a if p.witness else -1, p.witness.tri_b if p.witness else -1, i)
                for i, p in enumerate(parts)]
        best = parallel.combine_parts(kind, rows)
        assert best[0] == full.distance, (kind_, kind, world)
        assert (best[1], best[2]) == (full.witness.tri_a, full.witness.tri_b)
        win = parts[best[3]].witness
        assert win.point_a.tolist() == full.witness.point_a.tolist()
        # the work is dealt out (each part culls with its own bound, a valid
        # global bound, so a part far from the optimum may explore a little
        # more than its share)
        if full.expanded_pairs > 10_000:
            assert min(p.expanded_pairs for p in parts) < full.expanded_pairs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2411_11244_b200 as md

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = md.gen_scene("interlocked-rings", {"nu": 120, "nv": 60})
        ta, tb = md.build_f12(a), md.build_f12(b)
        out = {}
        for kind in ("min", "max"):
            for rep in range(2):  # the linked plan is cached: the second call reuses the IPC mapping
                r = md.run_split_query(a, b, ta, tb, kind)  # default: bound cells linked over CUDA IPC
                out[kind] = (r.distance, r.witness.tri_a, r.witness.tri_b, r.witness.point_a.tolist())
            loc = md.run_split_query(a, b, ta, tb, kind, share_bound=False)
            out[kind + "_local"] = (loc.distance, loc.witness.tri_a, loc.witness.tri_b, loc.witness.point_a.tolist())
            # the per-round all-reduce of the bound cells (SURVEY.md 8(e) as written)
            ar = md.run_split_query(a, b, ta, tb, kind, bound_exchange="allreduce")
            out[kind + "_allreduce"] = (ar.distance, ar.witness.tri_a, ar.witness.tri_b, ar.witness.point_a.tolist())
            out[kind + "_work"] = (r.expanded_pairs, loc.expanded_pairs, ar.expanded_pairs)
        tz, tbase = md.ring_pair_base(60, 30)
        za, zb = md.build_f12(tz), md.build_f12(tbase)
        xfs = [md.ring_frame_transforms(f) for f in range(0, 70, 10)]
        seq = md.run_sequence(tz, tbase, za, zb, xfs, "min")
        # config 3 on the ranks: frames sharded, each frame one CUDA graph replay
        both = md.run_sequence_minmax(tz, tbase, za, zb, xfs)
        out["graph_min_equal"] = bool(np.array_equal(both["min"], seq))
        md.parallel.release_split_plans()
        md.parallel.release_frame_graphs()
        q.put((rank, out, seq.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_processes_gloo(md, gpu):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = []
    for _ in range(world):
        try:
            got.append(q.get(timeout=240))
        except Exception:
            for p in procs:
                p.kill()
            raise AssertionError(f"worker failed: exit codes {[p.exitcode for p in procs]}")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a, b = md.gen_scene("interlocked-rings", {"nu": 120, "nv": 60})
    ta, tb = md.build_f12(a), md.build_f12(b)
    tz, tbase = md.ring_pair_base(60, 30)
    za, zb = md.build_f12(tz), md.build_f12(tbase)
    want_seq = []
    for f in range(0, 70, 10):
        xa, xb = md.ring_frame_transforms(f)
        fa, fb = md.apply_transform(tz, xa), md.apply_transform(tbase, xb)
        md.refit(za, fa)
        md.refit(zb, fb)
        r = md.run_min_query(fa, fb, za, zb)
        want_seq.append((r.distance, r.witness.tri_a, r.witness.tri_b))
    for rank, out, seq in got:
        for kind in ("min", "max"):
            r = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb)
            assert out[kind][:3] == (r.distance, r.witness.tri_a, r.witness.tri_b), (rank, kind)
            assert out[kind][3] == r.witness.point_a.tolist()
            assert out[kind + "_local"] == out[kind], (rank, kind)
            assert out[kind + "_allreduce"] == out[kind], (rank, kind)
            # exchanging bounds never makes a rank's part bigger than culling
            # with its own bound alone (same cells, tighter or equal bound)
            ipc, local, ar = out[kind + "_work"]
            assert ipc <= local * 1.02 and ar <= local * 1.02, (rank, kind, out[kind + "_work"])
        assert out["graph_min_equal"], rank
        assert np.array_equal(np.asarray(seq), np.asarray(want_seq, dtype=np.float64)), rank


@pytest.mark.parametrize("budget", [1, 2, 5])
@pytest.mark.parametrize("scene", [0, 2])
def test_budgeted_traversal_rounds(md, gpu, scene, budget):
    """gd_query_traverse / gd_query_finish (the allreduce mode's rounds):
    a traversal paused every `budget` sweeps and continued, with more rounds
    than it needs (the extra ones are no-ops), returns the one-launch answer
    and statistics; the bound cell view reads the bound; a small arena's
    chunked traversal still completes through the pending rounds."""
    import struct

    from paper_2411_11244_b200 import query as Q

    kind_, params = SCENES[scene]
    a, b = md.gen_scene(kind_, params)
    ta, tb = md.build_f12(a), md.build_f12(b)
    for kind in ("min", "max"):
        for arena in (0, 1 << 11):
            cfg = md.EngineConfig(front_hard_cap=1 << 28, arena_entries=arena, device_schedule=-1)
            want = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb, cfg)
            pq = Q.PreparedQuery(a, b, ta, tb, cfg, kind, private_workspace=True)
            for r in range(ta.depth + 3):
                pq.traverse(r, budget)
            bits = int(pq.bound_cell().item()) & 0xFFFFFFFF
            bound = struct.unpack("<f", struct.pack("<I", bits))[0]
            pq.finish()
            got = pq.collect()
            assert got.distance == want.distance, (kind, arena, budget)
            assert (got.witness.tri_a, got.witness.tri_b) == (want.witness.tri_a, want.witness.tri_b)
            its = got.iterations
            assert its and its[0].front_in == 1 and its[-1].front_out == 0
            da = db = 0
            for s in its:
                da, db = da + min(s.k, ta.depth - da), db + min(s.k, tb.depth - db)
            assert (da, db) == (ta.depth, tb.depth)
            # the cell holds the slack-carrying bound: at or beyond the answer
            assert (bound >= want.distance) if kind == "min" else (bound <= want.distance)


def test_sequence_pipelining_and_inflight_queries(md, gpu):
    """run_sequence with frame pipelining (second refit stream, two query plans
    in flight) equals the plain frame-by-frame loop; launch_fetch/fetch of two
    plans in flight equal run()."""
    from paper_2411_11244_b200 import query as Q

    tz, tbase = md.ring_pair_base(80, 40)
    za, zb = md.build_f12(tz), md.build_f12(tbase)
    xfs = [md.ring_frame_transforms(f) for f in range(0, 90, 7)]
    for kind in ("min", "max"):
        piped = md.run_sequence(tz, tbase, za, zb, xfs, kind)  # world frame, pipelined
        plain = md.run_sequence(tz, tbase, za, zb, xfs, kind, pipelined=False)
        local_b = md.run_sequence(tz, tbase, za, zb, xfs, kind, frame="b-local")
        assert np.array_equal(piped, plain) and np.array_equal(piped, local_b), kind
        # temporal warm start (device-side seed from the previous frame's record)
        warm = md.run_sequence(tz, tbase, za, zb, xfs, kind, warm=True)
        warm_plain = md.run_sequence(tz, tbase, za, zb, xfs, kind, pipelined=False, warm=True)
        assert np.array_equal(piped, warm) and np.array_equal(piped, warm_plain), kind
    a, b = md.gen_scene("interlocked-rings", {"nu": 90, "nv": 45})
    ta, tb = md.build_f12(a), md.build_f12(b)
    cfg = md.EngineConfig()
    p1 = Q.PreparedQuery(a, b, ta, tb, cfg, "min", private_workspace=True)
    p2 = Q.PreparedQuery(a, b, ta, tb, cfg, "max", private_workspace=True)
    p1.launch_fetch()
    p2.launch_fetch()
    r2, r1 = p2.fetch(), p1.fetch()
    for r, run in ((r1, md.run_min_query), (r2, md.run_max_query)):
        want = run(a, b, ta, tb, cfg)
        assert r.distance == want.distance and (r.witness.tri_a, r.witness.tri_b) == (want.witness.tri_a,
                                                                                       want.witness.tri_b)
        assert len(r.iterations) == len(want.iterations)  # front sizes depend on bound timing; depths do not


def test_seed_from_previous_frame(md, gpu):
    """PreparedQuery.seed_from: the seeded query returns the cold answer with
    no more expanded pairs than the cold run, also when the source record
    belongs to another scene's query (any pair is a valid seed)."""
    from paper_2411_11244_b200 import query as Q

    tz, tbase = md.ring_pair_base(120, 60)
    za, zb = md.build_f12(tz), md.build_f12(tbase)
    cfg = md.EngineConfig()
    xa, xb = md.ring_frame_transforms(10)
    a0, b0 = md.apply_transform(tz, xa), md.apply_transform(tbase, xb)
    for kind in ("min", "max"):
        src = Q.PreparedQuery(a0, b0, za, zb, cfg, kind, private_workspace=True)
        src.run()
        xa, xb = md.ring_frame_transforms(11)
        a1, b1 = md.apply_transform(tz, xa), md.apply_transform(tbase, xb)
        cold = (md.run_min_query if kind == "min" else md.run_max_query)(a1, b1, za, zb, cfg)
        pq = Q.PreparedQuery(a1, b1, za, zb, cfg, kind, private_workspace=True).seed_from(src)
        r = pq.run()
        assert r.distance == cold.distance and (r.witness.tri_a, r.witness.tri_b) == (cold.witness.tri_a,
                                                                                      cold.witness.tri_b)
        assert r.expanded_pairs <= cold.expanded_pairs
        assert pq.seed_from(None).g_cfg.warm_from is None
