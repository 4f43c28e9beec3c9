"""Multi-GPU drivers (the reference is single-process,
query.py:426-433 parallelises only over CPU threads).

* Frames of a rotation / trajectory sequence are independent: each rank (one
  process per GPU, torch.distributed) holds full replicas of both meshes and
  trees and evaluates frames f = rank, rank + world, ...; one all-gather at the
  end assembles every frame's (distance, tri_a, tri_b) on every rank.  No
  collective inside the frame loop ("scaling": "weak").
* A single large query is split by dealing the BVTT node pairs to the ranks
  by a hash of their ancestor pair at a fixed tree level (`split_level`,
  independent of each rank's adaptive-depth schedule); every rank expands its
  part independently -- its own bound is a valid global bound, so every pair
  that can attain the optimum survives on its owner -- and the exact answers
  are combined with the reference's lexicographic witness rule
  (query.py:205-220) in one all-gather.  The ranks' bounds are exchanged
  while they traverse (`bound_exchange`):
    "ipc" (the default for a process group): the bound cells are mapped into
      each other over CUDA IPC (NVLink peer memory); a rank that improves on
      its tile's bound snapshot also applies the bound to every peer cell with
      a system-scope atomic, inside the kernels -- no round, no host sync;
    "allreduce" (SURVEY.md 8(e) as written; the fallback when IPC mapping
      fails): the traversal runs in rounds of one expansion sweep per launch
      and the 4-byte bound cells are all-reduced (MIN / MAX) between rounds
      with torch.distributed (NCCL on GPUs), all on the stream;
    "none": every rank culls with its own bound only.

The collective plumbing is torch.distributed (NCCL on GPUs, gloo in the CPU
tests); the per-frame / per-part compute is libgdist's.
"""

from __future__ import annotations

import math

import numpy as np


def _dist():
    import torch.distributed as dist

    return dist


def world_info(group=None) -> tuple[int, int]:
    """(rank, world size) of `group`, (0, 1) without torch.distributed."""
    dist = _dist()
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def frames_of_rank(n_frames: int, rank: int, world: int) -> range:
    """Frames owned by `rank`: f = rank (mod world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return range(rank, n_frames, world)


def gather_frames(n_frames: int, local: dict, group=None, device=None) -> np.ndarray:
    """Assemble per-frame results (f -> (distance, tri_a, tri_b)) computed on
    the ranks into one (n_frames, 3) float64 array on every rank (one
    all-gather of a fixed-size padded tensor)."""
    import torch

    rank, world = world_info(group)
    per = math.ceil(n_frames / world) if n_frames else 0
    buf = torch.full((per, 4), -1.0, dtype=torch.float64)
    for i, f in enumerate(frames_of_rank(n_frames, rank, world)):
        d, ta, tb = local[f]
        buf[i] = torch.tensor([float(f), float(d), float(ta), float(tb)], dtype=torch.float64)
    if world == 1:
        rows = buf
    else:
        dist = _dist()
        dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                                  if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        buf = buf.to(dev)
        out = torch.empty((world * per, 4), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(out, buf, group=group)
        rows = out.cpu()
    res = np.full((n_frames, 3), np.nan)
    for f, d, ta, tb in rows.numpy():
        if f >= 0:
            res[int(f)] = (d, ta, tb)
    return res


def run_frames(n_frames: int, frame_fn, group=None, device=None) -> np.ndarray:
    """Evaluate frame_fn(f) -> (distance, tri_a, tri_b) for this rank's frames
    and gather all frames on every rank."""
    rank, world = world_info(group)
    local = {f: frame_fn(f) for f in frames_of_rank(n_frames, rank, world)}
    return gather_frames(n_frames, local, group, device)


def run_sequence_minmax(mesh_a, mesh_b, bvh_a, bvh_b, transforms, kinds=("min", "max"), cfg=None,
                        group=None) -> dict:
    """Config 3: every kind in `kinds` (min and max distance) at every frame
    of a rigid-motion sequence, frames sharded over the ranks like
    run_sequence.  Each frame -- refit A, refit B, the queries (traversals
    back to back, then their narrow / exact chains side by side) and the
    copies of their records -- is ONE CUDA graph replay (query.FrameGraph).
    Two graphs alternate on two streams, each replay waiting (on the device)
    for the previous frame's traversals only: frame f + 1's refits overlap
    frame f's narrow / exact phases, and the host reads frame f's records
    while frame f + 1 runs.  Returns {kind: (n_frames, 3) array of
    (distance, tri_a, tri_b)} on every rank."""
    import torch

    from .mesh import apply_transform
    from .query import FrameGraph, run_max_query, run_min_query

    rank, world = world_info(group)
    mine = list(frames_of_rank(len(transforms), rank, world))
    local = {k: {} for k in kinds}

    def moved(f):
        xa, xb = transforms[f]
        return (mesh_a if xa is None else apply_transform(mesh_a, xa),
                mesh_b if xb is None else apply_transform(mesh_b, xb))

    def take(f, g):
        res = g.results()
        if any(r is None for r in res.values()):
            # a chunked traversal (front larger than the arena) whose later
            # rounds would read boxes the next frame may have refit already:
            # wait for everything in flight, then this frame on its own
            torch.cuda.synchronize()
            a, b = moved(f)
            from .bvh import refit

            refit(bvh_a, a)
            refit(bvh_b, b)
            res = {k: (run_min_query if k == "min" else run_max_query)(a, b, bvh_a, bvh_b, cfg) for k in kinds}
            torch.cuda.synchronize()  # before the graphs' streams touch the boxes again
        for k, r in res.items():
            w = r.witness
            local[k][f] = (r.distance, -1 if w is None else w.tri_a, -1 if w is None else w.tri_b)

    # the two graphs (with their events and streams) are kept for the next
    # call on the same trees / meshes
    key = (id(bvh_a), id(bvh_b), id(mesh_a._root), id(mesh_b._root), tuple(kinds), cfg)
    ent = _FRAME_GRAPHS.get(key)
    if ent is None or ent[0] is not bvh_a or ent[1] is not bvh_b:
        release_frame_graphs()  # one sequence's graphs at a time (each holds its query workspaces)
        events = (torch.cuda.Event(), torch.cuda.Event())
        for e in events:
            e.record()  # a first replay's wait is then satisfied at once
        ent = (bvh_a, bvh_b, [], events, (torch.cuda.Stream(), torch.cuda.Stream()))
        _FRAME_GRAPHS[key] = ent
    graphs, events, streams = ent[2], ent[3], ent[4]
    if not mine:
        return {k: gather_frames(len(transforms), local[k], group) for k in kinds}
    # both graphs exist before any replay: creating one stages / refits on
    # the current stream, which must not race a replay on the side streams
    while len(graphs) < 2:
        j = len(graphs)
        a, b = moved(mine[0])
        graphs.append(FrameGraph(a, b, bvh_a, bvh_b, kinds, cfg, wait_event=events[1 - j], done_event=events[j]))
    cur = torch.cuda.current_stream()
    for st in streams:
        st.wait_stream(cur)  # after the caller's work (builds, refits, earlier frames)
    pending = None
    for i, f in enumerate(mine):
        a, b = moved(f)
        j = i % 2
        g = graphs[j].launch(a, b, stream=streams[j])
        if pending is not None:
            take(*pending)
        pending = (f, g)
    if pending is not None:
        take(*pending)
    for st in streams:
        cur.wait_stream(st)
    return {k: gather_frames(len(transforms), local[k], group) for k in kinds}


_FRAME_GRAPHS: dict = {}


def release_frame_graphs():
    """Destroy the cached frame graphs of run_sequence_minmax (and their
    query workspaces)."""
    for ent in _FRAME_GRAPHS.values():
        for st in ent[4]:
            st.synchronize()  # a replay may still be in flight
        for g in ent[2]:
            g.close()
    _FRAME_GRAPHS.clear()


def run_sequence(mesh_a, mesh_b, bvh_a, bvh_b, transforms, kind: str = "min", cfg=None, group=None,
                 pipelined: bool = True, frame: str = "world", warm: bool = False, graph: bool = False) -> np.ndarray:
    """Distance over a rigid-motion sequence, frames sharded over the ranks.

    transforms: list of (xf_a, xf_b) RigidTransform pairs (either may be
    None = identity).  Every rank holds both meshes and trees; returns the
    (n_frames, 3) array of (distance, tri_a, tri_b) on every rank.

    frame: "world" refits both trees per frame.  "b-local" traverses in B's
    local frame (GdConfig.frame = 1): B's boxes are computed once and only
    A's tree is refit per frame, under A's transform relative to B -- half
    the refit work when both meshes move -- but axis-aligned boxes cull
    differently in another frame: on the rings sequence the B-local
    traversal is slower than the refit it saves.  The exact pass
    stays in world coordinates, so the answers are bitwise the world ones.
    pipelined: the refit for frame f+1 runs on a second stream as soon as
    frame f's traversal has read the boxes (gd_query_async_ev), overlapping
    frame f's narrow and exact phases, and two query plans are in flight so
    the host never waits on the GPU between frames.
    warm: seed each frame's bound with the previous frame's witness pair on
    the device (PreparedQuery.seed_from; temporal coherence, exact).
    graph: each frame (refits + query + record copy) is one CUDA graph
    replay (run_sequence_minmax); world frame, no warm start."""
    import torch

    from .bvh import refit
    from .mesh import apply_transform, relative_mesh
    from .query import EngineConfig, PreparedQuery

    if frame not in ("world", "b-local"):
        raise ValueError(f"frame must be 'world' or 'b-local', got {frame!r}")
    if graph:
        if frame != "world" or warm:
            raise ValueError("graph=True runs world-frame frames without warm start")
        return run_sequence_minmax(mesh_a, mesh_b, bvh_a, bvh_b, transforms, (kind,), cfg, group)[kind]
    cfg = cfg or EngineConfig()
    rank, world = world_info(group)
    mine = list(frames_of_rank(len(transforms), rank, world))
    local_b = frame == "b-local"

    def moved(f):
        xa, xb = transforms[f]
        return (mesh_a if xa is None else apply_transform(mesh_a, xa),
                mesh_b if xb is None else apply_transform(mesh_b, xb))

    def refit_frame(a, b):
        if local_b:
            refit(bvh_a, relative_mesh(a, b))
        else:
            refit(bvh_a, a)
            refit(bvh_b, b)

    def row(r):
        w = r.witness
        return r.distance, (-1 if w is None else w.tri_a), (-1 if w is None else w.tri_b)

    local = {}
    if not mine:
        return gather_frames(len(transforms), local, group)
    if local_b:
        refit(bvh_b, mesh_b._root)  # B's boxes in its own frame, once
    if not pipelined:
        plan = None
        for f in mine:
            a, b = moved(f)
            refit_frame(a, b)
            if plan is None:
                plan = PreparedQuery(a, b, bvh_a, bvh_b, cfg, kind, private_workspace=warm, frame=frame)
            elif warm:
                plan.seed_from(plan)
            local[f] = row(plan.bind(a, b).run())
        return gather_frames(len(transforms), local, group)
    qs = torch.cuda.current_stream()
    rs = torch.cuda.Stream()
    rs.wait_stream(qs)

    def refit_on_rs(a, b, after=None):
        with torch.cuda.stream(rs):
            if after is not None:
                rs.wait_event(after)
            refit_frame(a, b)
            done = torch.cuda.Event()
            done.record(rs)
        return done

    cur = moved(mine[0])
    done = refit_on_rs(*cur)
    qs.wait_event(done)
    plans = [PreparedQuery(cur[0], cur[1], bvh_a, bvh_b, cfg, kind, private_workspace=True, frame=frame)
             for _ in range(2)]
    def take(f, pq):
        r = pq.fetch(rounds_ok=False)
        if r is None:
            # a chunked traversal (front larger than the arena): its later
            # rounds would read boxes the next frame's refit may have
            # rewritten -- wait for everything in flight, then this frame on
            # its own (and the boxes back to the frame in flight after it)
            torch.cuda.synchronize()
            a, b = moved(f)
            refit_frame(a, b)
            r = PreparedQuery(a, b, bvh_a, bvh_b, cfg, kind, frame=frame).run()
            refit_frame(*cur)
            torch.cuda.synchronize()
        local[f] = row(r)

    pending = None
    for i, f in enumerate(mine):
        if i:
            qs.wait_event(done)
        pq = plans[i % 2].bind(*cur)
        if warm and i:
            pq.seed_from(plans[(i - 1) % 2])
        trav = torch.cuda.Event()
        pq.launch_fetch(traversal_done=trav)
        if i + 1 < len(mine):
            nxt = moved(mine[i + 1])
            done = refit_on_rs(*nxt, after=trav)
            cur = nxt
        if pending is not None:
            take(*pending)
        pending = (f, pq)
    take(*pending)
    qs.wait_stream(rs)
    return gather_frames(len(transforms), local, group)


def combine_parts(kind: str, parts: list) -> tuple:
    """Combine per-rank exact answers (distance, tri_a, tri_b) of a split
    query with the reference's rule: best distance, then the
    lexicographically smallest (tri_a, tri_b) (query.py:205-220)."""
    found = [p for p in parts if p[1] >= 0]
    if not found:
        return parts[0]
    if kind == "min":
        return min(found, key=lambda p: (p[0], p[1], p[2]))
    return min(found, key=lambda p: (-p[0], p[1], p[2]))


_SPLIT_PLANS: dict = {}


def _link_bounds(pq, rank: int, world: int, group=None):
    """Map every rank's bound cell into this rank (CUDA IPC; collective over
    `group`) and point this plan's GdConfig.peer_bounds at the others'."""
    import ctypes as C

    import torch

    from . import _lib

    dist = _dist()
    L = _lib.lib()
    cell = C.c_void_p()
    _lib.check(L.gd_query_bound_device(C.byref(pq.g_cfg), _lib.ptr(pq.ws), C.byref(cell)), "query_bound_device")
    handle = (C.c_char * 64)()
    off = C.c_uint64()
    _lib.check(L.gd_ipc_handle(cell, handle, C.byref(off)), "ipc_handle")
    mine = (rank, bytes(handle), int(off.value))
    objs = [None] * world
    dist.all_gather_object(objs, mine, group=group)
    peers, opened = [], []
    for r, h, o in sorted(objs):
        if r == rank:
            continue
        ptr = C.c_void_p()
        _lib.check(L.gd_ipc_open((C.c_char * 64).from_buffer_copy(h), o, C.byref(ptr)), "ipc_open")
        peers.append(ptr.value)
        opened.append(ptr.value - o)
    arr = torch.tensor(peers, dtype=torch.int64, device=torch.device("cuda", torch.cuda.current_device()))
    pq._peer_arr, pq._peer_bases = arr, opened
    pq.g_cfg.peer_bounds = arr.data_ptr()
    pq.g_cfg.n_peers = len(peers)


def _split_plan(mesh_a, mesh_b, bvh_a, bvh_b, kind, cfg, rank, world, split_level, group):
    """The cached per-rank plan of a bound-sharing split query (private
    workspace whose bound cell is linked to the other ranks' once), or None
    when some rank could not map the others' cells (collective decision)."""
    import torch

    from . import _lib
    from .query import PreparedQuery

    key = (id(bvh_a), id(bvh_b), cfg, kind, rank, world, split_level, id(group))
    ent = _SPLIT_PLANS.get(key)
    if ent is None or ent[0] is not bvh_a or ent[1] is not bvh_b:
        pq = PreparedQuery(mesh_a, mesh_b, bvh_a, bvh_b, cfg, kind, private_workspace=True)
        pq.g_cfg.split_rank, pq.g_cfg.split_world, pq.g_cfg.split_level = int(rank), int(world), int(split_level)
        try:
            _link_bounds(pq, rank, world, group)
            ok = 1
        except RuntimeError:
            ok = 0
        dist = _dist()
        flag = torch.tensor([ok], dtype=torch.int32)
        if dist.get_backend(group) == "nccl":
            flag = flag.cuda()
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if not int(flag.item()):
            for base in getattr(pq, "_peer_bases", []):
                _lib.lib().gd_ipc_close(base)
            return None
        ent = (bvh_a, bvh_b, pq)
        _SPLIT_PLANS[key] = ent
    return ent[2].bind(mesh_a, mesh_b)


def _allreduce_rounds(mesh_a, mesh_b, bvh_a, bvh_b, kind, cfg, rank, world, split_level, group,
                      sweep_budget: int = 1):
    """This rank's part with the bound all-reduced between traversal rounds
    (SURVEY.md 8(e)): round r runs at most `sweep_budget` expansion sweeps
    (gd_query_traverse), then the ranks' 4-byte bound cells are combined
    with an all-reduce MIN (min query) / MAX (max query) -- the cells hold
    float bits of non-negative bounds, so the int32 order is the float order
    -- all enqueued on the stream (NCCL) without a host sync.  Every rank
    runs the same number of rounds (one per level of the deeper tree, the
    most sweeps a breadth-first traversal takes); rounds after a rank's
    traversal ended are no-ops on it.  Then the unbudgeted rest (a chunked
    traversal) and the narrow / exact phases."""
    from .query import PreparedQuery

    dist = _dist()
    pq = PreparedQuery(mesh_a, mesh_b, bvh_a, bvh_b, cfg, kind)
    pq.g_cfg.split_rank, pq.g_cfg.split_world, pq.g_cfg.split_level = int(rank), int(world), int(split_level)
    cell = pq.bound_cell()
    nccl = dist.get_backend(group) == "nccl"
    op = dist.ReduceOp.MAX if kind == "max" else dist.ReduceOp.MIN
    for r in range(max(bvh_a.depth, bvh_b.depth, 1)):
        pq.traverse(r, sweep_budget)
        if nccl:
            dist.all_reduce(cell, op=op, group=group)
        else:  # gloo (CPU tests, ranks sharing a GPU): through host memory
            host = cell.cpu()
            dist.all_reduce(host, op=op, group=group)
            cell.copy_(host)
    pq.finish()
    return pq.collect()


def release_split_plans(group=None):
    """Drop the bound-linked split plans and their workspaces (collective:
    after a barrier no rank writes into another's bound cell any more).
    Linked plans are kept until then -- a peer may still hold a mapping of
    their bound cells."""
    from . import _lib

    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        _lib.torch().cuda.synchronize()
        dist.barrier(group=group)
    for _, _, pq in list(_SPLIT_PLANS.values()):
        for base in getattr(pq, "_peer_bases", []):
            _lib.lib().gd_ipc_close(base)
    _SPLIT_PLANS.clear()


BOUND_EXCHANGES = ("ipc", "allreduce", "none")


def run_split_query(mesh_a, mesh_b, bvh_a, bvh_b, kind: str = "min", cfg=None, group=None, split_level: int | None = None,
                    rank: int | None = None, world: int | None = None, share_bound: bool | None = None,
                    bound_exchange: str | None = None):
    """One query split over the ranks of `group` (or, with explicit
    rank / world, one part of it -- e.g. to emulate the split on one GPU).

    Each rank expands only the node pairs whose ancestor pair at tree level
    `split_level` hashes to it (gdist.h GdConfig.split_*), and the exact
    per-rank answers are combined with the reference's witness rule.  The
    ranks' bounds are exchanged per `bound_exchange` (module docstring):
    "ipc" by default when a process group spans the ranks ("allreduce" if
    the IPC mapping fails), "none" for a single part.  `share_bound` is the
    older switch: True = "ipc", False = "none".  The returned QueryResult
    carries the global distance / witness and this rank's own iteration
    statistics.  Collective: every rank of the group calls it with the same
    arguments."""
    import torch

    from .query import EngineConfig, QueryResult, Witness

    dist = _dist()
    grouped = rank is None or world is None
    if grouped:
        rank, world = world_info(group)
    cfg = cfg or EngineConfig()
    if split_level is None:
        split_level = default_split_level(bvh_a, bvh_b)
    if bound_exchange is None:
        if share_bound is not None:
            bound_exchange = "ipc" if share_bound else "none"
        else:
            bound_exchange = "ipc"
    if bound_exchange not in BOUND_EXCHANGES:
        raise ValueError(f"bound_exchange must be one of {BOUND_EXCHANGES}, got {bound_exchange!r}")
    if not (grouped and world > 1):
        bound_exchange = "none"  # one part alone: nobody to exchange with
    if bound_exchange == "ipc":
        # every rank has finished its previous split query (the all-gather
        # below), so no peer cell is still in use by another query
        pq = _split_plan(mesh_a, mesh_b, bvh_a, bvh_b, kind, cfg, rank, world, split_level, group)
        if pq is None:  # the cells could not be mapped on some rank
            bound_exchange = "allreduce"
        else:
            r = pq.run()
    if bound_exchange == "allreduce":
        r = _allreduce_rounds(mesh_a, mesh_b, bvh_a, bvh_b, kind, cfg, rank, world, split_level, group)
    elif bound_exchange == "none":
        r = split_part(mesh_a, mesh_b, bvh_a, bvh_b, kind, cfg, rank, world, split_level)
    w = r.witness
    mine = torch.tensor([r.distance, -1.0 if w is None else w.tri_a, -1.0 if w is None else w.tri_b,
                         *(w.point_a if w is not None else np.zeros(3)), *(w.point_b if w is not None else np.zeros(3))],
                        dtype=torch.float64)
    if world > 1 and dist.is_available() and dist.is_initialized() and world == dist.get_world_size(group):
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else mine.device
        out = torch.empty(world * mine.numel(), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(out, mine.to(dev), group=group)
        rows = out.cpu().numpy().reshape(world, -1)
    else:
        rows = mine.numpy()[None]
    parts = [(float(x[0]), int(x[1]), int(x[2]), i) for i, x in enumerate(rows)]
    best = combine_parts(kind, parts)
    row = rows[best[3]]
    wit = None if best[1] < 0 else Witness(best[0], best[1], best[2], row[3:6].copy(), row[6:9].copy())
    return QueryResult(kind, best[0], wit, r.iterations, r.expanded_pairs, r.narrow_pairs, band_pairs=r.band_pairs)


def default_split_level(bvh_a, bvh_b) -> int:
    """Tree level whose ancestor pairs deal the work: 11 (4M ancestor pairs,
    the best balance measured on the rings / shells), at
    least 3 levels above the shallower tree's leaves."""
    return max(1, min(11, min(bvh_a.depth, bvh_b.depth) - 3))


def split_part(mesh_a, mesh_b, bvh_a, bvh_b, kind, cfg, rank: int, world: int, split_level: int | None = None):
    """This rank's part of a split query: its exact best over the node pairs
    it owns (QueryResult with the part's own witness and statistics)."""
    from .query import PreparedQuery

    if split_level is None:
        split_level = default_split_level(bvh_a, bvh_b)
    pq = PreparedQuery(mesh_a, mesh_b, bvh_a, bvh_b, cfg, kind)
    pq.g_cfg.split_rank, pq.g_cfg.split_world, pq.g_cfg.split_level = int(rank), int(world), int(split_level)
    return pq.run()
