"""Front-traversal distance queries on the device (reference query.py).

`run_min_query` / `run_max_query` run the whole BVTT traversal -- adaptive
depth, expansion with AABB culling, float32 narrow phase, exact pass -- as a
fixed launch sequence inside libgdist (csrc/query.cu) with one device->host
copy at the end.  The returned distance is the reference's exact value (its
float64 or float32 arithmetic, per `precision`), and the witness is the
lexicographically smallest (tri_a, tri_b) pair attaining it, i.e. the
brute-force witness (query.py:571-601).  See DESIGN.md "Exactness".

The single-step API (`expand_front`, `process_leaf_pair`, `QueryState`) is
kept with the reference's semantics; its arithmetic runs in libgdist's exact
batch kernels.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .bounds import _device_bounds, _device_tri_tri
from .bvh import F12Bvh
from .errors import ConfigError, FrontOverflowError, SizeGuardError
from .mesh import TriangleMesh

BRUTE_FORCE_PAIR_LIMIT = 10_000_000  # query.py:48


@dataclass(frozen=True)
class EngineConfig:
    """Engine knobs (query.py:51-102).  `threads` and `batch_size` are
    accepted for compatibility; the device engine has no use for them."""

    front_cap: int = 262_144
    depth_cap: int = 5
    precision: int = 64
    threads: int | str = 1
    enhanced_bounds: bool = True
    culling: bool = True
    guarantee_witness: bool = False
    front_hard_cap: int = 16_777_216
    batch_size: int = 65_536
    # device extension: front arena entries (12 B each); 0 = sized from the
    # free HBM.  Independent of front_hard_cap.
    arena_entries: int = 0
    # device extension: expansion schedule (GdConfig.schedule).  -1 = the
    # reference's adaptive_depth exactly (IterationStat.k follows
    # query.py:266-284); 0 = the device schedule (fronts up to its default
    # threshold expand two levels per iteration where the reference rule
    # gives one); > 0 = the device schedule with that threshold in entries.
    # Distances and witnesses do not depend on it.
    device_schedule: int = 0

    def __post_init__(self):
        if self.front_cap < 4:
            raise ConfigError(f"front_cap must be >= 4, got {self.front_cap}")
        if not 1 <= self.depth_cap <= 16:
            raise ConfigError(f"depth_cap must be in [1, 16], got {self.depth_cap}")
        if self.precision not in (32, 64):
            raise ConfigError(f"precision must be 32 or 64, got {self.precision}")
        if self.batch_size < 4:
            raise ConfigError(f"batch_size must be >= 4, got {self.batch_size}")
        if self.front_hard_cap < 4:
            raise ConfigError("front_hard_cap must be >= 4")
        if self.device_schedule < -1 or self.device_schedule >= 1 << 31:
            raise ConfigError(f"device_schedule must be -1, 0 or a front size < 2^31, got {self.device_schedule}")
        if self.arena_entries < 0:
            raise ConfigError(f"arena_entries must be >= 0, got {self.arena_entries}")
        if isinstance(self.threads, str):
            if self.threads != "auto":
                raise ConfigError(f"threads must be a positive int or 'auto', got {self.threads!r}")
        elif self.threads < 1:
            raise ConfigError(f"threads must be >= 1, got {self.threads}")

    @property
    def dtype(self):
        return np.float32 if self.precision == 32 else np.float64

    @property
    def worker_count(self) -> int:
        if self.threads == "auto":
            return os.cpu_count() or 1
        return int(self.threads)


@dataclass(frozen=True)
class FrontEntry:
    """One unresolved node pair with its cached culling key (query.py:105-113)."""

    node_a: int
    node_b: int
    lower: float


@dataclass
class Front:
    """A front as flat arrays at one depth pair (query.py:116-133)."""

    node_a: np.ndarray
    node_b: np.ndarray
    lower: np.ndarray
    depth_a: int
    depth_b: int

    def __len__(self) -> int:
        return len(self.node_a)

    def entries(self) -> list:
        return [FrontEntry(int(a), int(b), float(lo)) for a, b, lo in zip(self.node_a, self.node_b, self.lower)]


@dataclass(frozen=True)
class Witness:
    """Triangle pair (and points on them) attaining a distance (query.py:136-144)."""

    distance: float
    tri_a: int
    tri_b: int
    point_a: np.ndarray
    point_b: np.ndarray


@dataclass(frozen=True)
class IterationStat:
    k: int
    front_in: int
    front_out: int
    culled: int
    bound_after: float

    def to_json_dict(self) -> dict:
        return {"k": self.k, "front_in": self.front_in, "front_out": self.front_out, "culled": self.culled,
                "bound_after": self.bound_after}


class QueryState:
    """Monotone bound + lexicographic witness cell (query.py:165-227)."""

    def __init__(self, kind: str, bound: float):
        if kind not in ("min", "max"):
            raise ValueError(f"kind must be 'min' or 'max', got {kind!r}")
        self.kind = kind
        self._bound = float(bound)
        self._witness = None
        self._lock = threading.Lock()
        self.iterations: list = []
        self.expanded_pairs = 0
        self.narrow_pairs = 0

    @property
    def bound(self) -> float:
        with self._lock:
            return self._bound

    def offer_bound(self, value: float) -> None:
        value = float(value)
        with self._lock:
            if (value < self._bound) if self.kind == "min" else (value > self._bound):
                self._bound = value

    @property
    def witness(self):
        with self._lock:
            return self._witness

    def offer_witness(self, distance: float, tri_a: int, tri_b: int, point_a, point_b) -> None:
        distance = float(distance)
        with self._lock:
            w = self._witness
            if w is None:
                better = True
            else:
                better = distance < w.distance if self.kind == "min" else distance > w.distance
                if not better and distance == w.distance:
                    better = (tri_a, tri_b) < (w.tri_a, w.tri_b)
            if better:
                self._witness = Witness(distance, int(tri_a), int(tri_b), np.array(point_a), np.array(point_b))

    def add_narrow_pairs(self, n: int) -> None:
        with self._lock:
            self.narrow_pairs += n

    def record_iteration(self, k: int, front_in: int, front_out: int, culled: int) -> None:
        self.iterations.append(IterationStat(k, front_in, front_out, culled, self.bound))


@dataclass(frozen=True)
class QueryResult:
    """query.py:230-263; `band_pairs` counts exact-pass evaluations."""

    kind: str
    distance: float
    witness: Witness | None
    iterations: tuple
    expanded_pairs: int
    narrow_pairs: int
    visited_nodes: int | None = None
    band_pairs: int = field(default=0, compare=False)
    rounds: int = field(default=1, compare=False)  # traversal rounds

    @property
    def witness_exact(self) -> bool:
        return self.witness is not None and self.witness.distance == self.distance

    @property
    def peak_front(self) -> int:
        return max((s.front_out for s in self.iterations), default=0)

    def to_json_dict(self) -> dict:
        w = self.witness
        return {
            "kind": self.kind,
            "distance": self.distance,
            "witness_exact": self.witness_exact,
            "tri_a": None if w is None else w.tri_a,
            "tri_b": None if w is None else w.tri_b,
            "point_a": None if w is None else [float(x) for x in w.point_a],
            "point_b": None if w is None else [float(x) for x in w.point_b],
            "iterations": [s.to_json_dict() for s in self.iterations],
            "expanded_pairs": self.expanded_pairs,
            "narrow_pairs": self.narrow_pairs,
            "peak_front": self.peak_front,
            "visited_nodes": self.visited_nodes,
        }


def adaptive_depth(n: int, cfg: EngineConfig, max_remaining: int) -> int:
    """Largest k with 4^k n < C, clamped to [1, min(depth_cap, max_remaining)]
    (query.py:266-284)."""
    if n < 1:
        raise ValueError("front size must be >= 1")
    if max_remaining < 1:
        raise ValueError("max_remaining must be >= 1")
    k = 1
    while k < cfg.depth_cap and k < max_remaining and (n << (2 * (k + 1))) < cfg.front_cap:
        k += 1
    return k


# ---------------------------------------------------------------------------
# device engine
# ---------------------------------------------------------------------------
_MAX_STATS = 64


class _Workspace:
    """Query scratch (front arena, band, state), per device AND per host
    thread -- two threads querying at once never share a workspace -- grown
    on demand and reused."""

    _tls = threading.local()

    @classmethod
    def get(cls, nbytes: int):
        torch = _lib.torch()
        dev = torch.cuda.current_device()
        cache = getattr(cls._tls, "cache", None)
        if cache is None:
            cache = cls._tls.cache = {}
        t = cache.get(dev)
        if t is None or t.numel() < nbytes:
            cache.pop(dev, None)
            t = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", dev))
            cache[dev] = t
        return t


_ARENA_MIN, _ARENA_MAX = 1 << 26, 1 << 28
_arena_auto: dict = {}
_arena_lock = threading.Lock()


def _auto_arena() -> int:
    """Front arena entries from the free HBM of the current device: an
    eighth of it, clamped to [2^26, 2^28] entries (0.8 - 3.2 GB), a power of
    two so repeated plans share one workspace size; decided once per device."""
    torch = _lib.torch()
    dev = torch.cuda.current_device()
    with _arena_lock:
        n = _arena_auto.get(dev)
        if n is None:
            free, _total = torch.cuda.mem_get_info(dev)
            n = max(_ARENA_MIN, min(_ARENA_MAX, 1 << max(0, (free // 8 // 12).bit_length() - 1)))
            _arena_auto[dev] = n
        return n


def _gd_config(cfg: EngineConfig, kind: str, warm_pair, band_cap: int = 0) -> _lib.GdConfig:
    g = _lib.GdConfig()
    g.kind = 1 if kind == "max" else 0
    g.precision = cfg.precision
    g.front_cap = cfg.front_cap
    g.depth_cap = cfg.depth_cap
    g.enhanced_bounds = int(bool(cfg.enhanced_bounds))
    g.culling = int(bool(cfg.culling))
    g.guarantee_witness = int(bool(cfg.guarantee_witness))
    g.front_hard_cap = cfg.front_hard_cap
    if warm_pair is not None:
        g.warm_a, g.warm_b = int(warm_pair[0]), int(warm_pair[1])
    else:
        g.warm_a = g.warm_b = -1
    g.band_cap = band_cap
    g.split_rank, g.split_world, g.split_level = 0, 1, 11
    g.arena_entries = cfg.arena_entries or _auto_arena()
    g.schedule = cfg.device_schedule
    return g


def _check_build(cfg: EngineConfig, bvh_a: F12Bvh, bvh_b: F12Bvh) -> None:
    """query.py:471-477."""
    for name, bvh in (("A", bvh_a), ("B", bvh_b)):
        if bvh.dtype != np.dtype(cfg.dtype):
            raise ConfigError(
                f"BVH {name} was built as {bvh.dtype}, engine precision is {cfg.precision}-bit; "
                f"rebuild with build_f12(mesh, dtype=...) to match"
            )


class PreparedQuery:
    """A query bound to its trees / config (and, per `bind`, meshes): the
    device views and workspace are resolved once, so repeated launches
    (frames, benches) cost only the kernel sequence.  `launch()` is
    asynchronous; `collect()` does the single device->host copy."""

    def __init__(self, mesh_a, mesh_b, bvh_a, bvh_b, cfg: EngineConfig, kind: str, warm_pair=None,
                 private_workspace: bool = False, frame: str = "world"):
        _check_build(cfg, bvh_a, bvh_b)
        if frame not in ("world", "b-local"):
            raise ValueError(f"frame must be 'world' or 'b-local', got {frame!r}")
        self.frame = frame
        self._pinned = self._ready = None
        self.kind = kind
        self.warm_pair = warm_pair
        self.trees = (bvh_a, bvh_b)
        self.g_cfg = _gd_config(cfg, kind, warm_pair)
        self.g_cfg.frame = 1 if frame == "b-local" else 0
        self.bind(mesh_a, mesh_b)
        nbytes = C.c_size_t(0)
        L = _lib.lib()
        _lib.check(L.gd_query_workspace_size(C.byref(self.g_a), C.byref(self.g_b), C.byref(self.g_cfg),
                                             C.byref(nbytes)), "query_workspace_size")
        self.ws = _lib.empty(nbytes.value, _lib.torch().uint8) if private_workspace else _Workspace.get(nbytes.value)
        self.res = _lib.GdResult()
        self.stats = (_lib.GdIterStat * _MAX_STATS)()

    def bind(self, mesh_a, mesh_b):
        """Point the query at (possibly moved) meshes of the same trees."""
        bvh_a, bvh_b = self.trees
        if self.warm_pair is not None:
            ta, tb = int(self.warm_pair[0]), int(self.warm_pair[1])
            if not (0 <= ta < mesh_a.n_triangles and 0 <= tb < mesh_b.n_triangles):
                raise IndexError(f"warm_pair {self.warm_pair} out of range")
        if self.frame == "b-local":
            # boxes in B's local frame: B untransformed, A under the relative
            # transform; the exact pass still sees the world meshes
            from .mesh import relative_mesh

            bvh_a.ensure_device(relative_mesh(mesh_a, mesh_b))
            bvh_b.ensure_device(mesh_b._root)
        else:
            bvh_a.ensure_device(mesh_a)
            bvh_b.ensure_device(mesh_b)
        self.meshes = (mesh_a, mesh_b)
        self.g_ma, self.g_mb = mesh_a.device_view(), mesh_b.device_view()
        self.g_a, self.g_b = bvh_a.device_view(), bvh_b.device_view()
        return self

    def launch(self, stream=None, traversal_done=None):
        """Enqueue the query on `stream` (default: the current stream).
        `traversal_done` (a torch.cuda.Event) is recorded right after the
        traversal: the trees' boxes may be refit for the next frame once it
        fires (gd_query_async_ev)."""
        ev = None
        if traversal_done is not None:
            if not traversal_done.cuda_event:  # torch creates the event lazily
                traversal_done.record()
            ev = C.c_void_p(traversal_done.cuda_event)
        _lib.check(_lib.lib().gd_query_async_ev(C.byref(self.g_ma), C.byref(self.g_mb), C.byref(self.g_a),
                                                C.byref(self.g_b), C.byref(self.g_cfg), _lib.ptr(self.ws),
                                                self.ws.numel(), None, stream or _lib.stream_ptr(), ev), "query")

    # -- bound-exchange rounds (split query)
    def traverse(self, round: int, sweep_budget: int = 1, stream=None):
        """Enqueue only the traversal, at most `sweep_budget` expansion
        sweeps (round 0 starts the query, later rounds continue it; no-op
        once it ended) -- gd_query_traverse.  Between rounds the caller may
        combine the ranks' bound cells (`bound_cell`)."""
        _lib.check(_lib.lib().gd_query_traverse(C.byref(self.g_ma), C.byref(self.g_mb), C.byref(self.g_a),
                                                C.byref(self.g_b), C.byref(self.g_cfg), _lib.ptr(self.ws),
                                                self.ws.numel(), int(round), int(sweep_budget),
                                                stream or _lib.stream_ptr()), "query_traverse")

    def finish(self, stream=None):
        """Enqueue the rest of the traversal and the narrow / exact phases
        (gd_query_finish); collect() as after launch()."""
        _lib.check(_lib.lib().gd_query_finish(C.byref(self.g_ma), C.byref(self.g_mb), C.byref(self.g_a),
                                              C.byref(self.g_b), C.byref(self.g_cfg), _lib.ptr(self.ws),
                                              self.ws.numel(), None, stream or _lib.stream_ptr()), "query_finish")

    def bound_cell(self):
        """The workspace's bound cell as a 1-element int32 CUDA tensor view
        (float32 bits of a non-negative bound: integer MIN / MAX order is the
        float order), for an all-reduce between traversal rounds."""
        p = C.c_void_p()
        _lib.check(_lib.lib().gd_query_bound_device(C.byref(self.g_cfg), _lib.ptr(self.ws), C.byref(p)),
                   "query_bound_device")
        off = p.value - self.ws.data_ptr()
        return self.ws[off:off + 4].view(_lib.torch().int32)

    def collect(self, stream=None) -> QueryResult:
        s = stream or _lib.stream_ptr()
        L = _lib.lib()
        _lib.check(L.gd_query_collect(C.byref(self.g_a), C.byref(self.g_b), C.byref(self.g_cfg), _lib.ptr(self.ws),
                                      None, C.byref(self.res), self.stats, _MAX_STATS, s), "query")
        self._finish_rounds(self.res, s)
        return _result(self.kind, self.res, self.stats)

    def _finish_rounds(self, res, s, rounds_ok: bool = True) -> bool:
        """A front larger than the arena is expanded in chunks: every leaf
        chunk ends a traversal round, and the record says `pending` (bit 0)
        until the last one; a round whose band overflowed says bit 1 until the
        rescan pass has run (gd_query_round decides; DESIGN.md "Front
        arena", "Exactness").  rounds_ok=False: stop (return False) before a
        further traversal round -- the caller's trees may already describe
        another frame (pipelined sequences); the rescan pass reads no boxes."""
        L = _lib.lib()
        while res.pending and res.status == 0:
            if not rounds_ok and not res.pending & 2:
                return False
            _lib.check(L.gd_query_round(C.byref(self.g_ma), C.byref(self.g_mb), C.byref(self.g_a), C.byref(self.g_b),
                                        C.byref(self.g_cfg), _lib.ptr(self.ws), self.ws.numel(), int(res.rounds), s),
                       "query_round")
            _lib.check(L.gd_query_collect(C.byref(self.g_a), C.byref(self.g_b), C.byref(self.g_cfg),
                                          _lib.ptr(self.ws), None, C.byref(self.res), self.stats, _MAX_STATS, s),
                       "query")
            res = self.res
        return True

    def run(self) -> QueryResult:
        self.launch()
        return self.collect()

    def seed_from(self, other: "PreparedQuery | None"):
        """Temporal warm start: seed this query's
        bound with `other`'s witness pair, read on the device when this query
        starts (GdConfig.warm_from), so no host round trip is needed between
        frames.  `other` must have been launched earlier on the same stream
        (it may be this query: the record is read before it is rewritten).
        Exact like warm_pair: only the work changes."""
        if other is None:
            self.g_cfg.warm_from = None
            return self
        p = C.c_void_p()
        _lib.check(_lib.lib().gd_query_result_device(C.byref(other.g_cfg), _lib.ptr(other.ws), C.byref(p)),
                   "query_result_device")
        self.g_cfg.warm_from = p.value
        return self

    # -- several queries in flight (each PreparedQuery with its own workspace)
    def launch_fetch(self, stream=None, traversal_done=None):
        """launch() + an asynchronous copy of the result record and stats to
        pinned host memory; `fetch()` waits for it.  The query's workspace
        is busy until fetch() returns."""
        torch = _lib.torch()
        if self._pinned is None:
            n = C.sizeof(_lib.GdResult) + _MAX_STATS * C.sizeof(_lib.GdIterStat)
            self._pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            self._ready = torch.cuda.Event()
        self.launch(stream, traversal_done)
        s = stream or _lib.stream_ptr()
        _lib.check(_lib.lib().gd_query_result_async(C.byref(self.g_cfg), _lib.ptr(self.ws), _lib.ptr(self._pinned),
                                                    _MAX_STATS, s), "query_result_async")
        self._ready.record()
        return self

    def fetch(self, rounds_ok: bool = True) -> QueryResult | None:
        """Wait for the launched query's record.  rounds_ok=False: None when
        the query still needs traversal rounds (see _finish_rounds)."""
        self._ready.synchronize()
        base = self._pinned.data_ptr()
        r = _lib.GdResult.from_address(base)
        stats = (_lib.GdIterStat * _MAX_STATS).from_address(base + C.sizeof(_lib.GdResult))
        if r.pending and r.status == 0:
            if not self._finish_rounds(r, _lib.stream_ptr(), rounds_ok):
                return None
            return _result(self.kind, self.res, self.stats)
        return _result(self.kind, r, stats)


def launch_group(plans, stream=None, traversal_done=None, host_dst=None, max_stats: int = 0):
    """Enqueue several PreparedQuery plans on the same meshes and trees (the
    min and max query of one frame, config 3) as one group
    (gd_query_group_async): their traversals back to back, then their narrow
    / exact chains side by side on forked streams, joined back into `stream`.
    Each plan's record is read with collect() as after launch(); with
    `host_dst` (pinned buffers, one per plan) the records are also copied at
    the end of each chain.  `traversal_done` (a torch.cuda.Event) is recorded
    after the last traversal."""
    plans = list(plans)
    if not plans:
        raise ValueError("launch_group needs at least one query")
    p0 = plans[0]
    for p in plans[1:]:
        if (p.g_a.box, p.g_b.box, p.g_ma.vtx, p.g_mb.vtx) != (p0.g_a.box, p0.g_b.box, p0.g_ma.vtx, p0.g_mb.vtx) or \
                bytes(p.g_ma) != bytes(p0.g_ma) or bytes(p.g_mb) != bytes(p0.g_mb):
            raise ValueError("the queries of a group share their meshes, transforms and trees")
    n = len(plans)
    cfgs = (_lib.GdConfig * n)(*[p.g_cfg for p in plans])
    wss = (C.c_void_p * n)(*[p.ws.data_ptr() for p in plans])
    sizes = (C.c_size_t * n)(*[p.ws.numel() for p in plans])
    dst = None if host_dst is None else (C.c_void_p * n)(*[t.data_ptr() for t in host_dst])
    ev = None
    if traversal_done is not None:
        if not traversal_done.cuda_event:
            traversal_done.record()
        ev = C.c_void_p(traversal_done.cuda_event)
    _lib.check(_lib.lib().gd_query_group_async(C.byref(p0.g_ma), C.byref(p0.g_mb), C.byref(p0.g_a),
                                               C.byref(p0.g_b), n, cfgs, wss, sizes, dst, int(max_stats),
                                               stream or _lib.stream_ptr(), ev), "query_group")


class FrameGraph:
    """One frame of a rigid-motion sequence -- refit both trees, then one
    query per kind in `kinds` with the copy of each result record to pinned
    host memory -- captured once as a CUDA graph (gd_frame_graph_create,
    SURVEY.md 8(f) row 1) and replayed per frame for the frame's moved
    meshes (same base meshes, any rigid transforms): one host call per frame.
    The queries use private workspaces bound to the graph; their traversals
    run back to back, then their narrow / exact chains side by side
    (gd_query_group_async).  Single GPU (no split query).

    wait_event / done_event (torch.cuda.Event): every replay first waits for
    wait_event's latest record and records done_event once its traversals
    have read the trees' boxes -- two graphs alternating on two streams, each
    waiting for the other's done_event, run frame f + 1's refits while frame
    f's narrow / exact phases still run (run_sequence_minmax)."""

    def __init__(self, mesh_a, mesh_b, bvh_a, bvh_b, kinds=("min", "max"), cfg: EngineConfig | None = None,
                 wait_event=None, done_event=None):
        torch = _lib.torch()
        cfg = cfg or EngineConfig()
        if not kinds or any(k not in ("min", "max") for k in kinds):
            raise ValueError(f"kinds must be a non-empty sequence of 'min' / 'max', got {kinds!r}")
        self.kinds = tuple(kinds)
        self.trees = (bvh_a, bvh_b)
        self._roots = (mesh_a._root, mesh_b._root)
        # stage the base vertices (and lay out the leaves) outside the capture
        bvh_a.ensure_device(mesh_a)
        bvh_b.ensure_device(mesh_b)
        self.plans = [PreparedQuery(mesh_a, mesh_b, bvh_a, bvh_b, cfg, k, private_workspace=True) for k in self.kinds]
        nbytes = C.sizeof(_lib.GdResult) + _MAX_STATS * C.sizeof(_lib.GdIterStat)
        self._pinned = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in self.kinds]
        n = len(self.kinds)
        cfgs = (_lib.GdConfig * n)(*[p.g_cfg for p in self.plans])
        wss = (C.c_void_p * n)(*[p.ws.data_ptr() for p in self.plans])
        sizes = (C.c_size_t * n)(*[p.ws.numel() for p in self.plans])
        dst = (C.c_void_p * n)(*[t.data_ptr() for t in self._pinned])
        g_ma, g_mb = mesh_a.device_view(), mesh_b.device_view()

        def handle(ev):
            if ev is None:
                return None
            if not ev.cuda_event:  # torch creates the event lazily
                ev.record()
            return C.c_void_p(ev.cuda_event)

        self.overlapped = wait_event is not None
        h = C.c_void_p()
        _lib.check(_lib.lib().gd_frame_graph_create(C.byref(g_ma), C.byref(g_mb), C.byref(bvh_a.device_view()),
                                                    C.byref(bvh_b.device_view()), n, cfgs, wss, sizes, dst,
                                                    _MAX_STATS, 1, 1, handle(wait_event), handle(done_event),
                                                    C.byref(h)), "frame_graph_create")
        self._h = h
        self._ready = torch.cuda.Event()

    def launch(self, mesh_a, mesh_b, stream=None):
        """Enqueue the frame for `mesh_a` / `mesh_b` (rigid moves of the
        captured meshes' bases) on `stream` (a torch.cuda.Stream; default:
        the current stream)."""
        if (mesh_a._root, mesh_b._root) != self._roots:
            raise ValueError("a FrameGraph replays moves of the meshes it was captured with")
        g_ma, g_mb = mesh_a.device_view(), mesh_b.device_view()
        _lib.check(_lib.lib().gd_frame_graph_launch(self._h, C.byref(g_ma), C.byref(g_mb),
                                                    stream.cuda_stream if stream is not None else _lib.stream_ptr()),
                   "frame_graph_launch")
        for bvh, m in zip(self.trees, (mesh_a, mesh_b)):
            bvh._mesh = m  # the boxes now describe the moved mesh
            bvh._export_cache = None
            bvh._host_boxes = None
        for p in self.plans:
            p.meshes = (mesh_a, mesh_b)
            p.g_ma, p.g_mb = g_ma, g_mb
        self._ready.record(stream)
        return self

    def results(self) -> dict:
        """Wait for the launched frame; {kind: QueryResult}."""
        self._ready.synchronize()
        out = {}
        for kind, p, buf in zip(self.kinds, self.plans, self._pinned):
            base = buf.data_ptr()
            r = _lib.GdResult.from_address(base)
            stats = (_lib.GdIterStat * _MAX_STATS).from_address(base + C.sizeof(_lib.GdResult))
            if r.pending and r.status == 0:  # not final: the rescan pass / remaining rounds, synchronously
                # (overlapped: the next frame's refits may already have
                # rewritten the boxes further rounds would read -- then the
                # caller recomputes this frame, run_sequence_minmax)
                if not p._finish_rounds(r, _lib.stream_ptr(), rounds_ok=not self.overlapped):
                    out[kind] = None
                    continue
                out[kind] = _result(kind, p.res, p.stats)
            else:
                out[kind] = _result(kind, r, stats)
        return out

    def run(self, mesh_a, mesh_b) -> dict:
        return self.launch(mesh_a, mesh_b).results()

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().gd_frame_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# recently used query plans of this host thread (a plan uses the thread's
# workspace), keyed by (trees, config, kind, warm pair, device); the trees are
# held weakly
_PLANS_TLS = threading.local()
_PLANS_MAX = 16


def _plan(mesh_a, mesh_b, bvh_a, bvh_b, cfg, kind, warm_pair) -> PreparedQuery:
    import weakref

    _PLANS = getattr(_PLANS_TLS, "plans", None)
    if _PLANS is None:
        _PLANS = _PLANS_TLS.plans = {}
    wp = None if warm_pair is None else (int(warm_pair[0]), int(warm_pair[1]))
    key = (id(bvh_a), id(bvh_b), cfg, kind, wp, _lib.torch().cuda.current_device())
    ent = _PLANS.get(key)
    if ent is not None:
        ra, rb, pq = ent
        if ra() is bvh_a and rb() is bvh_b:
            _check_build(cfg, bvh_a, bvh_b)
            return pq.bind(mesh_a, mesh_b)
    pq = PreparedQuery(mesh_a, mesh_b, bvh_a, bvh_b, cfg, kind, wp)
    pq.trees = (weakref.proxy(bvh_a), weakref.proxy(bvh_b))
    if len(_PLANS) >= _PLANS_MAX:
        _PLANS.pop(next(iter(_PLANS)))
    _PLANS[key] = (weakref.ref(bvh_a), weakref.ref(bvh_b), pq)
    return pq


def _result(kind: str, r: _lib.GdResult, stats) -> QueryResult:
    if r.status == _lib.GD_ERR_FRONT_OVERFLOW:
        raise _lib.overflow_error(r)
    if r.status == _lib.GD_ERR_WORKSPACE:
        raise RuntimeError("front arena too small for this query (EngineConfig.arena_entries); "
                           "a few entries per tree level are needed")
    if r.status != 0:
        raise RuntimeError(f"device query failed with status {r.status}")
    its = tuple(
        IterationStat(int(s.k), int(s.front_in), int(s.front_out), int(s.culled), float(s.bound_after))
        for s in stats[: min(r.iterations, _MAX_STATS)]
    )
    w = None
    if r.tri_a >= 0:
        w = Witness(float(r.witness_distance), int(r.tri_a), int(r.tri_b), np.array(r.point_a[:], dtype=np.float64),
                    np.array(r.point_b[:], dtype=np.float64))
    return QueryResult(kind, float(r.distance), w, its, int(r.expanded_pairs), int(r.narrow_pairs),
                       band_pairs=int(r.band_pairs), rounds=max(1, int(r.rounds)))


def _run_query(mesh_a, mesh_b, bvh_a, bvh_b, cfg, kind, warm_pair=None) -> QueryResult:
    return _plan(mesh_a, mesh_b, bvh_a, bvh_b, cfg, kind, warm_pair).run()


def run_min_query(mesh_a: TriangleMesh, mesh_b: TriangleMesh, bvh_a: F12Bvh, bvh_b: F12Bvh,
                  cfg: EngineConfig | None = None, warm_pair=None) -> QueryResult:
    """Exact minimum distance between two meshes (query.py:540-555)."""
    return _run_query(mesh_a, mesh_b, bvh_a, bvh_b, cfg or EngineConfig(), "min", warm_pair)


def run_max_query(mesh_a: TriangleMesh, mesh_b: TriangleMesh, bvh_a: F12Bvh, bvh_b: F12Bvh,
                  cfg: EngineConfig | None = None, warm_pair=None) -> QueryResult:
    """Exact maximum distance between two meshes (query.py:558-568)."""
    return _run_query(mesh_a, mesh_b, bvh_a, bvh_b, cfg or EngineConfig(), "max", warm_pair)


# ---------------------------------------------------------------------------
# brute force (query.py:571-619) -- all pairs on the device
# ---------------------------------------------------------------------------
def _brute_force(mesh_a, mesh_b, kind, force, dtype):
    na, nb = mesh_a.n_triangles, mesh_b.n_triangles
    n_pairs = na * nb
    if n_pairs == 0:
        raise ValueError("both meshes need at least one triangle")
    if n_pairs > BRUTE_FORCE_PAIR_LIMIT and not force:
        raise SizeGuardError(n_pairs, BRUTE_FORCE_PAIR_LIMIT)
    torch = _lib.torch()
    dev = _lib.device()
    prec = 32 if np.dtype(dtype) == np.float32 else 64
    pa = torch.from_numpy(np.ascontiguousarray(mesh_a.triangle_points(dtype))).to(dev)
    pb = torch.from_numpy(np.ascontiguousarray(mesh_b.triangle_points(dtype))).to(dev)
    r = _lib.GdResult()
    _lib.check(_lib.lib().gd_brute_force(1 if kind == "max" else 0, prec, _lib.ptr(pa), na, _lib.ptr(pb), nb,
                                         C.byref(r), _lib.stream_ptr()), "brute_force")
    w = Witness(float(r.distance), int(r.tri_a), int(r.tri_b), np.array(r.point_a[:]), np.array(r.point_b[:]))
    return float(r.distance), w


def brute_force_min(mesh_a, mesh_b, force: bool = False, dtype=np.float64):
    """All-pairs exact minimum (query.py:604-612); lexicographic ties."""
    return _brute_force(mesh_a, mesh_b, "min", force, dtype)


def brute_force_max(mesh_a, mesh_b, force: bool = False, dtype=np.float64):
    """All-pairs exact maximum (query.py:615-619)."""
    return _brute_force(mesh_a, mesh_b, "max", force, dtype)


# ---------------------------------------------------------------------------
# single-step API with the reference's exact semantics
# ---------------------------------------------------------------------------
def _narrow_update(state: QueryState, ids_a, ids_b, pts_a, pts_b) -> None:
    """query.py:287-307 with the exact device kernels."""
    if len(ids_a) == 0:
        return
    d, p, q = _device_tri_tri(state.kind, pts_a[ids_a], pts_b[ids_b])
    if state.kind == "min":
        pick = np.lexsort((ids_b, ids_a, d))[0]
    else:
        pick = np.lexsort((ids_b, ids_a, -d))[0]
    state.add_narrow_pairs(len(ids_a))
    state.offer_bound(d[pick])
    state.offer_witness(d[pick], ids_a[pick], ids_b[pick], p[pick].astype(np.float64), q[pick].astype(np.float64))


def process_leaf_pair(leaf_a_prims, leaf_b_prims, mesh_a, mesh_b, state: QueryState) -> QueryState:
    """All 1..4 triangle pairs of two leaves into the state (query.py:310-331)."""
    ids_a = np.asarray([a for a in leaf_a_prims for _ in leaf_b_prims], dtype=np.int64)
    ids_b = np.asarray([b for _ in leaf_a_prims for b in leaf_b_prims], dtype=np.int64)
    _narrow_update(state, ids_a, ids_b, mesh_a.triangle_points(), mesh_b.triangle_points())
    return state


def _leaf_tri_pairs(bvh_a, bvh_b, na, nb):
    ta = bvh_a.leaf_tris[na - (bvh_a.leaf_count - 1)]
    tb = bvh_b.leaf_tris[nb - (bvh_b.leaf_count - 1)]
    outa, outb = [], []
    for i in (0, 1):
        for j in (0, 1):
            sel = (ta[:, i] >= 0) & (tb[:, j] >= 0)
            outa.append(ta[sel, i])
            outb.append(tb[sel, j])
    return np.concatenate(outa), np.concatenate(outb)


def expand_front(front: Front, k: int, state: QueryState, bvh_a: F12Bvh, bvh_b: F12Bvh, pts_a, pts_b,
                 cfg: EngineConfig, pool=None) -> Front:
    """One expansion sweep with the reference's batch semantics
    (query.py:349-451); bounds and narrow phase run in the exact device
    batch kernels, so results equal the reference's bit for bit."""
    rem_a = bvh_a.depth - front.depth_a
    rem_b = bvh_b.depth - front.depth_b
    ka, kb = min(k, rem_a), min(k, rem_b)
    shift = ka + kb
    n_in = len(front)
    n_candidates = n_in << shift
    if n_candidates > cfg.front_hard_cap:
        raise FrontOverflowError(n_candidates, n_in, cfg.front_hard_cap)
    to_leaves = k == max(rem_a, rem_b)
    state.expanded_pairs += n_candidates
    mask_b = (1 << kb) - 1
    amin_all, amax_all = bvh_a.node_min, bvh_a.node_max
    bmin_all, bmax_all = bvh_b.node_min, bvh_b.node_max
    is_min = state.kind == "min"
    outs, culled_total = [], 0
    for start in range(0, n_candidates, cfg.batch_size):
        idx = np.arange(start, min(start + cfg.batch_size, n_candidates), dtype=np.int64)
        e = idx >> shift
        off = idx & ((1 << shift) - 1)
        na = ((front.node_a[e] + 1) << ka) - 1 + (off >> kb)
        nb = ((front.node_b[e] + 1) << kb) - 1 + (off & mask_b)
        boxes = (amin_all[na], amax_all[na], bmin_all[nb], bmax_all[nb])
        key = _device_bounds(0 if is_min else 1, *boxes)
        bound = state.bound
        if not cfg.culling:
            keep = np.ones(len(idx), dtype=bool)
        elif is_min:
            keep = key <= bound if (to_leaves and cfg.guarantee_witness) else key < bound
        else:
            keep = key >= bound if (to_leaves and cfg.guarantee_witness) else key > bound
        culled_total += int(len(idx) - keep.sum())
        na, nb, key = na[keep], nb[keep], key[keep]
        if to_leaves:
            if len(na):
                ia, ib = _leaf_tri_pairs(bvh_a, bvh_b, na, nb)
                _narrow_update(state, ia, ib, pts_a, pts_b)
            continue
        if len(na):
            kept = tuple(b[keep] for b in boxes)
            which = (2 if cfg.enhanced_bounds else 1) if is_min else (3 if cfg.enhanced_bounds else 0)
            upd = _device_bounds(which, *kept)
            state.offer_bound(upd.min() if is_min else upd.max())
            outs.append((na, nb, key))
    out = Front(
        node_a=np.concatenate([o[0] for o in outs]) if outs else np.empty(0, dtype=np.int64),
        node_b=np.concatenate([o[1] for o in outs]) if outs else np.empty(0, dtype=np.int64),
        lower=np.concatenate([o[2] for o in outs]) if outs else np.empty(0, dtype=np.float64),
        depth_a=front.depth_a + ka,
        depth_b=front.depth_b + kb,
    )
    if len(out) > cfg.front_hard_cap:
        raise FrontOverflowError(len(out), n_in, cfg.front_hard_cap)
    state.record_iteration(k, n_in, len(out), culled_total)
    return out


def run_dfs_baseline(mesh_a, mesh_b, bvh_b, kind: str = "min") -> QueryResult:
    """Per-triangle descent comparator (query.py:622-708): every triangle of
    A walks B's tree depth-first, nearer child first, pruning against one
    shared monotone bound (csrc/dfs.cuh, one device thread per triangle).
    Same distance as the front engine (float64 exact pass); `visited_nodes`
    counts node examinations.  No iterations, expanded_pairs = 0."""
    if kind not in ("min", "max"):
        raise ValueError(f"kind must be 'min' or 'max', got {kind!r}")
    if mesh_a.n_triangles == 0:
        return QueryResult(kind, float("inf") if kind == "min" else float("-inf"), None, (), 0, 0, visited_nodes=0)
    g = _gd_config(EngineConfig(), kind, None)
    g.precision = 64  # the reference walks float64 triangle points
    bvh_b.ensure_device(mesh_b)
    g_ma, g_mb, g_b = mesh_a.device_view(), mesh_b.device_view(), bvh_b.device_view()
    L = _lib.lib()
    nbytes = C.c_size_t(0)
    _lib.check(L.gd_query_workspace_size(C.byref(g_b), C.byref(g_b), C.byref(g), C.byref(nbytes)),
               "query_workspace_size")
    ws = _Workspace.get(nbytes.value)
    r, visited = _lib.GdResult(), C.c_int64(0)
    _lib.check(L.gd_dfs_query(C.byref(g_ma), C.byref(g_mb), C.byref(g_b), C.byref(g), _lib.ptr(ws), ws.numel(),
                              C.byref(r), C.byref(visited), _lib.stream_ptr()), "dfs_query")
    res = _result(kind, r, ())
    return QueryResult(kind, res.distance, res.witness, (), 0, res.narrow_pairs, visited_nodes=int(visited.value),
                       band_pairs=res.band_pairs)
