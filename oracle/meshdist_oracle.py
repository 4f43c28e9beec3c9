"""CPU oracle for the gDist hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's algorithm
(`/root/reference/pkg/src/meshdist`, pure Python + numpy) for the path that
`BASELINE.json:north_star` names: f12-BVH build/refit -> front traversal with
AABB bounds -> exact triangle-triangle narrow phase.  It exists so that the
CUDA product (`paper_2411_11244_b200`) can be checked on machines where the
reference is absent (the GPU box).  Rules:

* Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s reference /
  cpu_baseline legs may import this module, and only as a checker or as the
  timed CPU baseline.  The product package never imports it.
* Every function cites the reference file:line it restates.  Arithmetic is
  written component-wise (x, y, z arrays) but in exactly the reference's
  operation order, so results are bitwise identical to the reference in both
  float64 and float32 (verified by `tests/test_oracle_reference.py` against
  the live reference in the build container and by the committed golden
  vectors in `tests/golden/`).

Parity pin: golden vectors generated from the reference itself by
`tests/golden/make_golden.py` (SPEC known-answer examples, random batteries,
tree dumps, engine runs) -- see tests/golden/README.md.
"""

from __future__ import annotations

import heapq
import math
from bisect import bisect_right
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

MORTON_BITS = 21
BRUTE_LIMIT = 10_000_000  # query.py:48


# ---------------------------------------------------------------------------
# small component-wise vector helpers (x, y, z) tuples of arrays
# ---------------------------------------------------------------------------

def _v(arr):
    """(N, 3) array -> tuple of three (N,) component views."""
    return (arr[..., 0], arr[..., 1], arr[..., 2])


def _sub(a, b):
    return (a[0] - b[0], a[1] - b[1], a[2] - b[2])


def _dot(a, b):
    # numpy's length-3 reduction is ((x + y) + z); bounds.py:38-39
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]


def _madd(p, t, u):
    """p + t*u component-wise (bounds.py:169, 195-199)."""
    return (p[0] + t * u[0], p[1] + t * u[1], p[2] + t * u[2])


def _cross(a, b):
    # numpy.cross order: (a1 b2 - a2 b1, a2 b0 - a0 b2, a0 b1 - a1 b0)
    return (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])


def _pick(cond, a, b):
    return (np.where(cond, a[0], b[0]), np.where(cond, a[1], b[1]), np.where(cond, a[2], b[2]))


def _stack(v):
    return np.stack(v, axis=-1)


# ---------------------------------------------------------------------------
# mesh (mesh.py)
# ---------------------------------------------------------------------------

def triangle_points(vertices, triangles, dtype=np.float64):
    """Cast first, then gather (mesh.py:64-66)."""
    return np.asarray(vertices).astype(dtype, copy=False)[np.asarray(triangles)]


def rodrigues(axis, angle):
    """c*I + s*[a]x + (1-c)*a a^T (mesh.py:86-99)."""
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    c, s = math.cos(angle), math.sin(angle)
    k = np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])
    return c * np.eye(3) + s * k + (1.0 - c) * np.outer(a, a)


def transform_vertices(vertices, rotation, translation):
    """V @ R^T + t (mesh.py:102-105)."""
    return np.asarray(vertices, dtype=np.float64) @ np.asarray(rotation).T + np.asarray(translation)


# ---------------------------------------------------------------------------
# box bounds (bounds.py:47-101)
# ---------------------------------------------------------------------------

def box_min_lower(amin, amax, bmin, bmax):
    """Exact box-box minimum distance (bounds.py:47-51, Eq. 5)."""
    g = np.maximum(amin - bmax, bmin - amax)
    g = np.maximum(g, 0.0)
    gx, gy, gz = _v(g)
    return np.sqrt((gx * gx + gy * gy) + gz * gz)


def box_max_upper(amin, amax, bmin, bmax):
    """Exact box-box maximum distance (bounds.py:54-57, Eqs. 6-7)."""
    h = np.maximum(np.abs(amin - bmax), np.abs(amax - bmin))
    hx, hy, hz = _v(h)
    return np.sqrt((hx * hx + hy * hy) + hz * hz)


def _face_intervals(lo, hi, face):
    """Face `face` of box [lo, hi] as a degenerate box (bounds.py:60-67):
    face 2*ax pins axis ax to lo, face 2*ax+1 pins it to hi."""
    flo = lo.copy()
    fhi = hi.copy()
    ax = face // 2
    if face % 2 == 0:
        fhi[..., ax] = lo[..., ax]
    else:
        flo[..., ax] = hi[..., ax]
    return flo, fhi


def enhanced_min_upper(amin, amax, bmin, bmax):
    """Min over 36 face pairs of the face-rectangle max distance
    (bounds.py:70-84, Eq. 9).  Evaluated pair by pair in the reference's
    face order so the minimum is bitwise the reference's."""
    best = None
    faces_a = [_face_intervals(amin, amax, f) for f in range(6)]
    faces_b = [_face_intervals(bmin, bmax, f) for f in range(6)]
    for fa in faces_a:
        for fb in faces_b:
            d = box_max_upper(fa[0], fa[1], fb[0], fb[1])
            best = d if best is None else np.minimum(best, d)
    return best


def enhanced_max_lower(amin, amax, bmin, bmax):
    """Max over 36 face pairs of the face-rectangle min distance
    (bounds.py:87-101, Eq. 10)."""
    best = None
    faces_a = [_face_intervals(amin, amax, f) for f in range(6)]
    faces_b = [_face_intervals(bmin, bmax, f) for f in range(6)]
    for fa in faces_a:
        for fb in faces_b:
            d = box_min_lower(fa[0], fa[1], fb[0], fb[1])
            best = d if best is None else np.maximum(best, d)
    return best


# ---------------------------------------------------------------------------
# exact triangle narrow phase (bounds.py:146-330)
# ---------------------------------------------------------------------------

def _clamp_ratio(num, den):
    """num/den clamped to [0,1], 0 where den == 0 (bounds.py:146-150)."""
    out = np.zeros_like(num)
    np.divide(num, den, out=out, where=den != 0)
    return np.clip(out, 0.0, 1.0)


def _segment_pair(p0, u, q0, v):
    """Lumelsky clamped closest points (bounds.py:153-169)."""
    w = _sub(q0, p0)
    uu = _dot(u, u)
    vv = _dot(v, v)
    uv = _dot(u, v)
    uw = _dot(u, w)
    vw = _dot(v, w)
    t = _clamp_ratio(uw * vv - vw * uv, uu * vv - uv * uv)
    s = _clamp_ratio(t * uv - vw, vv)
    t = _clamp_ratio(s * uv + uw, uu)
    return _madd(p0, t, u), _madd(q0, s, v)


def _point_triangle(p, a, b, c):
    """Ericson Voronoi walk with guarded divisions (bounds.py:172-221).
    The first matching region in the reference's list wins."""
    ab = _sub(b, a)
    ac = _sub(c, a)
    ap = _sub(p, a)
    d1 = _dot(ab, ap)
    d2 = _dot(ac, ap)
    bp = _sub(p, b)
    d3 = _dot(ab, bp)
    d4 = _dot(ac, bp)
    cp = _sub(p, c)
    d5 = _dot(ab, cp)
    d6 = _dot(ac, cp)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    on_ab = _madd(a, _clamp_ratio(d1, d1 - d3), ab)
    on_ac = _madd(a, _clamp_ratio(d2, d2 - d6), ac)
    e43 = d4 - d3
    e56 = d5 - d6
    on_bc = _madd(b, _clamp_ratio(e43, e43 + e56), _sub(c, b))
    total = (va + vb) + vc
    inv = np.zeros_like(total)
    np.divide(1.0, total, out=inv, where=total != 0)
    inner = _madd(_madd(a, vb * inv, ab), vc * inv, ac)
    regions = [
        ((d1 <= 0) & (d2 <= 0), a),
        ((d3 >= 0) & (d4 <= d3), b),
        ((vc <= 0) & (d1 >= 0) & (d3 <= 0), on_ab),
        ((d6 >= 0) & (d5 <= d6), c),
        ((vb <= 0) & (d2 >= 0) & (d6 <= 0), on_ac),
        ((va <= 0) & (e43 >= 0) & (e56 >= 0), on_bc),
        (total == 0, on_ab),
    ]
    out = inner
    for cond, choice in reversed(regions):
        out = _pick(cond, choice, out)
    return out


def _pierce(s0, s1, a, b, c):
    """Transversal segment-through-triangle test (bounds.py:224-242)."""
    ba = _sub(b, a)
    n = _cross(ba, _sub(c, a))
    d = _sub(s1, s0)
    den = _dot(n, d)
    ok = den != 0
    t = np.zeros_like(den)
    np.divide(_dot(n, _sub(a, s0)), den, out=t, where=ok)
    ok = ok & (t >= 0.0) & (t <= 1.0)
    x = _madd(s0, t, d)
    ok = ok & (_dot(n, _cross(ba, _sub(x, a))) >= 0)
    ok = ok & (_dot(n, _cross(_sub(c, b), _sub(x, b))) >= 0)
    ok = ok & (_dot(n, _cross(_sub(a, c), _sub(x, c))) >= 0)
    return ok, x


def tri_tri_min(t1, t2):
    """Exact min distance + witness points for (N,3,3) triangle batches
    (bounds.py:245-306): 9 edge-edge pairs (edge i of t1 outer), then
    6 vertex-triangle projections interleaved A_i->B, B_i->A, first strict
    minimum wins; pierce test only when the best is positive."""
    t1 = np.asarray(t1)
    t2 = np.asarray(t2)
    A = [_v(t1[:, i]) for i in range(3)]
    B = [_v(t2[:, i]) for i in range(3)]
    n = len(t1)
    best = np.full(n, np.inf, dtype=t1.dtype)
    bp = tuple(np.zeros(n, dtype=t1.dtype) for _ in range(3))
    bq = tuple(np.zeros(n, dtype=t1.dtype) for _ in range(3))

    def offer(p, q):
        nonlocal best, bp, bq
        w = _sub(p, q)
        d2 = _dot(w, w)
        take = d2 < best
        best = np.where(take, d2, best)
        bp = _pick(take, p, bp)
        bq = _pick(take, q, bq)

    for i in range(3):
        pa = A[i]
        ua = _sub(A[(i + 1) % 3], pa)
        for j in range(3):
            qb = B[j]
            vb = _sub(B[(j + 1) % 3], qb)
            offer(*_segment_pair(pa, ua, qb, vb))
    for i in range(3):
        offer(A[i], _point_triangle(A[i], B[0], B[1], B[2]))
        offer(_point_triangle(B[i], A[0], A[1], A[2]), B[i])

    positive = best > 0
    if positive.any():
        hit_any = np.zeros(n, dtype=bool)
        pt = tuple(np.zeros(n, dtype=t1.dtype) for _ in range(3))
        for i in range(3):
            for (s0, s1, tri) in ((A[i], A[(i + 1) % 3], B), (B[i], B[(i + 1) % 3], A)):
                hit, x = _pierce(s0, s1, tri[0], tri[1], tri[2])
                pt = _pick(hit & ~hit_any, x, pt)
                hit_any = hit_any | hit
        stab = positive & hit_any
        best = np.where(stab, 0.0, best)
        bp = _pick(stab, pt, bp)
        bq = _pick(stab, pt, bq)
    return np.sqrt(best), _stack(bp), _stack(bq)


def tri_tri_max(t1, t2):
    """Max over the 9 vertex pairs, first strict maximum (bounds.py:309-330)."""
    t1 = np.asarray(t1)
    t2 = np.asarray(t2)
    n = len(t1)
    best = np.full(n, -1.0, dtype=t1.dtype)
    bp = tuple(np.zeros(n, dtype=t1.dtype) for _ in range(3))
    bq = tuple(np.zeros(n, dtype=t1.dtype) for _ in range(3))
    for i in range(3):
        p = _v(t1[:, i])
        for j in range(3):
            q = _v(t2[:, j])
            w = _sub(p, q)
            d2 = _dot(w, w)
            take = d2 > best
            best = np.where(take, d2, best)
            bp = _pick(take, p, bp)
            bq = _pick(take, q, bq)
    return np.sqrt(best), _stack(bp), _stack(bq)


# ---------------------------------------------------------------------------
# f12-BVH (bvh.py)
# ---------------------------------------------------------------------------

def _spread3(x):
    """Spread 21 bits to every third bit (bvh.py:58-66)."""
    x = x.astype(np.uint64) & np.uint64(0x1FFFFF)
    for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                        (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        x = (x | (x << np.uint64(shift))) & np.uint64(mask)
    return x


def morton_order(vertices, triangles):
    """(codes, ids) sorted by (code, id) (bvh.py:69-95): fp64 centroids
    normalised into the box of ALL vertices, 21-bit quantisation, x at bit 0."""
    V = np.asarray(vertices, dtype=np.float64)
    T = np.asarray(triangles)
    if len(T) == 0:
        raise ValueError("mesh has no triangles")
    P = V[T]
    cen = ((P[:, 0] + P[:, 1]) + P[:, 2]) / 3.0
    lo = V.min(axis=0)
    span = V.max(axis=0) - lo
    span = np.where(span > 0.0, span, 1.0)
    frac = np.maximum((cen - lo) / span, 0.0)
    q = np.minimum((frac * float(1 << MORTON_BITS)).astype(np.uint64), np.uint64((1 << MORTON_BITS) - 1))
    code = _spread3(q[:, 0]) | (_spread3(q[:, 1]) << np.uint64(1)) | (_spread3(q[:, 2]) << np.uint64(2))
    ids = np.arange(len(T), dtype=np.int64)
    perm = np.lexsort((ids, code))
    return code[perm], ids[perm]


def pair_surface_areas(order, tri_lo, tri_hi):
    """Surface-area key of merging Morton neighbours i, i+1 (bvh.py:117-120)."""
    lo = np.minimum(tri_lo[order[:-1]], tri_lo[order[1:]])
    hi = np.maximum(tri_hi[order[:-1]], tri_hi[order[1:]])
    e = hi - lo
    ex, ey, ez = _v(e)
    return (ex * ey + ey * ez) + ez * ex


def greedy_pairs(sa, n):
    """Literal restatement of the reference's greedy merge loop
    (bvh.py:122-166): pop the smallest (SA, i); skip stale; defer merges at
    an odd offset of an even singleton run while supply == need; re-offer
    deferred items after every merge.  Returns the sorted left indices."""
    leaves = 1 << (n.bit_length() - 1)
    need = n - leaves
    if need == 0:
        return []
    heap = [(float(sa[i]), i) for i in range(n - 1)]
    heapq.heapify(heap)
    parked = []
    used = bytearray(n)
    starts = [0]
    ends = {0: n - 1}
    supply = n // 2
    lefts = []
    while need:
        if not heap:
            heap, parked = parked, []
            heapq.heapify(heap)
        key, i = heapq.heappop(heap)
        if used[i] or used[i + 1]:
            continue
        s = starts[bisect_right(starts, i) - 1]
        e = ends[s]
        m = e - s + 1
        j = i - s
        if (m % 2 == 0) and (j % 2 == 1) and supply - need <= 0:
            parked.append((key, i))
            continue
        used[i] = used[i + 1] = 1
        lefts.append(i)
        need -= 1
        supply += j // 2 + (m - j - 2) // 2 - m // 2
        k = bisect_right(starts, s) - 1
        del starts[k]
        del ends[s]
        if j > 0:
            starts.insert(k, s)
            ends[s] = i - 1
            k += 1
        if i + 2 <= e:
            starts.insert(k, i + 2)
            ends[i + 2] = e
        for item in parked:
            heapq.heappush(heap, item)
        parked = []
    return sorted(lefts)


_PAIRING = None


def greedy_pairs_fast(sa, n):
    """The same pairing as greedy_pairs (bvh.py:122-166) in O(n log n): the C
    restatement oracle/pairing.c (oracle_pair_greedy; see its header for the
    equivalence argument), loaded with ctypes.  Built by oracle/build.py
    (__graft_entry__.build()).  Returns the sorted left indices."""
    global _PAIRING
    import ctypes
    from pathlib import Path

    if _PAIRING is None:
        lib = Path(__file__).resolve().parent / "liboracle_pairing.so"
        if not lib.exists():
            from oracle import build as _b

            _b.build()
        h = ctypes.CDLL(str(lib))
        h.oracle_pair_greedy.restype = ctypes.c_int
        h.oracle_pair_greedy.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        _PAIRING = h
    sa = np.ascontiguousarray(sa, dtype=np.float64)
    is_left = np.zeros(n, dtype=np.uint8)
    if _PAIRING.oracle_pair_greedy(sa.ctypes.data_as(ctypes.c_void_p), n, is_left.ctypes.data_as(ctypes.c_void_p)):
        raise MemoryError("oracle_pair_greedy: out of memory")
    return np.flatnonzero(is_left)


def leaves_from_pairs(order, lefts, n):
    """Assemble (L, 2) leaf triangle ids, -1 for singles (bvh.py:168-181)."""
    L = 1 << (n.bit_length() - 1)
    is_left = np.zeros(n, dtype=bool)
    is_left[np.asarray(lefts, dtype=np.int64)] = True
    is_right = np.zeros(n, dtype=bool)
    is_right[1:] = is_left[:-1]
    firsts = np.flatnonzero(~is_right)
    assert len(firsts) == L
    out = np.full((L, 2), -1, dtype=np.int64)
    out[:, 0] = order[firsts]
    paired = is_left[firsts]
    out[paired, 1] = order[firsts[paired] + 1]
    return out


@dataclass
class Tree:
    """Implicit BFS full binary tree (bvh.py:184-239)."""

    node_min: np.ndarray
    node_max: np.ndarray
    leaf_tris: np.ndarray
    prim_order: np.ndarray
    depth: int

    @property
    def leaf_count(self):
        return len(self.leaf_tris)

    @property
    def n_nodes(self):
        return len(self.node_min)


def fill_boxes(tree: Tree, vertices, triangles):
    """Leaf unions then per-level child unions (bvh.py:242-264)."""
    P = triangle_points(vertices, triangles, tree.node_min.dtype)
    tlo = P.min(axis=1)
    thi = P.max(axis=1)
    L = tree.leaf_count
    a = tree.leaf_tris[:, 0]
    b = tree.leaf_tris[:, 1]
    two = b >= 0
    lo = tlo[a].copy()
    hi = thi[a].copy()
    lo[two] = np.minimum(tlo[a[two]], tlo[b[two]])
    hi[two] = np.maximum(thi[a[two]], thi[b[two]])
    tree.node_min[L - 1:] = lo
    tree.node_max[L - 1:] = hi
    for lvl in range(tree.depth - 1, -1, -1):
        f = (1 << lvl) - 1
        cf = (1 << (lvl + 1)) - 1
        cl = (1 << (lvl + 2)) - 1
        tree.node_min[f:cf] = np.minimum(tree.node_min[cf:cl:2], tree.node_min[cf + 1:cl:2])
        tree.node_max[f:cf] = np.maximum(tree.node_max[cf:cl:2], tree.node_max[cf + 1:cl:2])
    return tree


def build_tree(vertices, triangles, dtype=np.float64, lefts=None):
    """build_f12 (bvh.py:267-289).  `lefts` may supply a precomputed pairing
    (used at sizes where the literal greedy is too slow on a CPU)."""
    V = np.asarray(vertices, dtype=np.float64)
    T = np.asarray(triangles, dtype=np.int64)
    n = len(T)
    if n < 1:
        raise ValueError("cannot build a BVH over an empty mesh")
    _, order = morton_order(V, T)
    if lefts is None:
        P = V[T]
        lefts = greedy_pairs(pair_surface_areas(order, P.min(axis=1), P.max(axis=1)), n)
    leaf = leaves_from_pairs(order, lefts, n)
    L = len(leaf)
    nn = 2 * L - 1
    tree = Tree(np.empty((nn, 3), dtype=dtype), np.empty((nn, 3), dtype=dtype), leaf, order, L.bit_length() - 1)
    return fill_boxes(tree, V, T)


# ---------------------------------------------------------------------------
# traversal engine (query.py)
# ---------------------------------------------------------------------------

@dataclass
class Config:
    """EngineConfig defaults (query.py:67-75)."""

    front_cap: int = 262_144
    depth_cap: int = 5
    precision: int = 64
    workers: int = 1
    enhanced_bounds: bool = True
    culling: bool = True
    guarantee_witness: bool = False
    front_hard_cap: int = 16_777_216
    batch_size: int = 65_536

    @property
    def dtype(self):
        return np.float32 if self.precision == 32 else np.float64


class FrontOverflow(Exception):
    def __init__(self, candidates, front_in, cap):
        super().__init__(f"front expansion {candidates} from {front_in} > cap {cap}")
        self.candidates, self.front_in, self.cap = candidates, front_in, cap


def adaptive_k(n, cfg: Config, max_remaining):
    """query.py:266-284."""
    k = 1
    while k < cfg.depth_cap and k < max_remaining and (n << (2 * (k + 1))) < cfg.front_cap:
        k += 1
    return k


@dataclass
class Outcome:
    kind: str
    distance: float
    tri_a: int | None
    tri_b: int | None
    witness_distance: float | None
    point_a: np.ndarray | None
    point_b: np.ndarray | None
    iterations: list = field(default_factory=list)   # (k, front_in, front_out, culled, bound_after)
    expanded_pairs: int = 0
    narrow_pairs: int = 0


class _State:
    """Monotone bound + lexicographic witness cell (query.py:165-227)."""

    def __init__(self, kind, bound):
        import threading
        self.kind = kind
        self.bound = float(bound)
        self.w = None  # (dist, ta, tb, p, q)
        self.lock = threading.Lock()
        self.narrow = 0

    def offer_bound(self, v):
        v = float(v)
        with self.lock:
            if (v < self.bound) if self.kind == "min" else (v > self.bound):
                self.bound = v

    def offer_witness(self, d, ta, tb, p, q):
        d = float(d)
        with self.lock:
            w = self.w
            if w is None:
                better = True
            else:
                better = d < w[0] if self.kind == "min" else d > w[0]
                if not better and d == w[0]:
                    better = (ta, tb) < (w[1], w[2])
            if better:
                self.w = (d, int(ta), int(tb), np.array(p), np.array(q))


def _narrow(state: _State, ia, ib, pts_a, pts_b):
    """query.py:287-307."""
    if len(ia) == 0:
        return
    if state.kind == "min":
        d, p, q = tri_tri_min(pts_a[ia], pts_b[ib])
        k = np.lexsort((ib, ia, d))[0]
    else:
        d, p, q = tri_tri_max(pts_a[ia], pts_b[ib])
        k = np.lexsort((ib, ia, -d))[0]
    with state.lock:
        state.narrow += len(ia)
    state.offer_bound(d[k])
    state.offer_witness(d[k], ia[k], ib[k], p[k].astype(np.float64), q[k].astype(np.float64))


def _leaf_pairs(ta_rows, tb_rows):
    """Leaf pair -> 1..4 triangle pairs in (i, j) order (query.py:334-346)."""
    outa, outb = [], []
    for i in (0, 1):
        for j in (0, 1):
            ok = (ta_rows[:, i] >= 0) & (tb_rows[:, j] >= 0)
            outa.append(ta_rows[ok, i])
            outb.append(tb_rows[ok, j])
    return np.concatenate(outa), np.concatenate(outb)


def run_query(tree_a: Tree, tree_b: Tree, pts_a, pts_b, kind="min", cfg: Config | None = None, warm_pair=None):
    """_run_query (query.py:480-537) with expand_front (query.py:349-451).

    pts_a / pts_b: (m, 3, 3) triangle points in cfg.dtype."""
    cfg = cfg or Config()
    is_min = kind == "min"
    r = (tree_a.node_min[:1], tree_a.node_max[:1], tree_b.node_min[:1], tree_b.node_max[:1])
    if is_min:
        key0 = box_min_lower(*r)[0]
        b0 = (enhanced_min_upper if cfg.enhanced_bounds else box_max_upper)(*r)[0]
    else:
        key0 = box_max_upper(*r)[0]
        b0 = (enhanced_max_lower if cfg.enhanced_bounds else box_min_lower)(*r)[0]
    st = _State(kind, b0)
    out = Outcome(kind, 0.0, None, None, None, None, None)
    if warm_pair is not None:
        _narrow(st, np.asarray([warm_pair[0]]), np.asarray([warm_pair[1]]), pts_a, pts_b)
    fa = np.zeros(1, dtype=np.int64)
    fb = np.zeros(1, dtype=np.int64)
    da = db = 0
    La, Lb = tree_a.leaf_count, tree_b.leaf_count
    if tree_a.depth == 0 and tree_b.depth == 0:
        ia, ib = _leaf_pairs(tree_a.leaf_tris[fa], tree_b.leaf_tris[fb])
        _narrow(st, ia, ib, pts_a, pts_b)
        out.iterations.append((0, 1, 0, 0, st.bound))
        return _finish(out, st)
    pool = ThreadPoolExecutor(cfg.workers) if cfg.workers > 1 else None
    try:
        while len(fa):
            ra, rb = tree_a.depth - da, tree_b.depth - db
            k = adaptive_k(len(fa), cfg, max(ra, rb))
            ka, kb = min(k, ra), min(k, rb)
            sh = ka + kb
            n_in = len(fa)
            ncand = n_in << sh
            if ncand > cfg.front_hard_cap:
                raise FrontOverflow(ncand, n_in, cfg.front_hard_cap)
            leaves = k == max(ra, rb)
            out.expanded_pairs += ncand
            mb = (1 << kb) - 1

            def sweep(lo, hi, fa=fa, fb=fb, ka=ka, kb=kb, sh=sh, leaves=leaves, mb=mb):
                t = np.arange(lo, hi, dtype=np.int64)
                e = t >> sh
                off = t & ((1 << sh) - 1)
                na = ((fa[e] + 1) << ka) - 1 + (off >> kb)
                nb = ((fb[e] + 1) << kb) - 1 + (off & mb)
                amin, amax = tree_a.node_min[na], tree_a.node_max[na]
                bmin, bmax = tree_b.node_min[nb], tree_b.node_max[nb]
                key = (box_min_lower if is_min else box_max_upper)(amin, amax, bmin, bmax)
                bound = st.bound  # one snapshot per batch (query.py:396)
                if not cfg.culling:
                    keep = np.ones(len(t), dtype=bool)
                elif is_min:
                    keep = key <= bound if (leaves and cfg.guarantee_witness) else key < bound
                else:
                    keep = key >= bound if (leaves and cfg.guarantee_witness) else key > bound
                culled = int(len(t) - keep.sum())
                if leaves:
                    if keep.any():
                        ia, ib = _leaf_pairs(tree_a.leaf_tris[na[keep] - (La - 1)],
                                             tree_b.leaf_tris[nb[keep] - (Lb - 1)])
                        _narrow(st, ia, ib, pts_a, pts_b)
                    return culled, None
                if keep.any():
                    kept = (amin[keep], amax[keep], bmin[keep], bmax[keep])
                    if is_min:
                        f = enhanced_min_upper if cfg.enhanced_bounds else box_max_upper
                        st.offer_bound(f(*kept).min())
                    else:
                        f = enhanced_max_lower if cfg.enhanced_bounds else box_min_lower
                        st.offer_bound(f(*kept).max())
                return culled, (na[keep], nb[keep])

            spans = [(s, min(s + cfg.batch_size, ncand)) for s in range(0, ncand, cfg.batch_size)]
            res = list(pool.map(lambda s: sweep(*s), spans)) if (pool and len(spans) > 1) else [sweep(*s) for s in spans]
            culled = sum(r[0] for r in res)
            parts = [r[1] for r in res if r[1] is not None and len(r[1][0])]
            fa = np.concatenate([p[0] for p in parts]) if parts else np.empty(0, dtype=np.int64)
            fb = np.concatenate([p[1] for p in parts]) if parts else np.empty(0, dtype=np.int64)
            da += ka
            db += kb
            if len(fa) > cfg.front_hard_cap:
                raise FrontOverflow(len(fa), n_in, cfg.front_hard_cap)
            out.iterations.append((k, n_in, len(fa), culled, st.bound))
    finally:
        if pool is not None:
            pool.shutdown(wait=True)
    return _finish(out, st)


def _finish(out: Outcome, st: _State):
    out.distance = st.bound
    out.narrow_pairs = st.narrow
    if st.w is not None:
        out.witness_distance, out.tri_a, out.tri_b, out.point_a, out.point_b = st.w
    return out


def brute_force(pts_a, pts_b, kind="min", force=False):
    """All-pairs oracle with lexicographic tie-break (query.py:571-601)."""
    na, nb = len(pts_a), len(pts_b)
    total = na * nb
    if total == 0:
        raise ValueError("both meshes need at least one triangle")
    if total > BRUTE_LIMIT and not force:
        raise ValueError(f"brute force over {total} pairs exceeds {BRUTE_LIMIT}")
    best = None
    for s in range(0, total, 65_536):
        t = np.arange(s, min(s + 65_536, total), dtype=np.int64)
        ia, ib = t // nb, t % nb
        if kind == "min":
            d, p, q = tri_tri_min(pts_a[ia], pts_b[ib])
            k = np.lexsort((ib, ia, d))[0]
            cand = (float(d[k]), int(ia[k]), int(ib[k]))
            if best is None or cand < best[0]:
                best = (cand, p[k], q[k])
        else:
            d, p, q = tri_tri_max(pts_a[ia], pts_b[ib])
            k = np.lexsort((ib, ia, -d))[0]
            cand = (float(d[k]), int(ia[k]), int(ib[k]))
            if best is None or (-cand[0], cand[1], cand[2]) < (-best[0][0], best[0][1], best[0][2]):
                best = (cand, p[k], q[k])
    (d, ta, tb), p, q = best
    return d, ta, tb, p.astype(np.float64), q.astype(np.float64)
