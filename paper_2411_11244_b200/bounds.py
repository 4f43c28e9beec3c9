"""AABB distance bounds and the exact triangle narrow phase (reference
bounds.py:47-348), evaluated by libgdist's exact batch kernels.

conventional  aabb_min_lower / aabb_max_upper  (Eqs. 5-8)
enhanced      enhanced_min_upper / enhanced_max_lower (Eqs. 9-10): the 36
              face-rectangle pairs reduce to a closed form (9 sums per box
              pair) that is bitwise equal to the pairwise evaluation because
              each per-axis term depends on at most one face side and
              IEEE rounding is monotone.
narrow phase  tri_tri_min (9 edge-edge Lumelsky pairs, 6 point-triangle
              Voronoi walks, transversal pierce test) / tri_tri_max (9
              vertex pairs), in the reference's operation order.
Every `batch_*` accepts float32 or float64 arrays and computes in that type.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .bvh import Aabb
from .errors import TightnessError

_WHICH = {"min_lower": 0, "max_upper": 1, "enhanced_min_upper": 2, "enhanced_max_lower": 3}


def _prec(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return 32
    if dt == np.float64:
        return 64
    raise TypeError(f"unsupported dtype {dt}")


def _device_bounds(which: int, amin, amax, bmin, bmax) -> np.ndarray:
    arrs = [np.ascontiguousarray(a) for a in np.broadcast_arrays(
        np.asarray(amin), np.asarray(amax), np.asarray(bmin), np.asarray(bmax))]
    dt = np.result_type(*arrs)
    if dt not in (np.float32, np.float64):
        dt = np.dtype(np.float64)
    arrs = [np.ascontiguousarray(a, dtype=dt).reshape(-1, 3) for a in arrs]
    n = len(arrs[0])
    if n == 0:
        return np.empty(0, dtype=dt)
    torch = _lib.torch()
    dev = _lib.device()
    ts = [torch.from_numpy(a).to(dev) for a in arrs]
    out = torch.empty(n, dtype=ts[0].dtype, device=dev)
    _lib.check(_lib.lib().gd_box_bounds_batch(which, _prec(dt), *[_lib.ptr(t) for t in ts], n, _lib.ptr(out),
                                              _lib.stream_ptr()), "box_bounds")
    return out.cpu().numpy()


def _device_tri_tri(kind: str, t1, t2):
    t1 = np.asarray(t1)
    t2 = np.asarray(t2)
    dt = np.result_type(t1, t2)
    if dt not in (np.float32, np.float64):
        dt = np.dtype(np.float64)
    t1 = np.ascontiguousarray(t1, dtype=dt).reshape(-1, 3, 3)
    t2 = np.ascontiguousarray(t2, dtype=dt).reshape(-1, 3, 3)
    n = len(t1)
    if n == 0:
        return np.empty(0, dtype=dt), np.empty((0, 3), dtype=dt), np.empty((0, 3), dtype=dt)
    torch = _lib.torch()
    dev = _lib.device()
    a = torch.from_numpy(t1).to(dev)
    b = torch.from_numpy(t2).to(dev)
    d = torch.empty(n, dtype=a.dtype, device=dev)
    p = torch.empty((n, 3), dtype=a.dtype, device=dev)
    q = torch.empty((n, 3), dtype=a.dtype, device=dev)
    _lib.check(_lib.lib().gd_tri_tri_batch(1 if kind == "max" else 0, _prec(dt), _lib.ptr(a), _lib.ptr(b), n,
                                           _lib.ptr(d), _lib.ptr(p), _lib.ptr(q), _lib.stream_ptr()), "tri_tri")
    return d.cpu().numpy(), p.cpu().numpy(), q.cpu().numpy()


# -- batch kernels (bounds.py:47-101, 245-330) --------------------------------
def batch_min_lower(amin, amax, bmin, bmax) -> np.ndarray:
    """Exact box-box minimum distance (Eq. 5)."""
    return _device_bounds(0, amin, amax, bmin, bmax)


def batch_max_upper(amin, amax, bmin, bmax) -> np.ndarray:
    """Exact box-box maximum distance (Eqs. 6-7)."""
    return _device_bounds(1, amin, amax, bmin, bmax)


def batch_enhanced_min_upper(amin, amax, bmin, bmax) -> np.ndarray:
    """Upper bound on the content minimum for tight boxes (Eq. 9)."""
    return _device_bounds(2, amin, amax, bmin, bmax)


def batch_enhanced_max_lower(amin, amax, bmin, bmax) -> np.ndarray:
    """Lower bound on the content maximum for tight boxes (Eq. 10)."""
    return _device_bounds(3, amin, amax, bmin, bmax)


def batch_tri_tri_min(t1, t2):
    """Exact min distance + witness points for (N, 3, 3) batches."""
    return _device_tri_tri("min", t1, t2)


def batch_tri_tri_max(t1, t2):
    """Exact max distance + witness vertices for (N, 3, 3) batches."""
    return _device_tri_tri("max", t1, t2)


# -- scalar API (bounds.py:104-348) --------------------------------------------
def _pair(a: Aabb, b: Aabb):
    return a.min[None, :], a.max[None, :], b.min[None, :], b.max[None, :]


def aabb_min_lower(a: Aabb, b: Aabb) -> float:
    """Exact minimum distance between two boxes."""
    return float(batch_min_lower(*_pair(a, b))[0])


def aabb_max_upper(a: Aabb, b: Aabb) -> float:
    """Exact maximum distance between two boxes (the conventional upper
    bound on the content minimum)."""
    return float(batch_max_upper(*_pair(a, b))[0])


def _require_tight(a: Aabb, b: Aabb, op: str) -> None:
    if not (a.tight and b.tight):
        raise TightnessError(f"{op} requires both boxes tight (got {a.tight}, {b.tight})")


def enhanced_min_upper(a: Aabb, b: Aabb) -> float:
    _require_tight(a, b, "enhanced_min_upper")
    return float(batch_enhanced_min_upper(*_pair(a, b))[0])


def enhanced_max_lower(a: Aabb, b: Aabb) -> float:
    _require_tight(a, b, "enhanced_max_lower")
    return float(batch_enhanced_max_lower(*_pair(a, b))[0])


def tri_tri_min(t1, t2):
    """Exact minimum distance between two triangles + witness points."""
    d, p, q = batch_tri_tri_min(np.asarray(t1, dtype=np.float64)[None], np.asarray(t2, dtype=np.float64)[None])
    return float(d[0]), p[0], q[0]


def tri_tri_max(t1, t2):
    """Exact maximum distance between two triangles + the vertex pair."""
    d, p, q = batch_tri_tri_max(np.asarray(t1, dtype=np.float64)[None], np.asarray(t2, dtype=np.float64)[None])
    return float(d[0]), p[0], q[0]


def tri_tri_fast(kind: str, t1, t2) -> np.ndarray:
    """The traversal's float32 (FMA-contracted) narrow phase, distances only;
    exposed for the error-bound tests.  kind "min-lb": the conditioning-aware
    lower bound of the float32 min distance that the exact band windows on."""
    a = np.ascontiguousarray(np.asarray(t1, dtype=np.float32).reshape(-1, 3, 3))
    b = np.ascontiguousarray(np.asarray(t2, dtype=np.float32).reshape(-1, 3, 3))
    n = len(a)
    torch = _lib.torch()
    dev = _lib.device()
    ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.check(_lib.lib().gd_tri_tri_fast({"min": 0, "max": 1, "min-lb": 2}[kind], _lib.ptr(ta), _lib.ptr(tb), n,
                                          _lib.ptr(d),
                                          _lib.stream_ptr()), "tri_tri_fast")
    return d.cpu().numpy()
