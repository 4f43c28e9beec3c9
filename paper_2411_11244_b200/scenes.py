"""Deterministic two-mesh scenes (reference scenes.py:27-195) plus the
interlocked-ring workloads of BASELINE.json.

The four reference kinds reproduce the reference generators bit for bit
(same RNG streams, same arithmetic order; the UV sphere is vectorised, which
is elementwise identical).  New kinds:

  interlocked-rings   two tori of nu x nv quads (2 nu nv triangles each):
                      B = torus about y centred at (1, 0, 0); A = torus about
                      z moved by R_(1,1,0)(tilt) and `offset` -- a generic
                      interlock (the symmetric one makes the contact set a
                      curve and ties every witness).
  torus               a single torus pair helper used by the frame sequence.

`ring_frame_transforms(f)` gives the 1000-frame rotation sequence of config 3.
"""

from __future__ import annotations

import inspect
import math

import numpy as np

from .errors import SceneError
from .mesh import RigidTransform, TriangleMesh

_TAU = 2.0 * np.pi


def _soup(points: np.ndarray) -> TriangleMesh:
    """(m, 3, 3) corners -> unindexed soup (scenes.py:27-33)."""
    m = len(points)
    return TriangleMesh(points.reshape(m * 3, 3), np.arange(m * 3, dtype=np.int64).reshape(m, 3))


def _scatter(rng, n, center, spread, tri_size):
    """n small triangles with Gaussian centroids (scenes.py:36-41)."""
    cen = rng.normal(loc=center, scale=spread, size=(n, 3))
    cor = rng.normal(scale=tri_size, size=(n, 3, 3))
    cor -= cor.mean(axis=1, keepdims=True)
    return cen[:, None, :] + cor


def _gen_random_blobs(n: int = 200, seed: int = 0, gap: float = 0.5, spread: float = 1.0, tri_size: float = 0.05):
    if n < 1:
        raise SceneError("random-blobs: n must be >= 1")
    if gap < 0:
        raise SceneError("random-blobs: gap must be >= 0")
    sa, sb = np.random.SeedSequence(seed).spawn(2)
    ta = _scatter(np.random.default_rng(sa), n, (0.0, 0.0, 0.0), spread, tri_size)
    tb = _scatter(np.random.default_rng(sb), n, (0.0, 0.0, 0.0), spread, tri_size)
    tb[..., 0] += ta[..., 0].max() - tb[..., 0].min() + gap
    return _soup(ta), _soup(tb)


def _gen_intersecting_clusters(n: int = 1000, seed: int = 0, spread: float = 1.0, separation: float = 4.0,
                               tri_size: float = 0.05, point=(0.0, 0.0, 0.0)):
    """Two clusters plus one anchor triangle each through `point`, so the
    true minimum distance is exactly 0 (scenes.py:58-88)."""
    if n < 1:
        raise SceneError("intersecting-clusters: n must be >= 1")
    p0 = np.asarray(point, dtype=np.float64)
    sa, sb = np.random.SeedSequence(seed).spawn(2)
    half = 0.5 * separation * spread

    def one(rng, center):
        blob = _scatter(rng, max(n - 1, 1), center, spread, tri_size)
        u = rng.normal(size=3)
        v = rng.normal(size=3)
        anchor = np.stack([p0, p0 + tri_size * u, p0 + tri_size * v])
        return _soup(np.concatenate([blob, anchor[None]]) if n > 1 else anchor[None])

    return (one(np.random.default_rng(sa), p0 + np.array([-half, 0.0, 0.0])),
            one(np.random.default_rng(sb), p0 + np.array([half, 0.0, 0.0])))


def uv_sphere_points(lat: int, lon: int, radius: float, center) -> np.ndarray:
    """Corner points of a UV sphere, 2 lon (lat - 1) triangles, in the
    reference's order (scenes.py:91-120), vectorised."""
    c = np.asarray(center, dtype=np.float64)
    th = np.linspace(0.0, np.pi, lat + 1)[1:-1]
    ph = np.arange(lon) * (_TAU / lon)
    rs = radius * np.sin(th)
    rings = np.empty((len(th), lon, 3))
    rings[..., 0] = rs[:, None] * np.cos(ph)[None, :]
    rings[..., 1] = rs[:, None] * np.sin(ph)[None, :]
    rings[..., 2] = (radius * np.cos(th))[:, None]
    rings += c
    north = c + np.array([0.0, 0.0, radius])
    south = c + np.array([0.0, 0.0, -radius])
    j = np.arange(lon)
    k = (j + 1) % lon
    first, last = rings[0], rings[-1]
    caps = np.empty((lon, 2, 3, 3))
    caps[:, 0, 0] = north
    caps[:, 0, 1] = first[j]
    caps[:, 0, 2] = first[k]
    caps[:, 1, 0] = south
    caps[:, 1, 1] = last[k]
    caps[:, 1, 2] = last[j]
    a, b = rings[:-1], rings[1:]
    bands = np.empty((len(th) - 1, lon, 2, 3, 3))
    bands[:, :, 0, 0] = a[:, j]
    bands[:, :, 0, 1] = b[:, j]
    bands[:, :, 0, 2] = b[:, k]
    bands[:, :, 1, 0] = a[:, j]
    bands[:, :, 1, 1] = b[:, k]
    bands[:, :, 1, 2] = a[:, k]
    return np.concatenate([caps.reshape(-1, 3, 3), bands.reshape(-1, 3, 3)])


def _gen_nested_shells(lat: int = 8, lon: int = 12, r_inner: float = 0.8, r_outer: float = 1.2,
                       center=(0.0, 0.0, 0.0)):
    if lat < 2 or lon < 3:
        raise SceneError("nested-shells: need lat >= 2 and lon >= 3")
    if not 0 < r_inner < r_outer:
        raise SceneError("nested-shells: need 0 < r_inner < r_outer")
    return _soup(uv_sphere_points(lat, lon, r_inner, center)), _soup(uv_sphere_points(lat, lon, r_outer, center))


def _gen_offset_grids(res: int = 12, gap: float = 0.5, amp: float = 0.3, extent: float = 4.0, seed: int = 0):
    """Bumpy grids stacked in z with one pinned column forcing min == gap
    (scenes.py:131-159)."""
    if res < 2:
        raise SceneError("offset-grids: res must be >= 2")
    if gap <= 0:
        raise SceneError("offset-grids: gap must be > 0")
    rng = np.random.default_rng(seed)
    xs = np.linspace(0.0, extent, res)
    gx, gy = np.meshgrid(xs, xs, indexing="ij")
    ha = amp * rng.uniform(size=(res, res))
    hb = gap + amp + amp * rng.uniform(size=(res, res))
    pin = res // 2
    ha[pin, pin] = amp
    hb[pin, pin] = gap + amp
    idx = np.arange(res * res).reshape(res, res)
    a, b = idx[:-1, :-1].ravel(), idx[1:, :-1].ravel()
    c, d = idx[1:, 1:].ravel(), idx[:-1, 1:].ravel()
    tris = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)])

    def grid(h):
        return TriangleMesh(np.stack([gx, gy, h], axis=-1).reshape(res * res, 3), tris)

    return grid(ha), grid(hb)


# ---------------------------------------------------------------------------
# tori / rings (BASELINE.json configs 1-3, 5)
# ---------------------------------------------------------------------------
def torus_mesh(nu: int, nv: int, R: float = 1.0, r: float = 0.25, center=(0.0, 0.0, 0.0), axis: str = "z"):
    """Indexed torus: vertex i*nv + j at ((R + r cos v) cos u, (R + r cos v)
    sin u, r sin v), u = 2 pi i / nu, v = 2 pi j / nv; axis 'y' swaps to
    (x, z, y).  Triangles: every (a, b, c), then every (a, c, d) of the quad
    a=(i,j), b=(i+1,j), c=(i+1,j+1), d=(i,j+1), wrapping around."""
    if nu < 3 or nv < 3:
        raise SceneError("torus: need nu >= 3 and nv >= 3")
    if not 0 < r < R:
        raise SceneError("torus: need 0 < r < R")
    if axis not in ("y", "z"):
        raise SceneError("torus: axis must be 'y' or 'z'")
    u = np.arange(nu) * (_TAU / nu)
    v = np.arange(nv) * (_TAU / nv)
    ring = R + r * np.cos(v)
    V = np.empty((nu, nv, 3))
    V[..., 0] = ring[None, :] * np.cos(u)[:, None]
    V[..., 1] = ring[None, :] * np.sin(u)[:, None]
    V[..., 2] = (r * np.sin(v))[None, :]
    V = V.reshape(nu * nv, 3)
    if axis == "y":
        V = V[:, [0, 2, 1]]
    V = V + np.asarray(center, dtype=np.float64)
    i = np.arange(nu)[:, None]
    j = np.arange(nv)[None, :]
    i1 = (i + 1) % nu
    j1 = (j + 1) % nv
    a = (i * nv + j).ravel()
    b = (i1 * nv + j).ravel()
    c = (i1 * nv + j1).ravel()
    d = (i * nv + j1).ravel()
    tris = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)])
    return TriangleMesh(V, tris)


RING_TILT_AXIS = (1.0, 1.0, 0.0)
RING_OFFSET = (0.05, 0.03, 0.02)


def ring_pair_base(nu: int, nv: int, R: float = 1.0, r: float = 0.25):
    """(torus_z, torus_b): A before its placement, B in place."""
    return torus_mesh(nu, nv, R, r, (0.0, 0.0, 0.0), "z"), torus_mesh(nu, nv, R, r, (R, 0.0, 0.0), "y")


def _gen_interlocked_rings(nu: int = 100, nv: int = 50, R: float = 1.0, r: float = 0.25, tilt: float = 0.25,
                           offset=RING_OFFSET):
    """Configs 1/2: A = torus_z moved by R_(1,1,0)(tilt) + offset, B = torus
    about y through (R, 0, 0).  A's vertices are materialised on the host
    (V @ R^T + t, the reference's apply_transform)."""
    tz, tb = ring_pair_base(nu, nv, R, r)
    xf = RigidTransform.from_axis_angle(RING_TILT_AXIS, tilt, offset)
    va = tz.vertices @ xf.rotation.T + xf.translation
    return TriangleMesh(va, tz.triangles), tb


def ring_frame_transforms(f: int, n_frames: int = 1000, R: float = 1.0, base_tilt: float = 0.25):
    """Config 3 rotation sequence: theta_f = 2 pi 37 phi f / N
    (phi the golden ratio conjugate, an incommensurate spin),
    alpha_f = tilt + 0.05 sin(2 pi f / N).  Returns (xf_A, xf_B) relative to
    ring_pair_base(): A = R_(1,1,0)(alpha_f) R_z(theta_f) + offset, B spun by
    R_y(-theta_f) about its own axis through (R, 0, 0)."""
    phi = (math.sqrt(5.0) - 1.0) / 2.0
    theta = _TAU * 37.0 * phi * f / n_frames
    alpha = base_tilt + 0.05 * math.sin(_TAU * f / n_frames)
    ra = RigidTransform.from_axis_angle(RING_TILT_AXIS, alpha).rotation @ RigidTransform.from_axis_angle(
        (0.0, 0.0, 1.0), theta).rotation
    xf_a = RigidTransform(ra, RING_OFFSET)
    rb = RigidTransform.from_axis_angle((0.0, 1.0, 0.0), -theta).rotation
    c = np.array([R, 0.0, 0.0])
    xf_b = RigidTransform(rb, c - rb @ c)
    return xf_a, xf_b


_GENERATORS = {
    "random-blobs": _gen_random_blobs,
    "intersecting-clusters": _gen_intersecting_clusters,
    "nested-shells": _gen_nested_shells,
    "offset-grids": _gen_offset_grids,
    "interlocked-rings": _gen_interlocked_rings,
}


def scene_kinds() -> list:
    return sorted(_GENERATORS)


def gen_scene(kind: str, params: dict | None = None):
    """(mesh A, mesh B) for a scene kind (scenes.py:174-195)."""
    if kind not in _GENERATORS:
        raise SceneError(f"unknown scene kind {kind!r}; known kinds: {', '.join(scene_kinds())}")
    gen = _GENERATORS[kind]
    params = dict(params or {})
    allowed = set(inspect.signature(gen).parameters)
    unknown = set(params) - allowed
    if unknown:
        raise SceneError(f"{kind}: unknown parameter(s) {sorted(unknown)}; accepted: {sorted(allowed)}")
    try:
        return gen(**params)
    except SceneError:
        raise
    except (TypeError, ValueError) as exc:
        raise SceneError(f"{kind}: invalid parameters: {exc}") from None
