"""Triangle meshes, rigid motion and OBJ ingest (reference mesh.py:21-163).

`TriangleMesh` keeps the reference's host contract (float64 / int64
read-only arrays, same validation errors) and adds a device view: the base
vertices are uploaded once and cached on the object.  `apply_transform` is
lazy on the device: the moved mesh shares the base upload and carries the
rigid transform, which the refit and exact kernels apply on the fly (no
per-frame vertex upload), in numpy dgemm's arithmetic (bit for bit the
reference's `V @ R.T + t`).  A transform of an already-moved mesh
materialises that mesh with the reference formula first (the reference
applies transforms one by one; a composed transform could differ by an ulp).
Reading `.vertices` of a moved mesh materialises it on the host the same way.
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from . import _lib
from .errors import DegenerateTriangleError, ObjParseError

_IDENTITY = np.eye(3)


def _validated(vertices, triangles):
    verts = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64))
    tris = np.ascontiguousarray(np.asarray(triangles, dtype=np.int64))
    if verts.ndim != 2 or verts.shape[1] != 3:
        raise ValueError(f"vertices must be (n, 3), got {verts.shape}")
    if tris.size == 0:
        tris = tris.reshape(0, 3)
    if tris.ndim != 2 or tris.shape[1] != 3:
        raise ValueError(f"triangles must be (m, 3), got {tris.shape}")
    if tris.size:
        if tris.min() < 0 or tris.max() >= len(verts):
            raise ValueError("triangle index out of range")
        bad = (tris[:, 0] == tris[:, 1]) | (tris[:, 1] == tris[:, 2]) | (tris[:, 0] == tris[:, 2])
        if bad.any():
            raise DegenerateTriangleError([(int(i), tuple(int(v) for v in tris[i])) for i in np.flatnonzero(bad)])
    verts.setflags(write=False)
    tris.setflags(write=False)
    return verts, tris


class TriangleMesh:
    """Immutable indexed triangle soup (mesh.py:21-66).

    vertices: (n, 3) float64, triangles: (m, 3) int64, both read-only."""

    __slots__ = ("_vertices", "_triangles", "_root", "_chain", "_rot", "_trans", "_dev", "_gview", "__weakref__")

    def __init__(self, vertices, triangles):
        self._vertices, self._triangles = _validated(vertices, triangles)
        self._root = self
        self._chain = ()          # host transform still to apply to root.vertices (at most one)
        self._rot = None          # device transform (None = identity)
        self._trans = None
        self._dev = None
        self._gview = None

    # -- lazily moved mesh (apply_transform) ------------------------------
    @classmethod
    def _trusted(cls, vertices: np.ndarray, triangles: np.ndarray) -> "TriangleMesh":
        """A mesh over already-validated read-only arrays (no O(m) checks)."""
        out = cls.__new__(cls)
        out._vertices, out._triangles = vertices, triangles
        out._root = out
        out._chain = ()
        out._rot = out._trans = None
        out._dev = out._gview = None
        return out

    @classmethod
    def _moved(cls, src: "TriangleMesh", xf: "RigidTransform") -> "TriangleMesh":
        if src._chain:
            # a transform of an already-moved mesh: the reference applies the
            # transforms one by one (mesh.py:104), and one composed (R, t) on
            # the device can differ from that by an ulp -- so the moved mesh's
            # vertices are materialised with the reference formula and become
            # the new base (one upload), keeping the device bit-exact
            src = cls._trusted(src.vertices, src._triangles)
        out = cls.__new__(cls)
        out._vertices = None
        out._triangles = src._triangles
        out._root = src._root
        out._chain = src._chain + (xf,)
        R0 = _IDENTITY if src._rot is None else src._rot
        t0 = np.zeros(3) if src._trans is None else src._trans
        out._rot = xf.rotation @ R0
        out._trans = xf.rotation @ t0 + xf.translation
        out._dev = None
        out._gview = None
        return out

    def deformed(self, vertices) -> "TriangleMesh":
        """Same connectivity, new base vertex positions (deformable meshes,
        SURVEY.md 8(f) row 2): `refit(bvh, mesh.deformed(V))` keeps the tree's
        topology and re-stages the vertices on the device.  `vertices` is an
        (n_vertices, 3) array, or a float64 CUDA tensor of that shape used in
        place -- a simulation that keeps its vertices on the GPU never sends
        them through the host (`.vertices` downloads them only if read).
        Transforms applied to `self` are not carried over."""
        root = self._root
        out = TriangleMesh.__new__(TriangleMesh)
        out._triangles = root._triangles
        out._root = out
        out._chain = ()
        out._rot = out._trans = None
        out._gview = None
        torch = _lib.torch()
        if isinstance(vertices, torch.Tensor) and vertices.is_cuda:
            if tuple(vertices.shape) != (root.n_vertices, 3) or vertices.dtype != torch.float64:
                raise ValueError(f"deformed vertices must be a ({root.n_vertices}, 3) float64 tensor, "
                                 f"got {tuple(vertices.shape)} {vertices.dtype}")
            out._vertices = None
            out._dev = (vertices.contiguous(), root._upload()[1])
            return out
        v = np.array(vertices, dtype=np.float64, order="C")
        if v.shape != (root.n_vertices, 3):
            raise ValueError(f"deformed vertices must be ({root.n_vertices}, 3), got {v.shape}")
        v.setflags(write=False)
        out._vertices = v
        out._dev = None
        if root._dev is not None:  # share the uploaded connectivity, send only the vertices
            out._dev = (torch.from_numpy(v.copy()).to(root._dev[1].device), root._dev[1])
        return out

    def _host_vertices(self) -> np.ndarray:
        """Base vertices on the host (downloaded once for a device-made mesh)."""
        root = self._root
        if root._vertices is None:
            v = root._dev[0].cpu().numpy()
            v.setflags(write=False)
            root._vertices = v
        return root._vertices

    @property
    def vertices(self) -> np.ndarray:
        if self._vertices is None:
            v = self._host_vertices()
            for xf in self._chain:
                v = v @ xf.rotation.T + xf.translation  # mesh.py:104, transform by transform
            v = np.ascontiguousarray(v)
            v.setflags(write=False)
            self._vertices = v
        return self._vertices

    @property
    def triangles(self) -> np.ndarray:
        return self._triangles

    @property
    def n_triangles(self) -> int:
        return len(self._triangles)

    @property
    def n_vertices(self) -> int:
        root = self._root
        return len(root._vertices) if root._vertices is not None else int(root._dev[0].shape[0])

    def triangle_points(self, dtype=np.float64) -> np.ndarray:
        """(m, 3, 3) corners: cast first, then gather (mesh.py:64-66)."""
        return self.vertices.astype(dtype, copy=False)[self._triangles]

    def __repr__(self) -> str:
        return f"TriangleMesh(n_vertices={self.n_vertices}, n_triangles={self.n_triangles})"

    # -- device view --------------------------------------------------------
    def _upload(self):
        """Upload the root's float64 vertices and int32 indices once."""
        root = self._root
        if root._dev is None:
            torch = _lib.torch()
            dev = _lib.device()
            if len(root._triangles) >= 2**31 or len(root._vertices) >= 2**31:
                raise ValueError("meshes above 2^31 vertices/triangles are not supported")
            vt = torch.from_numpy(np.array(root._vertices, dtype=np.float64, order="C")).to(dev)
            tr = torch.from_numpy(root._triangles.astype(np.int32)).to(dev)
            root._dev = (vt, tr)
        return root._dev

    def device_view(self) -> _lib.GdMesh:
        """C view (include/gdist.h GdMesh); cached -- the mesh is immutable."""
        if self._gview is not None:
            _lib.check_device(self._root._dev[0], "mesh")
            return self._gview
        vt, tr = self._upload()
        _lib.check_device(vt, "mesh")
        g = _lib.GdMesh()
        g.vtx = vt.data_ptr()
        g.tri = tr.data_ptr()
        g.nv = vt.shape[0]
        g.m = tr.shape[0]
        # the host BLAS's transform order, also on unmoved meshes: the exact
        # pass is instantiated per order (a frame graph captured with an
        # unmoved mesh replays moved ones)
        g.xf_order = blas_order()
        if self._rot is None:
            g.rot[:] = [1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0]
            g.trans[:] = [0.0, 0.0, 0.0]
            g.has_xf = 0
        else:
            g.rot[:] = [float(x) for x in self._rot.reshape(9)]
            g.trans[:] = [float(x) for x in self._trans.reshape(3)]
            g.has_xf = 1
        self._gview = g
        return g

    def _geometry_key(self):
        """Identity of the geometry the device sees (root + transform)."""
        if self._rot is None:
            return (id(self._root), None)
        return (id(self._root), self._rot.tobytes() + self._trans.tobytes())


def relative_mesh(mesh_a: "TriangleMesh", mesh_b: "TriangleMesh") -> "TriangleMesh":
    """mesh_a's base geometry under A's transform expressed in B's local
    frame (Rb^T Ra, Rb^T (ta - tb); gd_mesh_relative, the transform a
    GdConfig.frame = 1 query applies to A)."""
    L = _lib.lib()
    out = _lib.GdMesh()
    _lib.check(L.gd_mesh_relative(C.byref(mesh_a.device_view()), C.byref(mesh_b.device_view()), C.byref(out)),
               "mesh_relative")
    rot = np.array(out.rot[:], dtype=np.float64).reshape(3, 3)
    trans = np.array(out.trans[:], dtype=np.float64)
    return TriangleMesh._moved(mesh_a._root, RigidTransform(rot, trans))


class RigidTransform:
    """Rotation (3x3 orthonormal within 1e-6) then translation (mesh.py:69-99)."""

    __slots__ = ("rotation", "translation")

    def __init__(self, rotation=None, translation=None):
        rot = np.asarray(np.eye(3) if rotation is None else rotation, dtype=np.float64).reshape(3, 3).copy()
        t = np.asarray(np.zeros(3) if translation is None else translation, dtype=np.float64).reshape(3).copy()
        if not np.allclose(rot @ rot.T, np.eye(3), atol=1e-6):
            raise ValueError("rotation matrix is not orthonormal within 1e-6")
        rot.setflags(write=False)
        t.setflags(write=False)
        object.__setattr__(self, "rotation", rot)
        object.__setattr__(self, "translation", t)

    def __setattr__(self, name, value):
        raise AttributeError("RigidTransform is immutable")

    @classmethod
    def from_axis_angle(cls, axis, angle_rad: float, translation=(0.0, 0.0, 0.0)) -> "RigidTransform":
        """Rodrigues: c I + s [a]x + (1 - c) a a^T (mesh.py:86-99)."""
        a = np.asarray(axis, dtype=np.float64)
        n = np.linalg.norm(a)
        if n == 0.0:
            raise ValueError("rotation axis must be nonzero")
        a = a / n
        c, s = math.cos(angle_rad), math.sin(angle_rad)
        skew = np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])
        rot = c * np.eye(3) + s * skew + (1.0 - c) * np.outer(a, a)
        return cls(rotation=rot, translation=np.asarray(translation, dtype=np.float64))

    def compose(self, inner: "RigidTransform") -> "RigidTransform":
        """self o inner: v -> R_self (R_inner v + t_inner) + t_self."""
        return RigidTransform(self.rotation @ inner.rotation, self.rotation @ inner.translation + self.translation)

    def __repr__(self) -> str:
        return f"RigidTransform(rotation={self.rotation.tolist()}, translation={self.translation.tolist()})"


_BLAS_ORDER = None


def _fma(a: float, b: float, c: float) -> float:
    """Correctly rounded a * b + c (exact rational arithmetic; for probes)."""
    from fractions import Fraction

    return float(Fraction(a) * Fraction(b) + Fraction(c))


def blas_order() -> int:
    """Operation order of numpy's `V @ R.T` on this host (GdMesh.xf_order):
    probed once on random rows against the candidate orders, so the device
    transform reproduces the reference's float64 vertices bit for bit
    whatever BLAS numpy links.  0 (OpenBLAS dgemm on this image) when no
    candidate matches -- then moved vertices agree to an ulp, not bitwise."""
    global _BLAS_ORDER
    if _BLAS_ORDER is not None:
        return _BLAS_ORDER
    rng = np.random.default_rng(12345)
    V = rng.normal(size=(257, 3)) * 10.0 ** rng.uniform(-3, 3, size=(257, 1))
    R = rng.normal(size=(3, 3))
    got = V @ R.T
    cands = {
        0: lambda r, v: _fma(r[2], v[2], _fma(r[1], v[1], r[0] * v[0])),
        1: lambda r, v: (r[0] * v[0] + r[1] * v[1]) + r[2] * v[2],
        2: lambda r, v: _fma(r[0], v[0], _fma(r[1], v[1], r[2] * v[2])),
    }
    order = 0
    for k, f in cands.items():
        if all(got[i, j] == f([float(x) for x in R[j]], [float(x) for x in V[i]])
               for i in range(len(V)) for j in range(3)):
            order = k
            break
    _BLAS_ORDER = order
    return order


def apply_transform(mesh: TriangleMesh, xf: RigidTransform) -> TriangleMesh:
    """Map every vertex v to R v + t; topology shared (mesh.py:102-105).
    O(1): the device applies the transform inside refit / the exact pass."""
    return TriangleMesh._moved(mesh, xf)


def load_obj(path) -> TriangleMesh:
    """Wavefront OBJ subset with the reference's semantics (mesh.py:108-163):
    `v` and `f` records, `#` comments, polygons fan-triangulated, negative
    indices relative to the vertex count at the point of use, everything
    else ignored.  Parsed natively (csrc/obj.cpp, host C++); a malformed
    record raises ObjParseError(path, line_no, message)."""
    path = os.fspath(path)
    L = _lib.lib()
    h = C.c_void_p()
    nv, nt, line = C.c_int64(), C.c_int64(), C.c_int64()
    st = L.gd_obj_open(os.fsencode(path), C.byref(h), C.byref(nv), C.byref(nt), C.byref(line))
    if st != 0:
        msg = L.gd_last_error().decode("utf-8", "replace")
        if line.value == 0:
            raise OSError(msg)
        raise ObjParseError(path, int(line.value), msg)
    try:
        verts = np.empty((nv.value, 3), dtype=np.float64)
        tris = np.empty((nt.value, 3), dtype=np.int64)
        L.gd_obj_read(h, verts.ctypes.data_as(C.c_void_p), tris.ctypes.data_as(C.c_void_p))
    finally:
        L.gd_obj_close(h)
    return TriangleMesh(verts, tris)
