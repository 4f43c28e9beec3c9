"""f12-BVH on the device (reference bvh.py:36-335).

`build_f12` runs Morton codes + radix sort on the GPU, the exact greedy
power-of-two pairing (host C++, O(n log n)) and a device refit.  The tree
lives in device memory (traversal boxes, leaf layout, float32 vertices);
`node_min` / `node_max` are exported on demand with the reference's dtype
semantics, `leaf_tris` / `prim_order` are host arrays with the reference's
meaning.  `refit` recomputes every box on the device for a moved mesh.
"""

from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from . import _lib
from .errors import TopologyMismatchError
from .mesh import TriangleMesh

_MORTON_BITS = 21


class Aabb:
    """Axis-aligned box; `tight` asserts every face touches the contents
    (bvh.py:36-55)."""

    __slots__ = ("min", "max", "tight")

    def __init__(self, min, max, tight: bool = False):  # noqa: A002 - reference field names
        lo = np.asarray(min, dtype=np.float64).reshape(3).copy()
        hi = np.asarray(max, dtype=np.float64).reshape(3).copy()
        if not (lo <= hi).all():
            raise ValueError(f"invalid box: min {lo} exceeds max {hi}")
        object.__setattr__(self, "min", lo)
        object.__setattr__(self, "max", hi)
        object.__setattr__(self, "tight", bool(tight))

    def __setattr__(self, name, value):
        raise AttributeError("Aabb is immutable")

    @classmethod
    def from_points(cls, points) -> "Aabb":
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        return cls(pts.min(axis=0), pts.max(axis=0), tight=True)

    def __repr__(self) -> str:
        return f"Aabb(min={self.min.tolist()}, max={self.max.tolist()}, tight={self.tight})"


class F12Bvh:
    """Full binary AABB tree in implicit BFS storage (bvh.py:184-239).

    Device state (include/gdist.h GdBvh): `_box` ((n_nodes + 1) x 6 float32
    traversal boxes, node i at slot i + 1), `_leaf_rec` (L x 8 int32 leaf
    records), `_vtx32` (float32 copy of the base vertices of `_staged`, in
    first-use order), `_vmap` (staged slot of each mesh vertex), and the
    streamed per-leaf vertex sets `_leaf_vtx`, `_leaf_x`, `_leaf_xvtx`, and
    `_leaf_tri` (both triangles of every leaf, for the narrow phase).
    Host state: `leaf_tris` (L, 2) int64, `prim_order` (m,) int64, `depth`.
    """

    def __init__(self, node_min=None, node_max=None, leaf_tris=None, prim_order=None, depth=None, tight=True,
                 dtype=np.float64):
        self.leaf_tris = None if leaf_tris is None else np.asarray(leaf_tris, dtype=np.int64)
        self.prim_order = None if prim_order is None else np.asarray(prim_order, dtype=np.int64)
        self.depth = None if depth is None else int(depth)
        self.tight = tight
        self._dtype = np.dtype(dtype if node_min is None else np.asarray(node_min).dtype)
        self._host_boxes = None
        if node_min is not None:
            self._host_boxes = (np.asarray(node_min), np.asarray(node_max))
        self._box = self._leaf_rec = self._vtx32 = self._vmap = None
        self._leaf_vtx = self._leaf_x = self._leaf_xvtx = self._leaf_tri = None
        self._mesh = None            # mesh of the last device refit
        self._staged = None          # root mesh whose base vertices are in _vtx32
        self._layout_tris = None     # index buffer the leaf records were built from
        self._export_cache = None

    # -- reference-compatible accessors ------------------------------------
    @property
    def n_nodes(self) -> int:
        return 2 * self.leaf_count - 1

    @property
    def leaf_count(self) -> int:
        return len(self.leaf_tris)

    @property
    def dtype(self) -> np.dtype:
        return self._dtype

    @property
    def n_triangles(self) -> int:
        return len(self.prim_order)

    def _export(self):
        if self._host_boxes is not None and self._box is None:
            return self._host_boxes
        if self._export_cache is None:
            if self._mesh is None:
                raise RuntimeError("tree has no device boxes yet (build or refit it)")
            torch = _lib.torch()
            prec = 32 if self._dtype == np.float32 else 64
            tdt = torch.float32 if prec == 32 else torch.float64
            nmin = _lib.empty((self.n_nodes, 3), tdt)
            nmax = _lib.empty((self.n_nodes, 3), tdt)
            g = self._mesh.device_view()
            v = self.device_view()
            _lib.check(_lib.lib().gd_export_boxes(C.byref(g), C.byref(v), prec, _lib.ptr(nmin), _lib.ptr(nmax),
                                                  _lib.stream_ptr()), "export_boxes")
            self._export_cache = (nmin.cpu().numpy(), nmax.cpu().numpy())
        return self._export_cache

    @property
    def node_min(self) -> np.ndarray:
        return self._export()[0]

    @property
    def node_max(self) -> np.ndarray:
        return self._export()[1]

    def is_leaf(self, node: int) -> bool:
        return node >= self.leaf_count - 1

    def leaf_rank(self, node: int) -> int:
        return node - (self.leaf_count - 1)

    def leaf_prims(self, rank: int) -> tuple:
        t0, t1 = self.leaf_tris[rank]
        return (int(t0),) if t1 < 0 else (int(t0), int(t1))

    def node_box(self, node: int) -> Aabb:
        return Aabb(self.node_min[node], self.node_max[node], tight=self.tight)

    def to_debug_dict(self) -> dict:
        return {
            "depth": self.depth,
            "leaf_count": self.leaf_count,
            "node_min": self.node_min.astype(np.float64).tolist(),
            "node_max": self.node_max.astype(np.float64).tolist(),
            "leaf_tris": self.leaf_tris.tolist(),
            "prim_order": self.prim_order.tolist(),
        }

    def dump_json(self, path) -> None:
        with open(os.fspath(path), "w", encoding="utf-8") as fh:
            json.dump(self.to_debug_dict(), fh, indent=1)

    # -- device ------------------------------------------------------------
    def _alloc(self, nv: int):
        torch = _lib.torch()
        L = self.leaf_count
        self._box = _lib.empty(2 * L * 6, torch.float32)  # slot 0 = padding (gdist.h)
        self._leaf_rec = _lib.empty(L * 8, torch.int32)
        self._vtx32 = _lib.empty(max(nv, 1) * 4, torch.float32)
        self._vmap = _lib.empty(max(nv, 1), torch.int32)
        self._leaf_vtx = _lib.empty(3 * L * 4, torch.float32)
        self._leaf_x = _lib.torch().zeros(2 * ((L + 31) // 32) + 1 + 2 * (L >> 16) + 5, dtype=torch.int32,
                                          device=_lib.device())
        self._leaf_xvtx = _lib.empty(2 * L * 4, torch.float32)
        self._leaf_tri = _lib.empty(L * 20, torch.float32)

    def device_view(self) -> _lib.GdBvh:
        """C view (include/gdist.h GdBvh), cached until a buffer changes."""
        _lib.check_device(self._box, "BVH")
        nv = self._vtx32.numel() // 4 if self._mesh is None else self._mesh.n_vertices
        gv = getattr(self, "_gview", None)
        if gv is not None and gv.vtx32 == self._vtx32.data_ptr() and gv.nv == nv:
            return gv
        g = _lib.GdBvh()
        g.box = self._box.data_ptr()
        g.leaf_rec = self._leaf_rec.data_ptr()
        g.vtx32 = self._vtx32.data_ptr()
        g.vmap = self._vmap.data_ptr()
        g.leaf_vtx = self._leaf_vtx.data_ptr()
        g.leaf_x = self._leaf_x.data_ptr()
        g.leaf_xvtx = self._leaf_xvtx.data_ptr()
        g.leaf_tri = self._leaf_tri.data_ptr()
        g.leaf_count = self.leaf_count
        g.n_tris = len(self.prim_order)
        g.nv = nv
        g.depth = self.depth
        self._gview = g
        return g

    def _ensure_layout(self, mesh: TriangleMesh):
        """Device leaf records for a tree given as host arrays (the reference
        allows constructing F12Bvh directly, bvh.py:184-199)."""
        if self._box is not None:
            return
        self._alloc(mesh.n_vertices)
        counts = 1 + (self.leaf_tris[:, 1] >= 0)
        first = np.zeros(self.leaf_count + 1, dtype=np.int64)
        np.cumsum(counts, out=first[1:])
        # leaf_tris must list Morton-order neighbours: slot order == prim_order
        if not np.array_equal(self.prim_order[first[:-1]], self.leaf_tris[:, 0]):
            raise ValueError("leaf_tris is not consistent with prim_order")
        self._write_records(mesh)
        self._layout_tris = mesh.triangles

    def _write_records(self, mesh: TriangleMesh):
        """Leaf records {a0, a1, a2, b0, b1, b2, tri0, tri1} (gdist.h) from
        leaf_tris and mesh.triangles (a single repeats triangle 0), then the
        device layout pass renumbers their vertices by first use and stages
        the mesh's vertices (gd_bvh_layout)."""
        t0 = self.leaf_tris[:, 0]
        t1 = self.leaf_tris[:, 1]
        tris = mesh.triangles
        rec = np.empty((self.leaf_count, 8), dtype=np.int32)
        rec[:, 0:3] = tris[t0]
        rec[:, 3:6] = tris[np.where(t1 >= 0, t1, t0)]
        rec[:, 6] = t0
        rec[:, 7] = t1
        torch = _lib.torch()
        nv = max(mesh.n_vertices, 1)
        if self._vtx32.numel() != nv * 4:
            self._vtx32 = _lib.empty(nv * 4, torch.float32)
            self._vmap = _lib.empty(nv, torch.int32)
        self._leaf_rec.copy_(torch.from_numpy(rec.reshape(-1)))
        L = _lib.lib()
        sizes = _lib.GdBvhSizes()
        _lib.check(L.gd_bvh_sizes(len(self.prim_order), mesh.n_vertices, C.byref(sizes)), "bvh_sizes")
        ws = _lib.empty(max(int(sizes.build_workspace_bytes), 1), torch.uint8)
        g = mesh.device_view()
        v = _lib.GdBvh.from_buffer_copy(self.device_view())
        v.nv = mesh.n_vertices
        _lib.check(L.gd_bvh_layout(C.byref(g), C.byref(v), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "bvh_layout")
        self._staged = mesh._root

    def _stage(self, mesh: TriangleMesh):
        """float32 copy of the mesh's base vertices (once per base buffer)."""
        if self._staged is mesh._root:
            return
        if self._vtx32.numel() != max(mesh.n_vertices, 1) * 4:
            # another vertex count: the staged numbering must be rebuilt
            self._write_records(mesh)
            return
        g = mesh.device_view()
        v = _lib.GdBvh.from_buffer_copy(self.device_view())
        v.nv = mesh.n_vertices
        _lib.check(_lib.lib().gd_stage_vertices(C.byref(g), C.byref(v), _lib.stream_ptr()), "stage_vertices")
        self._staged = mesh._root

    def _device_refit(self, mesh: TriangleMesh):
        if mesh.n_triangles != len(self.prim_order):
            raise TopologyMismatchError(
                f"refit mesh has {mesh.n_triangles} triangles, tree was built over {len(self.prim_order)}"
            )
        self._ensure_layout(mesh)
        if self._layout_tris is not mesh.triangles:
            # same triangle count but possibly another index buffer: the
            # reference refits from mesh.triangles (bvh.py:244), so re-lay
            if self._layout_tris is None or not np.array_equal(self._layout_tris, mesh.triangles):
                self._write_records(mesh)
            self._layout_tris = mesh.triangles
        self._stage(mesh)
        self._mesh = mesh
        g = mesh.device_view()
        v = self.device_view()
        _lib.check(_lib.lib().gd_refit(C.byref(g), C.byref(v), _lib.stream_ptr()), "refit")
        self._export_cache = None
        self._host_boxes = None

    def ensure_device(self, mesh: TriangleMesh):
        """Make the device boxes describe `mesh` (refit if another geometry)."""
        if self._mesh is None or self._mesh._geometry_key() != mesh._geometry_key():
            self._device_refit(mesh)


def _spread_bits_3(x: np.ndarray) -> np.ndarray:
    """Spread 21 bits to every third bit (bvh.py:58-66); host helper."""
    x = x.astype(np.uint64) & np.uint64(0x1FFFFF)
    for sh, mk in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                   (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        x = (x | (x << np.uint64(sh))) & np.uint64(mk)
    return x


def morton_codes(mesh: TriangleMesh):
    """(codes, triangle_ids) sorted by (code, id) (bvh.py:69-95).  Host
    utility with the reference semantics; the build computes the same codes
    on the device."""
    if mesh.n_triangles == 0:
        raise ValueError("mesh has no triangles")
    V = mesh.vertices
    P = V[mesh.triangles]
    cen = ((P[:, 0] + P[:, 1]) + P[:, 2]) / 3.0
    lo = V.min(axis=0)
    span = V.max(axis=0) - lo
    span = np.where(span > 0.0, span, 1.0)
    f = np.maximum((cen - lo) / span, 0.0)
    q = np.minimum((f * float(1 << _MORTON_BITS)).astype(np.uint64), np.uint64((1 << _MORTON_BITS) - 1))
    code = _spread_bits_3(q[:, 0]) | (_spread_bits_3(q[:, 1]) << np.uint64(1)) | (_spread_bits_3(q[:, 2]) << np.uint64(2))
    ids = np.arange(mesh.n_triangles, dtype=np.int64)
    perm = np.lexsort((ids, code))
    return code[perm], ids[perm]


def build_f12(mesh: TriangleMesh, dtype=np.float64) -> F12Bvh:
    """Build the tree on the device (bvh.py:267-289).  `dtype` selects the
    precision of the exported boxes and of the exact query pass; Morton
    ordering always runs in float64, so both precisions share a topology."""
    if mesh.n_triangles < 1:
        raise ValueError("cannot build a BVH over an empty mesh")
    dt = np.dtype(dtype)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError(f"dtype must be float32 or float64, got {dt}")
    L = _lib.lib()
    sizes = _lib.GdBvhSizes()
    _lib.check(L.gd_bvh_sizes(mesh.n_triangles, mesh.n_vertices, C.byref(sizes)), "bvh_sizes")
    m = mesh.n_triangles
    bvh = F12Bvh(leaf_tris=np.empty((sizes.leaf_count, 2), dtype=np.int64), prim_order=np.empty(m, dtype=np.int64),
                 depth=sizes.depth, dtype=dt)
    # the build sees exactly the host vertices the reference would (a lazily
    # moved mesh is materialised once, reference formula)
    src = mesh if mesh._rot is None else TriangleMesh(mesh.vertices, mesh.triangles)
    bvh._alloc(src.n_vertices)
    torch = _lib.torch()
    ws = _lib.empty(max(int(sizes.build_workspace_bytes), 1), torch.uint8)
    g = src.device_view()
    v = _lib.GdBvh.from_buffer_copy(bvh.device_view())
    v.nv = src.n_vertices
    _lib.check(
        L.gd_bvh_build(C.byref(g), C.byref(v), _lib.ptr(ws), ws.numel(), bvh.prim_order.ctypes.data_as(C.c_void_p),
                       bvh.leaf_tris.ctypes.data_as(C.c_void_p), _lib.stream_ptr()),
        "bvh_build",
    )
    bvh._mesh = src
    bvh._staged = src._root
    bvh._layout_tris = src.triangles
    bvh.prim_order.setflags(write=False)
    bvh.leaf_tris.setflags(write=False)
    if src is not mesh:
        bvh._device_refit(mesh)
    return bvh


def refit(bvh: F12Bvh, mesh: TriangleMesh) -> F12Bvh:
    """Recompute every box for moved vertices, in place (bvh.py:292-306).
    Asynchronous on the current stream; returns the same tree."""
    if mesh.n_triangles != len(bvh.prim_order):
        raise TopologyMismatchError(
            f"refit mesh has {mesh.n_triangles} triangles, tree was built over {len(bvh.prim_order)}"
        )
    bvh._device_refit(mesh)
    return bvh


def descendant(node: int, k: int, offset: int, n_nodes: int | None = None) -> int:
    """((node + 1) << k) - 1 + offset (bvh.py:309-323)."""
    if k < 0 or not 0 <= offset < (1 << k):
        raise ValueError(f"bad descendant query: k={k}, offset={offset}")
    out = ((node + 1) << k) - 1 + offset
    if n_nodes is not None and out >= n_nodes:
        raise IndexError(
            f"descendant {out} of node {node} (k={k}, offset={offset}) is outside the {n_nodes}-node array"
        )
    return out


def node_level(node: int) -> int:
    """Levels between the root and `node` (bvh.py:326-328)."""
    return (node + 1).bit_length() - 1


def remaining_depth(bvh: F12Bvh, node: int) -> int:
    """Levels from `node` down to the leaves (bvh.py:331-335)."""
    if not 0 <= node < bvh.n_nodes:
        raise ValueError(f"node {node} outside the {bvh.n_nodes}-node array")
    return bvh.depth - node_level(node)
