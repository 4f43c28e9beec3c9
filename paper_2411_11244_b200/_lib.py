"""ctypes binding of libgdist.so (include/gdist.h).

The library is built in-tree (`_build.py`) and loaded from the package
directory.  There is no CPU fallback: if the library is missing, or no CUDA
device is visible when a device operation runs, a RuntimeError is raised.
Torch is used only to allocate device buffers and to supply the current
stream; all computation happens in libgdist's CUDA kernels.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ConfigError, FrontOverflowError, MeshDistError, TopologyMismatchError

_LIB_PATH = Path(__file__).resolve().parent / os.environ.get("GDIST_LIB_VARIANT", "libgdist.so")

GD_OK = 0
GD_ERR_INVALID = 1
GD_ERR_CONFIG = 2
GD_ERR_TOPOLOGY = 3
GD_ERR_FRONT_OVERFLOW = 4
GD_ERR_WORKSPACE = 5
GD_ERR_CUDA = 6
GD_ERR_NO_DEVICE = 7


class GdMesh(C.Structure):
    _fields_ = [
        ("vtx", C.c_void_p),
        ("tri", C.c_void_p),
        ("nv", C.c_int64),
        ("m", C.c_int64),
        ("rot", C.c_double * 9),
        ("trans", C.c_double * 3),
        ("has_xf", C.c_int32),
        ("xf_order", C.c_int32),
    ]


class GdBvhSizes(C.Structure):
    _fields_ = [
        ("leaf_count", C.c_int64),
        ("n_nodes", C.c_int64),
        ("depth", C.c_int32),
        ("_pad", C.c_int32),
        ("build_workspace_bytes", C.c_size_t),
    ]


class GdBvh(C.Structure):
    _fields_ = [
        ("box", C.c_void_p),
        ("leaf_rec", C.c_void_p),
        ("vtx32", C.c_void_p),
        ("vmap", C.c_void_p),
        ("leaf_vtx", C.c_void_p),
        ("leaf_x", C.c_void_p),
        ("leaf_xvtx", C.c_void_p),
        ("leaf_count", C.c_int64),
        ("n_tris", C.c_int64),
        ("nv", C.c_int64),
        ("depth", C.c_int32),
        ("_pad", C.c_int32),
        ("leaf_tri", C.c_void_p),
    ]


class GdConfig(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("precision", C.c_int32),
        ("front_cap", C.c_int64),
        ("depth_cap", C.c_int32),
        ("enhanced_bounds", C.c_int32),
        ("culling", C.c_int32),
        ("guarantee_witness", C.c_int32),
        ("front_hard_cap", C.c_int64),
        ("warm_a", C.c_int64),
        ("warm_b", C.c_int64),
        ("band_cap", C.c_int64),
        ("split_rank", C.c_int32),
        ("split_world", C.c_int32),
        ("split_level", C.c_int32),
        ("frame", C.c_int32),
        ("warm_from", C.c_void_p),
        ("peer_bounds", C.c_void_p),
        ("n_peers", C.c_int32),
        ("schedule", C.c_int32),
        ("arena_entries", C.c_int64),
    ]


class GdResult(C.Structure):
    _fields_ = [
        ("distance", C.c_double),
        ("witness_distance", C.c_double),
        ("point_a", C.c_double * 3),
        ("point_b", C.c_double * 3),
        ("tri_a", C.c_int64),
        ("tri_b", C.c_int64),
        ("expanded_pairs", C.c_int64),
        ("narrow_pairs", C.c_int64),
        ("band_pairs", C.c_int64),
        ("overflow_candidates", C.c_int64),
        ("overflow_front_in", C.c_int64),
        ("overflow_cap", C.c_int64),
        ("iterations", C.c_int32),
        ("status", C.c_int32),
        ("rounds", C.c_int32),
        ("pending", C.c_int32),
    ]


class GdIterStat(C.Structure):
    _fields_ = [
        ("front_in", C.c_int64),
        ("front_out", C.c_int64),
        ("culled", C.c_int64),
        ("bound_after", C.c_double),
        ("k", C.c_int32),
        ("_pad", C.c_int32),
    ]


P = C.c_void_p
_SIGNATURES = {
    "gd_version": (C.c_char_p, []),
    "gd_last_error": (C.c_char_p, []),
    "gd_abi_version": (C.c_int, []),
    "gd_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "gd_launch_count": (C.c_longlong, []),
    "gd_set_profiling": (C.c_int, [C.c_int]),
    "gd_query_phase_ms": (C.c_int, [C.POINTER(C.c_float), C.c_int]),
    "gd_bvh_sizes": (C.c_int, [C.c_int64, C.c_int64, C.POINTER(GdBvhSizes)]),
    "gd_bvh_build": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdBvh), P, C.c_size_t, P, P, P]),
    "gd_bvh_layout": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdBvh), P, C.c_size_t, P]),
    "gd_build_pairing_mode": (C.c_int, []),
    "gd_stage_vertices": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdBvh), P]),
    "gd_mesh_relative": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdMesh)]),
    "gd_refit": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdBvh), P]),
    "gd_export_boxes": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdBvh), C.c_int, P, P, P]),
    "gd_pair_greedy": (C.c_int, [P, C.c_int64, P]),
    "gd_query_workspace_size": (C.c_int, [C.POINTER(GdBvh), C.POINTER(GdBvh), C.POINTER(GdConfig),
                                          C.POINTER(C.c_size_t)]),
    "gd_query": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdBvh),
                           C.POINTER(GdConfig), P, C.c_size_t, C.POINTER(GdResult), C.POINTER(GdIterStat),
                           C.c_int, P]),
    "gd_query_async": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdBvh),
                                 C.POINTER(GdConfig), P, C.c_size_t, P, P]),
    "gd_query_round": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdBvh),
                                 C.POINTER(GdConfig), P, C.c_size_t, C.c_int, P]),
    "gd_query_async_ev": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdBvh),
                                    C.POINTER(GdConfig), P, C.c_size_t, P, P, P]),
    "gd_query_traverse": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdBvh),
                                    C.POINTER(GdConfig), P, C.c_size_t, C.c_int, C.c_int, P]),
    "gd_query_finish": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdBvh),
                                  C.POINTER(GdConfig), P, C.c_size_t, P, P]),
    "gd_query_group_async": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdBvh),
                                       C.c_int, C.POINTER(GdConfig), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                       C.POINTER(C.c_void_p), C.c_int, P, P]),
    "gd_frame_graph_create": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdBvh),
                                        C.c_int, C.POINTER(GdConfig), C.POINTER(C.c_void_p),
                                        C.POINTER(C.c_size_t), C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                        P, P, C.POINTER(C.c_void_p)]),
    "gd_frame_graph_launch": (C.c_int, [P, C.POINTER(GdMesh), C.POINTER(GdMesh), P]),
    "gd_frame_graph_destroy": (C.c_int, [P]),
    "gd_query_result_device": (C.c_int, [C.POINTER(GdConfig), P, C.POINTER(C.c_void_p)]),
    "gd_query_bound_device": (C.c_int, [C.POINTER(GdConfig), P, C.POINTER(C.c_void_p)]),
    "gd_ipc_handle": (C.c_int, [P, P, C.POINTER(C.c_uint64)]),
    "gd_ipc_open": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_void_p)]),
    "gd_ipc_close": (C.c_int, [P]),
    "gd_query_result_async": (C.c_int, [C.POINTER(GdConfig), P, P, C.c_int, P]),
    "gd_query_collect": (C.c_int, [C.POINTER(GdBvh), C.POINTER(GdBvh), C.POINTER(GdConfig), P, P,
                                   C.POINTER(GdResult), C.POINTER(GdIterStat), C.c_int, P]),
    "gd_dfs_query": (C.c_int, [C.POINTER(GdMesh), C.POINTER(GdMesh), C.POINTER(GdBvh), C.POINTER(GdConfig), P,
                               C.c_size_t, C.POINTER(GdResult), C.POINTER(C.c_int64), P]),
    "gd_obj_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                              C.POINTER(C.c_int64)]),
    "gd_obj_read": (C.c_int, [P, P, P]),
    "gd_obj_close": (None, [P]),
    "gd_tri_tri_batch": (C.c_int, [C.c_int, C.c_int, P, P, C.c_int64, P, P, P, P]),
    "gd_tri_tri_fast": (C.c_int, [C.c_int, P, P, C.c_int64, P, P]),
    "gd_box_bounds_batch": (C.c_int, [C.c_int, C.c_int, P, P, P, P, C.c_int64, P, P]),
    "gd_brute_force": (C.c_int, [C.c_int, C.c_int, P, C.c_int64, P, C.c_int64, C.POINTER(GdResult), P]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libgdist.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not _LIB_PATH.exists():
                    raise RuntimeError(
                        f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                        "(no CPU fallback exists)"
                    )
                h = C.CDLL(str(_LIB_PATH))
                for name, (res, args) in _SIGNATURES.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = h
    return _lib


def exported_symbols():
    return sorted(_SIGNATURES)


def last_error() -> str:
    msg = lib().gd_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Map a GdStatus onto the reference's exception classes."""
    if status == GD_OK:
        return
    msg = last_error()
    if status == GD_ERR_CONFIG:
        raise ConfigError(msg)
    if status == GD_ERR_TOPOLOGY:
        raise TopologyMismatchError(msg)
    if status == GD_ERR_INVALID:
        raise ValueError(msg)
    if status == GD_ERR_FRONT_OVERFLOW:
        raise MeshDistError(msg)  # callers re-raise with counts as FrontOverflowError
    raise RuntimeError(f"libgdist{(' ' + what) if what else ''}: {msg} (status {status})")


def overflow_error(res: GdResult) -> FrontOverflowError:
    return FrontOverflowError(int(res.overflow_candidates), int(res.overflow_front_in), int(res.overflow_cap))


# ---------------------------------------------------------------------------
# device plumbing (torch = buffers + streams only)
# ---------------------------------------------------------------------------
_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def require_device():
    """Fail loudly when no CUDA device is visible: there is no CPU path."""
    cnt = C.c_int(0)
    check(lib().gd_device_count(C.byref(cnt)))
    if cnt.value < 1 or not torch().cuda.is_available():
        raise RuntimeError("paper_2411_11244_b200 needs a CUDA device (B200, sm_100a); none is visible")


def device():
    require_device()
    t = torch()
    return t.device("cuda", t.cuda.current_device())


def check_device(t, what: str):
    """Device objects (mesh uploads, trees, workspaces) live on the GPU that
    was current when they were created; using them from another device would
    hand the kernels foreign pointers."""
    cur = torch().cuda.current_device()
    if t.device.index != cur:
        raise ValueError(f"{what} lives on cuda:{t.device.index} but the current device is cuda:{cur}; "
                         f"create one per device (one process per GPU)")


def stream_ptr():
    return C.c_void_p(torch().cuda.current_stream().cuda_stream)


def empty(shape, dtype, dev=None):
    t = torch()
    return t.empty(shape, dtype=dtype, device=dev or device())


def ptr(tensor) -> C.c_void_p:
    return C.c_void_p(tensor.data_ptr())


def env_flag(name: str, default: str = "") -> str:
    return os.environ.get(name, default)
