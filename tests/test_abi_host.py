"""C-ABI library and host-side logic, no GPU needed: the .so loads and
exports every symbol include/gdist.h declares; the host C++ greedy pairing
equals the reference's literal greedy; host API contracts (validation,
transforms, OBJ, config, scenes) match the reference."""

import ctypes as C
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent


def _declared():
    text = (REPO / "include" / "gdist.h").read_text()
    return sorted(set(re.findall(r"\b(gd_\w+)\s*\(", text)))


def test_library_exports_header(md):
    from paper_2411_11244_b200 import _lib

    lib = _lib.lib()
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == declared
    assert lib.gd_abi_version() == 15
    assert b"sm_100a" in lib.gd_version()


def test_struct_sizes_match_header(tmp_path):
    """ctypes mirrors of the C structs have the layout the C compiler gives
    include/gdist.h (sizes and every field offset)."""
    import shutil
    import subprocess

    from paper_2411_11244_b200 import _lib

    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    structs = {"GdMesh": _lib.GdMesh, "GdBvhSizes": _lib.GdBvhSizes, "GdBvh": _lib.GdBvh, "GdConfig": _lib.GdConfig,
               "GdResult": _lib.GdResult, "GdIterStat": _lib.GdIterStat}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "gdist.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "sizes.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-I", str(REPO / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def test_no_device_fails_loudly(md):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2411_11244_b200 import _lib

    cnt = C.c_int(-1)
    assert _lib.lib().gd_device_count(C.byref(cnt)) == 0 and cnt.value == 0
    a, b = md.gen_scene("random-blobs", {"n": 10})
    with pytest.raises(RuntimeError, match="CUDA device"):
        md.build_f12(a)
    with pytest.raises(RuntimeError, match="CUDA device"):
        md.tri_tri_min(np.eye(3), np.eye(3) + 1)


def _greedy_native(sa, n):
    from paper_2411_11244_b200 import _lib

    out = np.zeros(n, dtype=np.uint8)
    sa = np.ascontiguousarray(sa, dtype=np.float64)
    _lib.check(_lib.lib().gd_pair_greedy(sa.ctypes.data_as(C.c_void_p), n, out.ctypes.data_as(C.c_void_p)))
    return np.flatnonzero(out).tolist()


@pytest.mark.parametrize("seed", range(6))
def test_pairing_matches_literal_greedy(oracle, seed):
    rng = np.random.default_rng(seed)
    sizes = list(range(2, 70)) + [127, 255, 300, 511, 513, 767, 1023, 1500, 3001]
    for n in sizes:
        if seed % 2:
            sa = np.round(rng.random(n - 1) * 8) / 8  # many exact ties
        else:
            sa = rng.random(n - 1)
        assert _greedy_native(sa, n) == oracle.greedy_pairs(sa, n), (seed, n)


def test_pairing_torus_golden(golden, golden_meta, oracle):
    from paper_2411_11244_b200.scenes import ring_pair_base

    for rec in golden_meta["pairings"]:
        tz, _ = ring_pair_base(rec["nu"], rec["nv"])
        V, T = tz.vertices, tz.triangles
        _, order = oracle.morton_order(V, T)
        P = V[T]
        sa = oracle.pair_surface_areas(order, P.min(axis=1), P.max(axis=1))
        lefts = _greedy_native(sa, len(T))
        leaf = oracle.leaves_from_pairs(order, lefts, len(T))
        assert np.array_equal(leaf.astype(np.int32), golden[f"pair_{rec['name']}_leaf"])


def test_pairing_large_is_fast():
    import time

    rng = np.random.default_rng(0)
    n = 1_500_000
    sa = rng.random(n - 1)
    t0 = time.time()
    lefts = _greedy_native(sa, n)
    assert len(lefts) == n - (1 << (n.bit_length() - 1))
    assert time.time() - t0 < 30


# -- host API contracts --------------------------------------------------------
def test_mesh_validation(md):
    with pytest.raises(ValueError):
        md.TriangleMesh(np.zeros((3, 2)), [[0, 1, 2]])
    with pytest.raises(ValueError, match="out of range"):
        md.TriangleMesh(np.zeros((3, 3)), [[0, 1, 3]])
    with pytest.raises(md.DegenerateTriangleError) as ei:
        md.TriangleMesh(np.zeros((3, 3)), [[0, 1, 2], [1, 1, 2]])
    assert ei.value.faces == [(1, (1, 1, 2))]
    m = md.TriangleMesh(np.eye(3), [[0, 1, 2]])
    assert not m.vertices.flags.writeable and m.triangles.dtype == np.int64
    assert m.triangle_points(np.float32).dtype == np.float32


def test_rigid_transform(md):
    with pytest.raises(ValueError):
        md.RigidTransform(np.ones((3, 3)))
    xf = md.RigidTransform.from_axis_angle((0, 0, 1), np.pi / 2)
    v = md.apply_transform(md.TriangleMesh([[1.0, 0, 0], [0, 1, 0], [0, 0, 1]], [[0, 1, 2]]), xf).vertices
    assert np.allclose(v[0], [0, 1, 0], atol=1e-6)
    ident = md.TriangleMesh(np.random.default_rng(0).normal(size=(5, 3)), [[0, 1, 2], [2, 3, 4]])
    assert np.array_equal(md.apply_transform(ident, md.RigidTransform()).vertices, ident.vertices)


def test_apply_transform_matches_reference_formula(md, oracle):
    rng = np.random.default_rng(1)
    V = rng.normal(size=(1000, 3))
    m = md.TriangleMesh(V, np.arange(999).reshape(333, 3))
    x1 = md.RigidTransform.from_axis_angle((1, 2, 3), 0.7, (0.1, -2, 3))
    x2 = md.RigidTransform.from_axis_angle((0, 1, 0), -1.1, (5, 0, 0))
    moved = md.apply_transform(md.apply_transform(m, x1), x2)
    want = oracle.transform_vertices(oracle.transform_vertices(V, x1.rotation, x1.translation), x2.rotation,
                                     x2.translation)
    assert np.array_equal(moved.vertices, want)
    assert moved.triangles is m.triangles


def test_load_obj(md, tmp_path):
    p = tmp_path / "a.obj"
    p.write_text("# c\nv 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nvn 0 0 1\nf 1 2 3 4\nf -4 -3 -2\n")
    m = md.load_obj(p)
    assert m.triangles.tolist() == [[0, 1, 2], [0, 2, 3], [0, 1, 2]]
    bad = tmp_path / "b.obj"
    bad.write_text("v 0 0 0\nv 1 0 0\nv 1 1 0\nf 1 1 2\n")
    with pytest.raises(md.DegenerateTriangleError):
        md.load_obj(bad)
    bad.write_text("v 0 0\n")
    with pytest.raises(md.ObjParseError) as ei:
        md.load_obj(bad)
    assert ei.value.line_no == 1
    bad.write_text("v 0 0 0\nf 1 2 0\n")
    with pytest.raises(md.ObjParseError):
        md.load_obj(bad)


def test_engine_config_and_adaptive(md, golden_meta):
    with pytest.raises(md.ConfigError):
        md.EngineConfig(front_cap=3)
    with pytest.raises(md.ConfigError):
        md.EngineConfig(depth_cap=17)
    with pytest.raises(md.ConfigError):
        md.EngineConfig(precision=16)
    with pytest.raises(md.ConfigError):
        md.EngineConfig(threads="many")
    cfg = md.EngineConfig()
    k = golden_meta["kat"]
    assert md.adaptive_depth(1, cfg, 10) == k["adaptive_1"]
    assert md.adaptive_depth(100000, cfg, 10) == k["adaptive_100000"]
    assert md.adaptive_depth(1000, cfg, 2) == k["adaptive_1000_rem2"]
    for n in (1, 3, 17, 1000, 16383, 16384, 65535, 65536, 10**6):
        for rem in (1, 2, 5, 9):
            kk = md.adaptive_depth(n, cfg, rem)
            assert 1 <= kk <= min(5, rem)
            if kk > 1:
                assert (n << (2 * kk)) < cfg.front_cap


def test_descendant(md, golden_meta):
    k = golden_meta["kat"]
    assert md.descendant(0, 1, 0) == k["descendant_0_1_0"]
    assert md.descendant(0, 2, 3) == k["descendant_0_2_3"]
    assert md.descendant(2, 2, 0) == k["descendant_2_2_0"]
    with pytest.raises(ValueError):
        md.descendant(0, 1, 2)
    with pytest.raises(IndexError):
        md.descendant(3, 2, 0, n_nodes=7)
    seen = {md.descendant(1, 3, o) for o in range(8)}
    assert len(seen) == 8


def _sha(mesh):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(mesh.vertices, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(mesh.triangles, dtype=np.int64).tobytes())
    return h.hexdigest()


def test_scenes_bitwise(md, golden_meta):
    for rec in golden_meta["scenes"] + golden_meta["engine"]:
        a, b = md.gen_scene(rec["kind"], rec["params"])
        assert (_sha(a), _sha(b)) == (rec["hash_a"], rec["hash_b"]), rec
    g = golden_meta["config1"]
    a, b = md.gen_scene("interlocked-rings", {"nu": 100, "nv": 50})
    assert (_sha(a), _sha(b)) == (g["hash_a"], g["hash_b"])
    with pytest.raises(md.SceneError):
        md.gen_scene("nope")
    with pytest.raises(md.SceneError):
        md.gen_scene("random-blobs", {"bogus": 1})
    with pytest.raises(md.SceneError):
        md.gen_scene("random-blobs", {"n": 0})
    assert "interlocked-rings" in md.scene_kinds()


def test_frame_sequence_hashes(md, golden_meta):
    tz, tb = md.ring_pair_base(100, 50)
    for rec in golden_meta["frames"]:
        xa, xb = md.ring_frame_transforms(rec["frame"])
        a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
        assert (_sha(a), _sha(b)) == (rec["hash_a"], rec["hash_b"])


def test_exception_hierarchy(md):
    for cls in (md.ObjParseError, md.DegenerateTriangleError, md.SceneError, md.TightnessError,
                md.TopologyMismatchError, md.FrontOverflowError, md.SizeGuardError, md.ConfigError):
        assert issubclass(cls, md.MeshDistError)
    e = md.FrontOverflowError(10, 2, 4)
    assert (e.candidates, e.front_in, e.cap) == (10, 2, 4)


def test_integration_doc_lists_every_entry_point():
    """INTEGRATION.md maps every C entry point of include/gdist.h to the
    reference interface it replaces."""
    import re
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    names = set(re.findall(r"^\w[\w\s\*]*?\b(gd_\w+)\(", (root / "include" / "gdist.h").read_text(), re.M))
    doc = (root / "INTEGRATION.md").read_text()
    assert names and not [n for n in sorted(names) if n not in doc]


def test_blas_order_probe_reproduces_numpy():
    """GdMesh.xf_order: the probed operation order reproduces numpy's
    `V @ R.T` (the reference's apply_transform, mesh.py:104) bit for bit on
    fresh data, so the device transform gives the reference's vertices."""
    import numpy as np

    from paper_2411_11244_b200 import mesh

    order = mesh.blas_order()
    assert order in (0, 1, 2)
    rng = np.random.default_rng(7)
    V = rng.normal(size=(200, 3)) * 10.0 ** rng.uniform(-4, 4, size=(200, 1))
    R = rng.normal(size=(3, 3))
    got = V @ R.T
    f = mesh._fma
    for i in range(len(V)):
        for j in range(3):
            r, v = [float(x) for x in R[j]], [float(x) for x in V[i]]
            want = {0: f(r[2], v[2], f(r[1], v[1], r[0] * v[0])),
                    1: (r[0] * v[0] + r[1] * v[1]) + r[2] * v[2],
                    2: f(r[0], v[0], f(r[1], v[1], r[2] * v[2]))}[order]
            assert got[i, j] == want, (i, j, order)
