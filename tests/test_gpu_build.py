"""The device build (csrc/build.cu, csrc/sort.cu): the repo's own radix sort
and the device pairing, against the oracle's build (numpy restatement of
bvh.py:69-289 with the literal greedy) and against the exact host greedy
(GD_FORCE_HOST_PAIRING) at the rings' full size."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mode(md):
    from paper_2411_11244_b200 import _lib

    return _lib.lib().gd_build_pairing_mode()


@pytest.mark.parametrize("seed", range(12))
def test_build_matches_oracle_random(md, gpu, oracle, seed):
    """Random soups, blobs, shells, grids of 3 .. 20K triangles (sizes off
    powers of two, so merges are needed): prim_order (Morton radix sort) and
    leaf_tris (pairing + leaf assembly) equal the oracle's."""
    rng = np.random.default_rng(seed)
    kinds = [("random-blobs", {"n": int(rng.integers(3, 20000)), "seed": seed}),
             ("nested-shells", {"lat": int(rng.integers(4, 40)), "lon": int(rng.integers(4, 40))}),
             ("offset-grids", {"res": int(rng.integers(3, 60))})]
    modes = set()
    for kind, params in kinds:
        a, _ = md.gen_scene(kind, params)
        t = md.build_f12(a)
        modes.add(_mode(md))
        want = oracle.build_tree(a.vertices, a.triangles)
        np.testing.assert_array_equal(t.prim_order, want.prim_order, err_msg=f"{kind} {params}")
        np.testing.assert_array_equal(t.leaf_tris, want.leaf_tris, err_msg=f"{kind} {params}")
        np.testing.assert_array_equal(t.node_min, want.node_min)
    assert modes <= {0, 1, 2}


def test_build_matches_oracle_small_sizes(md, gpu, oracle):
    """Every size 1 .. 80 (the pairing's slack starts at 0 for several,
    e.g. 3, 5, 6, 7, 11): the device build equals the oracle's."""
    for n in range(1, 81):
        a, _ = md.gen_scene("random-blobs", {"n": n, "seed": n})
        t = md.build_f12(a)
        want = oracle.build_tree(a.vertices, a.triangles)
        np.testing.assert_array_equal(t.prim_order, want.prim_order, err_msg=str(n))
        np.testing.assert_array_equal(t.leaf_tris, want.leaf_tris, err_msg=str(n))


def test_device_pairing_used_and_exact_on_tori(md, gpu, oracle):
    """Tori (sizes the reference pairs in seconds): the device pairing runs
    (mode 1) and equals the literal greedy."""
    used = 0
    for nu, nv in ((30, 17), (61, 23), (100, 50), (77, 41)):
        tz, _ = md.ring_pair_base(nu, nv)
        t = md.build_f12(tz)
        used += _mode(md) == 1
        want = oracle.build_tree(tz.vertices, tz.triangles)
        np.testing.assert_array_equal(t.leaf_tris, want.leaf_tris, err_msg=f"{nu}x{nv}")
        np.testing.assert_array_equal(t.prim_order, want.prim_order)
    assert used >= 2


def test_device_pairing_equals_host_greedy_full_rings(md, gpu):
    """2 x 7.5M-triangle rings (config 2): the device-built tree equals the
    one built with the exact host greedy, and the device path was taken."""
    tz, _ = md.ring_pair_base(2500, 1500)
    dev = md.build_f12(tz)
    assert _mode(md) == 1
    os.environ["GD_FORCE_HOST_PAIRING"] = "1"
    try:
        host = md.build_f12(tz)
        assert _mode(md) == 2
    finally:
        del os.environ["GD_FORCE_HOST_PAIRING"]
    np.testing.assert_array_equal(dev.prim_order, host.prim_order)
    np.testing.assert_array_equal(dev.leaf_tris, host.leaf_tris)
    np.testing.assert_array_equal(dev.node_min, host.node_min)
