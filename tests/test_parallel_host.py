"""Multi-process host logic of the multi-GPU drivers (parallel.py) on CPU:
world_size-2 gloo groups, frame sharding and gathering, the split-query
combination rule.  The per-frame compute is a CPU stand-in here; the GPU
paths are covered by tests/test_gpu_parallel.py."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frame_value(f):
    # a deterministic stand-in for one frame's (distance, tri_a, tri_b)
    return (0.25 + 0.001 * f, 3 * f % 97, 7 * f % 89)


def _worker(rank, world, port, n_frames, q):
    import torch.distributed as dist

    from paper_2411_11244_b200 import parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seen = []

        def fn(f):
            seen.append(f)
            return _frame_value(f)

        res = parallel.run_frames(n_frames, fn, device="cpu")
        q.put((rank, seen, res.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [0, 1, 7, 40])
def test_frames_sharded_and_gathered(n_frames):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_frames, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.array([_frame_value(f) for f in range(n_frames)], dtype=np.float64).reshape(n_frames, 3)
    seen_all = []
    for rank, seen, res in out:
        # each rank evaluated exactly its frames f = rank (mod world) ...
        assert seen == list(range(rank, n_frames, world))
        seen_all += seen
        # ... and every rank holds every frame afterwards
        assert np.array_equal(np.asarray(res, dtype=np.float64).reshape(n_frames, 3), want)
    assert sorted(seen_all) == list(range(n_frames))


def test_frames_single_process():
    from paper_2411_11244_b200 import parallel

    res = parallel.run_frames(5, _frame_value)
    assert np.array_equal(res, np.array([_frame_value(f) for f in range(5)]))
    assert list(parallel.frames_of_rank(10, 1, 4)) == [1, 5, 9]
    with pytest.raises(ValueError):
        parallel.frames_of_rank(10, 4, 4)


def test_combine_parts_rule():
    """best distance first, then the lexicographically smallest (tri_a, tri_b)
    (query.py:205-220); parts without a witness never win unless all lack one"""
    from paper_2411_11244_b200.parallel import combine_parts

    parts = [(0.5, 9, 9), (0.25, 7, 3), (0.25, 2, 8), (0.1, -1, -1)]
    assert combine_parts("min", parts) == (0.25, 2, 8)
    assert combine_parts("max", parts) == (0.5, 9, 9)
    assert combine_parts("max", [(3.0, 4, 1), (3.0, 4, 0), (2.0, 0, 0)]) == (3.0, 4, 0)
    assert combine_parts("min", [(0.3, -1, -1), (0.2, -1, -1)]) == (0.3, -1, -1)
