"""Config 5 on N GPUs: one query split over the ranks (run_split_query;
SURVEY.md 8(d) config 5 "single query on 1 and on 8 GPUs").  One process per
GPU under torchrun; prints one JSON line per (size, kind) on rank 0 with the
max-over-ranks device time of the split part, the part's work, and the
single-GPU time of the same query on rank 0 for comparison.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/bench_split.py [nu nv ...]

More ranks than GPUs share devices over gloo (a functional check only)."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import parallel  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
n_dev = torch.cuda.device_count()
torch.cuda.set_device(rank % n_dev)
backend = "nccl" if world <= n_dev else "gloo"
if world > 1:
    dist.init_process_group(backend, **({"device_id": torch.device("cuda", rank % n_dev)} if backend == "nccl" else {}))
red = torch.device("cuda", rank % n_dev) if backend == "nccl" else torch.device("cpu")
sizes = [int(x) for x in sys.argv[1:]] or [1000, 250, 2500, 1000, 5000, 1500]
cfg = md.EngineConfig(front_hard_cap=1 << 27)


def timed(fn, reps=5, collective=True):
    fn()
    best = 1e30
    for _ in range(reps):
        if world > 1 and collective:
            dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = fn()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e)], dtype=torch.float64, device=red)
        if world > 1 and collective:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        best = min(best, float(t.item()))
    return best, r


for nu, nv in zip(sizes[::2], sizes[1::2]):
    a, b = md.gen_scene("interlocked-rings", {"nu": nu, "nv": nv})
    ta, tb = md.build_f12(a), md.build_f12(b)
    for kind in ("min", "max"):
        run = md.run_min_query if kind == "min" else md.run_max_query
        # every rank times the single-GPU query on its own (no collective)
        single_ms, single = timed(lambda: run(a, b, ta, tb, cfg), collective=False)
        split_ms, part = timed(lambda: md.run_split_query(a, b, ta, tb, kind, cfg))
        work = torch.tensor([part.expanded_pairs], dtype=torch.float64, device=red)
        works = [torch.zeros_like(work) for _ in range(world)]
        if world > 1:
            dist.all_gather(works, work)
        else:
            works = [work]
        if rank == 0:
            assert part.distance == single.distance
            print(json.dumps({"tris_total": 2 * a.n_triangles, "kind": kind, "world": world, "backend": backend,
                              "single_gpu_ms": round(single_ms, 4), "split_ms_max_over_ranks": round(split_ms, 4),
                              "single_expanded": single.expanded_pairs,
                              "part_expanded": [int(w.item()) for w in works]}), flush=True)
parallel.release_split_plans()
if world > 1:
    dist.destroy_process_group()
