"""Work per rank of a split query with and without the IPC-linked bound
(run under torchrun; more ranks than GPUs share cuda:0 over gloo -- the
counts are meaningful, timings are not).
torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/exp_split_share.py"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
n_dev = torch.cuda.device_count()
torch.cuda.set_device(rank % n_dev)
dist.init_process_group("nccl" if world <= n_dev else "gloo")
cfg = md.EngineConfig(front_hard_cap=1 << 25)
scenes = [("rings 2x7.5M", md.gen_scene("interlocked-rings", {"nu": 2500, "nv": 1500})),
          ("nested shells 2x180K", md.gen_scene("nested-shells", {"lat": 301, "lon": 300, "r_inner": 0.8,
                                                                   "r_outer": 0.81}))]
from paper_2411_11244_b200.parallel import release_split_plans  # noqa: E402

for name, (a, b) in scenes:
    release_split_plans()
    ta, tb = md.build_f12(a), md.build_f12(b)
    for kind in ("min", "max"):
        if name.startswith("nested") and kind == "max":
            continue
        full = (md.run_min_query if kind == "min" else md.run_max_query)(a, b, ta, tb, cfg)
        row = {}
        for share, lvl in ((False, 5), (True, 5), (True, 8), (True, 11)):
            r = md.run_split_query(a, b, ta, tb, kind, cfg, share_bound=share, split_level=lvl)
            assert r.distance == full.distance
            t = torch.tensor([r.expanded_pairs, r.narrow_pairs], dtype=torch.float64)
            out = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            row[("shared" if share else "local") + f" L{lvl}"] = [int(o[0]) for o in out]
            release_split_plans()
        if rank == 0:
            print(json.dumps({"scene": name, "kind": kind, "world": world, "single_gpu_expanded": full.expanded_pairs,
                              "per_rank_expanded": row}), flush=True)
dist.destroy_process_group()
