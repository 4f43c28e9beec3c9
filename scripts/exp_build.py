"""Build time of build_f12 (device Morton codes + sort, pairing, leaf
records, vertex layout, first refit) on rings of 7.5M and 15M triangles:
wall clock of the public call after a warm-up build (CUDA context, kernels
loaded), with the mesh generation and upload timed apart.
python scripts/exp_build.py [nu nv ...pairs]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402

sizes = [(int(a), int(b)) for a, b in zip(sys.argv[1::2], sys.argv[2::2])] or [(2500, 1500), (5000, 1500)]
w, _ = md.ring_pair_base(100, 50)
md.build_f12(w)  # warm-up
for nu, nv in sizes:
    t0 = time.perf_counter()
    tz, tb = md.ring_pair_base(nu, nv)
    t1 = time.perf_counter()
    tz.device_view()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        s = time.perf_counter()
        A = md.build_f12(tz)
        torch.cuda.synchronize()
        t = time.perf_counter() - s
        best = t if best is None else min(best, t)
    print(json.dumps({"tris": tz.n_triangles, "scene_s": round(t1 - t0, 3), "upload_s": round(t2 - t1, 3),
                      "build_f12_s": round(best, 4), "leaf_count": A.leaf_count, "depth": A.depth}), flush=True)
