"""Phase anatomy of one query on a gen_scene scene (CUDA events + device
timestamps).  python scripts/exp_scene.py KIND '{"param": v}' min|max [hard_cap_log2]"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import _lib  # noqa: E402
from paper_2411_11244_b200 import query as Q  # noqa: E402

kind_s, params, kind = sys.argv[1], json.loads(sys.argv[2]), sys.argv[3]
cap = 1 << int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 28
a, b = md.gen_scene(kind_s, params)
ta, tb = md.build_f12(a), md.build_f12(b)
pq = Q.PreparedQuery(a, b, ta, tb, md.EngineConfig(front_hard_cap=cap), kind)
r = pq.run()
L = _lib.lib()
L.gd_set_profiling(1)
r = pq.run()
ph = (C.c_float * 160)()
n = L.gd_query_phase_ms(ph, 160)
L.gd_set_profiling(0)
it = len(r.iterations)
print(json.dumps({"scene": kind_s, "params": params, "kind": kind, "distance": r.distance,
                  "phases_ms": [round(x, 4) for x in ph[:5]], "narrow_pairs": r.narrow_pairs, "band": r.band_pairs,
                  "iters": [(s.k, s.front_in, s.front_out, round(ph[5 + i], 4), round(ph[5 + it + i], 4))
                            for i, s in enumerate(r.iterations)]}))
