"""Config 4 (nested shells 2 x 2M) min query: phases and the rescan path
(band overflow) timing.  python scripts/exp_shells.py [band_cap ...]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200 import _lib  # noqa: E402
from paper_2411_11244_b200 import query as Q  # noqa: E402

a, b = md.gen_scene("nested-shells", {"lat": 1001, "lon": 1000, "r_inner": 0.8, "r_outer": 0.81})
ta, tb = md.build_f12(a), md.build_f12(b)
cfg = md.EngineConfig(front_hard_cap=1 << 28)
L = _lib.lib()
for cap in [0] + [int(x) for x in sys.argv[1:]]:
    pq = Q.PreparedQuery(a, b, ta, tb, cfg, "min", private_workspace=True)
    if cap:
        pq.g_cfg.band_cap = cap
        nbytes = C.c_size_t(0)
        L.gd_query_workspace_size(C.byref(pq.g_a), C.byref(pq.g_b), C.byref(pq.g_cfg), C.byref(nbytes))
        pq.ws = _lib.empty(nbytes.value, _lib.torch().uint8)
    pq.run()
    L.gd_set_profiling(1)
    r = pq.run()
    ph = (C.c_float * 5)()
    L.gd_query_phase_ms(ph, 5)
    L.gd_set_profiling(0)
    print("band_cap", cap or "default", "phases ms", [round(x, 2) for x in ph], "distance", r.distance,
          "witness", (r.witness.tri_a, r.witness.tri_b), "band_pairs", r.band_pairs, flush=True)
