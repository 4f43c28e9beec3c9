"""Desk-scale workload for compute-sanitizer (scripts/ncu_r2.sh): builds,
refits (the k_refit cascade over several 256-leaf groups), min and max
queries through k_traverse's grid barriers (breadth first and chunked in
small arenas, reference and device schedules), the narrow / exact kernels
and the band-overflow rescan, each checked against the device brute force."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2411_11244_b200 as md  # noqa: E402

for nu, nv in ((40, 25), (250, 100)):
    tz, tb = md.ring_pair_base(nu, nv)
    A, B = md.build_f12(tz), md.build_f12(tb)
    for f in (0, 3):
        xa, xb = md.ring_frame_transforms(f)
        a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
        md.refit(A, a)
        md.refit(B, b)
        for kind in ("min", "max"):
            run = md.run_min_query if kind == "min" else md.run_max_query
            want_d, _w = (md.brute_force_min if kind == "min" else md.brute_force_max)(a, b, force=True)
            for cfg in (md.EngineConfig(), md.EngineConfig(device_schedule=-1),
                        md.EngineConfig(arena_entries=1 << 12, front_hard_cap=1 << 30)):
                r = run(a, b, A, B, cfg)
                assert r.distance == want_d, (nu, f, kind, cfg, r.distance, want_d)
            print(nu, nv, f, kind, r.distance, r.witness.tri_a, r.witness.tri_b, flush=True)
a, b = md.gen_scene("nested-shells", {"lat": 30, "lon": 36, "r_inner": 0.8, "r_outer": 0.81})
A, B = md.build_f12(a), md.build_f12(b)
r = md.run_min_query(a, b, A, B, md.EngineConfig(front_hard_cap=1 << 30))
print("shells", r.distance, r.witness.tri_a, r.witness.tri_b)
print("sanitize_desk done")
