"""Error of the float32 narrow-phase distance (tri_tri_fast, the FMA-
contracted float32 arithmetic k_ntest / k_nfilter use) against the exact
float64 reference arithmetic (batch_tri_tri_min/max), in float32 ulps of the
pair's coordinate scale M = max |coordinate|: the margin the exact band's
window (E = 2^-15 M = 256 ulps) keeps.  The float64
triangles are first rounded to float32 (as the staged vertices are), so the
error measured is the float32 pipeline's, vertex rounding included.
Adversarial families: random, near-parallel edges, slivers / needles,
coplanar overlaps, near-touching, far from the origin, scale sweep."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

import paper_2411_11244_b200 as md  # noqa: E402
from paper_2411_11244_b200.bounds import tri_tri_fast  # noqa: E402

rng = np.random.default_rng(0)
N = 1 << 20


def fam_random(n):
    return rng.normal(size=(n, 3, 3)), rng.normal(size=(n, 3, 3)) + rng.normal(size=(n, 1, 3)) * 2


def fam_parallel(n):
    a = rng.normal(size=(n, 3, 3))
    d = rng.normal(size=(n, 1, 3)) * 1e-3
    eps = 10.0 ** rng.uniform(-9, -2, size=(n, 1, 1))
    b = a + d + rng.normal(size=(n, 3, 3)) * eps  # nearly a translate: parallel edges / faces
    return a, b


def fam_sliver(n):
    a = rng.normal(size=(n, 3, 3))
    t = rng.uniform(size=(n, 1, 1))
    a[:, 2] = a[:, 0] * t[:, 0] + a[:, 1] * (1 - t[:, 0]) + rng.normal(size=(n, 3)) * 10.0 ** rng.uniform(-8, -3, (n, 1))
    b = rng.normal(size=(n, 3, 3)) * 0.5 + rng.normal(size=(n, 1, 3))
    return a, b


def fam_coplanar(n):
    a = rng.normal(size=(n, 3, 3))
    a[:, :, 2] = 0.0
    b = rng.normal(size=(n, 3, 3))
    b[:, :, 2] = 10.0 ** rng.uniform(-9, -1, size=(n, 1)) * rng.choice([-1, 1, 0], size=(n, 1))
    return a, b


def fam_touching(n):
    a = rng.normal(size=(n, 3, 3))
    b = rng.normal(size=(n, 3, 3))
    # translate b so its vertex 0 sits near a's edge midpoint
    mid = 0.5 * (a[:, 0] + a[:, 1])
    b += (mid - b[:, 0])[:, None, :] + rng.normal(size=(n, 1, 3)) * 10.0 ** rng.uniform(-8, -2, (n, 1, 1))
    return a, b


def fam_far(n):
    a, b = fam_parallel(n)
    off = rng.normal(size=(n, 1, 3)) * 10.0 ** rng.uniform(0, 4, (n, 1, 1))
    s = 10.0 ** rng.uniform(-3, 0, (n, 1, 1))
    return a * s + off, b * s + off


def fam_mesh_like(n):
    """small (1e-3) triangles 0.3 apart, like the rings' contact region"""
    c = rng.normal(size=(n, 1, 3))
    a = c + rng.normal(size=(n, 3, 3)) * 1e-3
    nrm = rng.normal(size=(n, 1, 3))
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    b = c + 0.3 * nrm + rng.normal(size=(n, 3, 3)) * 1e-3
    return a, b


out = {}
for name, fam in [("random", fam_random), ("near-parallel", fam_parallel), ("sliver", fam_sliver),
                  ("coplanar", fam_coplanar), ("touching", fam_touching), ("far-from-origin", fam_far),
                  ("mesh-like", fam_mesh_like)]:
    a, b = fam(N)
    a32, b32 = a.astype(np.float32), b.astype(np.float32)
    for kind in ("min", "max"):
        fast = tri_tri_fast(kind, a32, b32).astype(np.float64)
        exact = (md.batch_tri_tri_min if kind == "min" else md.batch_tri_tri_max)(a32.astype(np.float64),
                                                                              b32.astype(np.float64))[0]
        ref = (md.batch_tri_tri_min if kind == "min" else md.batch_tri_tri_max)(a, b)[0]
        M = np.maximum(np.abs(a).reshape(N, -1).max(1), np.abs(b).reshape(N, -1).max(1))
        ulp = M * 2.0 ** -23
        e_arith = np.abs(fast - exact) / ulp  # float32 arithmetic on the rounded triangles
        e_total = np.abs(fast - ref) / ulp    # including the vertex rounding
        top = np.argsort(-e_total)[:5]
        for t in top:
            print("   worst", name, kind, "err_ulps %.1f" % e_total[t], "exact/M %.3e" % (ref[t] / M[t]),
                  "fast/M %.3e" % (fast[t] / M[t]), "M %.3g" % M[t], flush=True)
        # error above 32 ulps: how close to contact are those pairs
        big = e_total > 32
        if big.any():
            print("   >32 ulps:", int(big.sum()), "of", N, "max exact/M among them %.3e" % float((ref[big] / M[big]).max()),
                  flush=True)
        if kind == "min":
            # the lower bound the band windows on: never above the reference
            # distance by more than rounding; how much looser than the estimate
            lb = tri_tri_fast("min-lb", a32, b32).astype(np.float64)
            over = (lb - ref) / ulp
            loose = (fast - lb) / ulp
            print("   lb", name, ": max (lb - exact) ulps %.2f, loose (fast - lb) ulps: p50 %.2f p99 %.2f max %.1f; pairs with "
                  "fast - lb > 64 ulps: %d" % (over.max(), np.median(loose), np.quantile(loose, 0.99), loose.max(),
                                               int((loose > 64).sum())), flush=True)
            out[f"{name}/lb"] = {"max_lb_minus_exact_ulps": float(over.max()), "loose_p99_ulps": float(np.quantile(loose, 0.99)),
                                 "loose_max_ulps": float(loose.max())}
        out[f"{name}/{kind}"] = {"max_ulps_arith": float(e_arith.max()), "p99999_arith": float(np.quantile(e_arith, 0.99999)),
                                 "max_ulps_total": float(e_total.max()), "argmax": int(e_total.argmax())}
        print(name, kind, json.dumps(out[f"{name}/{kind}"]), flush=True)
print(json.dumps({"worst_total_ulps": max(v["max_ulps_total"] for v in out.values() if "max_ulps_total" in v),
                  "worst_lb_minus_exact_ulps": max(v["max_lb_minus_exact_ulps"] for v in out.values()
                                                   if "max_lb_minus_exact_ulps" in v), "E_ulps": 256}))
