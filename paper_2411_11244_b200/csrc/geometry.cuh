// geometry.cuh -- box bounds and the triangle-triangle narrow phase.
//
// The narrow phase is written once and instantiated twice:
//   Exact<T>  (T = double / float): IEEE round-to-nearest, no FMA, in the
//             reference's operation order -> bitwise equal to
//             bounds.batch_tri_tri_min / batch_tri_tri_max (bounds.py:245-330)
//   Fast<float>: same algorithm, FMA-contracted; the traversal's filter.
#pragma once

#include "common.cuh"

namespace gd {

// num/den clamped to [0, 1]; 0 when den == 0 (bounds.py:146-150)
template <typename A, typename T>
__device__ __forceinline__ T clamp_ratio(T num, T den) {
  T r = (den != T(0)) ? A::div(num, den) : T(0);
  r = r > T(0) ? r : T(0);  // np.clip(x, 0, 1) = min(max(x, 0), 1)
  return r < T(1) ? r : T(1);
}

// Lumelsky clamped closest points of p0 + t u and q0 + s v (bounds.py:153-169)
template <typename A, typename T>
__device__ __forceinline__ void segment_pair(V3<T> p0, V3<T> u, V3<T> q0, V3<T> v, V3<T>& p,
                                             V3<T>& q) {
  V3<T> w = vsub<A>(q0, p0);
  T uu = vdot<A>(u, u), vv = vdot<A>(v, v), uv = vdot<A>(u, v);
  T uw = vdot<A>(u, w), vw = vdot<A>(v, w);
  T t = clamp_ratio<A>(A::sub(A::mul(uw, vv), A::mul(vw, uv)), A::sub(A::mul(uu, vv), A::mul(uv, uv)));
  T s = clamp_ratio<A>(A::sub(A::mul(t, uv), vw), vv);
  t = clamp_ratio<A>(A::add(A::mul(s, uv), uw), uu);
  p = vmadd<A>(p0, t, u);
  q = vmadd<A>(q0, s, v);
}

// Closest point on triangle abc to p, Ericson's Voronoi walk with guarded
// divisions; first matching region wins (bounds.py:172-221)
template <typename A, typename T>
__device__ __forceinline__ V3<T> point_triangle(V3<T> p, V3<T> a, V3<T> b, V3<T> c) {
  V3<T> ab = vsub<A>(b, a), ac = vsub<A>(c, a), ap = vsub<A>(p, a);
  T d1 = vdot<A>(ab, ap), d2 = vdot<A>(ac, ap);
  V3<T> bp = vsub<A>(p, b);
  T d3 = vdot<A>(ab, bp), d4 = vdot<A>(ac, bp);
  V3<T> cp = vsub<A>(p, c);
  T d5 = vdot<A>(ab, cp), d6 = vdot<A>(ac, cp);
  T vc = A::sub(A::mul(d1, d4), A::mul(d3, d2));
  T vb = A::sub(A::mul(d5, d2), A::mul(d1, d6));
  T va = A::sub(A::mul(d3, d6), A::mul(d5, d4));
  if (d1 <= T(0) && d2 <= T(0)) return a;
  if (d3 >= T(0) && d4 <= d3) return b;
  if (vc <= T(0) && d1 >= T(0) && d3 <= T(0)) return vmadd<A>(a, clamp_ratio<A>(d1, A::sub(d1, d3)), ab);
  if (d6 >= T(0) && d5 <= d6) return c;
  if (vb <= T(0) && d2 >= T(0) && d6 <= T(0)) return vmadd<A>(a, clamp_ratio<A>(d2, A::sub(d2, d6)), ac);
  T e43 = A::sub(d4, d3), e56 = A::sub(d5, d6);
  if (va <= T(0) && e43 >= T(0) && e56 >= T(0))
    return vmadd<A>(b, clamp_ratio<A>(e43, A::add(e43, e56)), vsub<A>(c, b));
  T total = A::add(A::add(va, vb), vc);
  if (total == T(0)) return vmadd<A>(a, clamp_ratio<A>(d1, A::sub(d1, d3)), ab);
  T inv = A::div(T(1), total);
  return vmadd<A>(vmadd<A>(a, A::mul(vb, inv), ab), A::mul(vc, inv), ac);
}

// transversal segment-through-triangle test (bounds.py:224-242)
template <typename A, typename T>
__device__ __forceinline__ bool pierce(V3<T> s0, V3<T> s1, V3<T> a, V3<T> b, V3<T> c, V3<T>& x) {
  V3<T> ba = vsub<A>(b, a);
  V3<T> n = vcross<A>(ba, vsub<A>(c, a));
  V3<T> d = vsub<A>(s1, s0);
  T den = vdot<A>(n, d);
  bool ok = den != T(0);
  T t = ok ? A::div(vdot<A>(n, vsub<A>(a, s0)), den) : T(0);
  ok = ok && t >= T(0) && t <= T(1);
  x = vmadd<A>(s0, t, d);
  ok = ok && vdot<A>(n, vcross<A>(ba, vsub<A>(x, a))) >= T(0);
  ok = ok && vdot<A>(n, vcross<A>(vsub<A>(c, b), vsub<A>(x, b))) >= T(0);
  ok = ok && vdot<A>(n, vcross<A>(vsub<A>(a, c), vsub<A>(x, c))) >= T(0);
  return ok;
}

template <typename T> struct Tri {
  V3<T> v[3];
};

// Exact minimum distance^2 + witness points (bounds.py:245-306).  Returns the
// squared distance; the caller takes sqrt (the reference does sqrt last).
template <typename A, typename T, bool kPoints>
__device__ __forceinline__ T tri_tri_min_d2(const Tri<T>& t1, const Tri<T>& t2, V3<T>* bp, V3<T>* bq) {
  T best = T(INFINITY);
  V3<T> P{T(0), T(0), T(0)}, Q{T(0), T(0), T(0)};
  auto offer = [&](V3<T> p, V3<T> q) {
    V3<T> w = vsub<A>(p, q);
    T d2 = vdot<A>(w, w);
    if (d2 < best) {
      best = d2;
      if (kPoints) {
        P = p;
        Q = q;
      }
    }
  };
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    V3<T> pa = t1.v[i], ua = vsub<A>(t1.v[(i + 1) % 3], pa);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      V3<T> qb = t2.v[j], vb = vsub<A>(t2.v[(j + 1) % 3], qb);
      V3<T> p, q;
      segment_pair<A>(pa, ua, qb, vb, p, q);
      offer(p, q);
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    offer(t1.v[i], point_triangle<A>(t1.v[i], t2.v[0], t2.v[1], t2.v[2]));
    offer(point_triangle<A>(t2.v[i], t1.v[0], t1.v[1], t1.v[2]), t2.v[i]);
  }
  if (best > T(0)) {
    bool hit = false;
    V3<T> pt{T(0), T(0), T(0)};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      V3<T> x;
      bool h = pierce<A>(t1.v[i], t1.v[(i + 1) % 3], t2.v[0], t2.v[1], t2.v[2], x);
      if (h && !hit) pt = x;
      hit = hit || h;
      h = pierce<A>(t2.v[i], t2.v[(i + 1) % 3], t1.v[0], t1.v[1], t1.v[2], x);
      if (h && !hit) pt = x;
      hit = hit || h;
    }
    if (hit) {
      best = T(0);
      P = pt;
      Q = pt;
    }
  }
  if (kPoints) {
    *bp = P;
    *bq = Q;
  }
  return best;
}

// ---------------------------------------------------------------------------
// float32 filter with a conditioning-aware LOWER BOUND.
// A float32 closest-point pair always lies on the triangles (up to rounding),
// so a float32 feature distance never UNDERestimates by more than a few ulps;
// but it can OVERestimate when the closest points are ill-conditioned: the
// Lumelsky solve of nearly parallel edges (its 2x2 determinant is
// |u|^2 |v|^2 sin^2 theta) and the barycentric solve of a point over a thin or
// distant triangle.  Measured on adversarial pairs (scripts/exp_narrow_error.py):
// up to ~290 float32 ulps of the coordinate scale for near-contact pairs,
// beyond the exact band's E / 2 = 128.  Each feature therefore also gets a
// first-order bound D of the displacement of its computed closest point; the
// distance excess along the (convex) feature profile is at most D when the
// distance is below 2 D, else D^2 / (2 (d - D)).  lb = min over features of
// (d - excess) (0 when a pierce is found) is what the exact band admits and
// k_refine windows on; d itself still feeds the bound and f_best.
constexpr float kU32 = 0x1p-24f;  // float32 unit roundoff

__device__ __forceinline__ float feature_excess(float d, float disp) {
  return d > 2.f * disp ? disp * disp / (2.f * (d - disp)) : disp;
}

// Lumelsky (segment_pair) in float32 + the displacement bound of its result
__device__ __forceinline__ void segment_pair_lb(V3<float> p0, V3<float> u, V3<float> q0, V3<float> v,
                                                V3<float>& p, V3<float>& q, float& disp) {
  using A = Fast<float>;
  V3<float> w = vsub<A>(q0, p0);
  const float uu = vdot<A>(u, u), vv = vdot<A>(v, v), uv = vdot<A>(u, v);
  const float uw = vdot<A>(u, w), vw = vdot<A>(v, w);
  const float num = uw * vv - vw * uv, den = uu * vv - uv * uv;
  float t = clamp_ratio<A>(num, den);
  const float s = clamp_ratio<A>(t * uv - vw, vv);
  t = clamp_ratio<A>(s * uv + uw, uu);
  p = vmadd<A>(p0, t, u);
  q = vmadd<A>(q0, s, v);
  // first-step parameter error: dot products carry <= 3 u |.||.|, the
  // differences of products <= 2 u more; x2 safety (16 u below)
  if (!(uu > 0.f && vv > 0.f)) {  // a point: the projections are 1D, well conditioned
    disp = 0.f;
    return;
  }
  const float lu = sqrtf(uu), lv = sqrtf(vv), lw = sqrtf(vdot<A>(w, w));
  const float dden = 16.f * kU32 * uu * vv;
  const float dnum = 16.f * kU32 * lw * (lu * vv + lv * fabsf(uv));
  float dt = 1.f;
  if (den > dden) dt = fminf(1.f, (dnum + fabsf(num) / den * dden) / (den - dden));
  const float sin2 = fminf(1.f, (den + dden) / (uu * vv));
  // (both computed points lie on their segments: never more than |u| + |v|)
  disp = fminf(2.f * dt * fmaxf(lu, lv) * sqrtf(fmaxf(sin2, 0.f)), lu + lv);
}

// point_triangle in float32 + the displacement bound of the closest point
__device__ __forceinline__ V3<float> point_triangle_lb(V3<float> p, V3<float> a, V3<float> b, V3<float> c,
                                                       float& disp) {
  using A = Fast<float>;
  const V3<float> q = point_triangle<A>(p, a, b, c);
  const V3<float> ab = vsub<A>(b, a), ac = vsub<A>(c, a), bc = vsub<A>(c, b);
  const V3<float> ap = vsub<A>(p, a), bp = vsub<A>(p, b), cp = vsub<A>(p, c);
  const float L = sqrtf(fmaxf(fmaxf(vdot<A>(ab, ab), vdot<A>(ac, ac)), vdot<A>(bc, bc)));
  const float R = sqrtf(fmaxf(fmaxf(vdot<A>(ap, ap), vdot<A>(bp, bp)), vdot<A>(cp, cp)));
  const V3<float> n = vcross<A>(ab, ac);
  const float tot = vdot<A>(n, n);                   // |ab x ac|^2, the solve's determinant
  const float dtot = 64.f * kU32 * L * L * R * R;    // its error as computed from the d_i products
  // barycentric error (x2 safety) times the edge length -- but the computed
  // point lies on the triangle in every region (interior barycentrics are
  // positive ratios of a common sum, edges / vertices are clamped), so it is
  // never farther than the triangle's diameter L from the true closest point
  disp = tot > 2.f * dtot ? fminf(2.f * 2.f * 32.f * kU32 * L * L * R * R / (tot - dtot) * L, L) : L;
  return q;
}

__device__ __forceinline__ void tri_tri_min_fast_lb(const Tri<float>& t1, const Tri<float>& t2, float& d,
                                                    float& lb) {
  using A = Fast<float>;
  float best = INFINITY, blb = INFINITY;
  auto offer = [&](V3<float> p, V3<float> q, float disp) {
    const V3<float> w = vsub<A>(p, q);
    const float d2 = vdot<A>(w, w), df = sqrtf(d2);
    best = fminf(best, d2);
    blb = fminf(blb, df - feature_excess(df, disp));
  };
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const V3<float> pa = t1.v[i], ua = vsub<A>(t1.v[(i + 1) % 3], pa);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const V3<float> qb = t2.v[j], vb = vsub<A>(t2.v[(j + 1) % 3], qb);
      V3<float> p, q;
      float disp;
      segment_pair_lb(pa, ua, qb, vb, p, q, disp);
      offer(p, q, disp);
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float disp;
    V3<float> q = point_triangle_lb(t1.v[i], t2.v[0], t2.v[1], t2.v[2], disp);
    offer(t1.v[i], q, disp);
    q = point_triangle_lb(t2.v[i], t1.v[0], t1.v[1], t1.v[2], disp);
    offer(q, t2.v[i], disp);
  }
  if (best > 0.f) {
    bool hit = false;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      V3<float> x;
      hit = hit || pierce<A>(t1.v[i], t1.v[(i + 1) % 3], t2.v[0], t2.v[1], t2.v[2], x);
      hit = hit || pierce<A>(t2.v[i], t2.v[(i + 1) % 3], t1.v[0], t1.v[1], t1.v[2], x);
    }
    if (hit) best = 0.f;
  }
  d = sqrtf(best);
  lb = best == 0.f ? 0.f : fmaxf(fminf(blb, d), 0.f);
}

// The same minimum distance^2 without witness points, features evaluated one
// at a time (no unrolling): a fraction of the registers, so many more warps
// per SM hide the float64 latency of the exact pass.  The minimum over the
// features does not depend on their order, so the value equals
// tri_tri_min_d2's bit for bit.
template <typename T>
__device__ __forceinline__ V3<T> pick3(int i, const V3<T>& a, const V3<T>& b, const V3<T>& c) {
  return i == 0 ? a : (i == 1 ? b : c);
}
template <typename A, typename T>
__device__ __noinline__ T tri_tri_min_d2_lean(const Tri<T> t1, const Tri<T> t2) {
  T best = T(INFINITY);
#pragma unroll 1
  for (int f = 0; f < 9; ++f) {
    const int i = f / 3, j = f - 3 * (f / 3);
    const V3<T> pa = pick3(i, t1.v[0], t1.v[1], t1.v[2]), pa1 = pick3(i == 2 ? 0 : i + 1, t1.v[0], t1.v[1], t1.v[2]);
    const V3<T> qb = pick3(j, t2.v[0], t2.v[1], t2.v[2]), qb1 = pick3(j == 2 ? 0 : j + 1, t2.v[0], t2.v[1], t2.v[2]);
    V3<T> p, q;
    segment_pair<A>(pa, vsub<A>(pa1, pa), qb, vsub<A>(qb1, qb), p, q);
    const V3<T> w = vsub<A>(p, q);
    const T d2 = vdot<A>(w, w);
    best = d2 < best ? d2 : best;
  }
#pragma unroll 1
  for (int f = 0; f < 6; ++f) {
    const bool a_to_b = (f & 1) == 0;
    const int i = f >> 1;
    const Tri<T>& src = a_to_b ? t1 : t2;
    const Tri<T>& dst = a_to_b ? t2 : t1;
    const V3<T> p = pick3(i, src.v[0], src.v[1], src.v[2]);
    const V3<T> q = point_triangle<A>(p, dst.v[0], dst.v[1], dst.v[2]);
    const V3<T> w = vsub<A>(p, q);
    const T d2 = vdot<A>(w, w);
    best = d2 < best ? d2 : best;
  }
  if (best > T(0)) {
#pragma unroll 1
    for (int f = 0; f < 6; ++f) {
      const bool a_edge = (f & 1) == 0;
      const int i = f >> 1;
      const Tri<T>& e = a_edge ? t1 : t2;
      const Tri<T>& tr = a_edge ? t2 : t1;
      V3<T> x;
      if (pierce<A>(pick3(i, e.v[0], e.v[1], e.v[2]), pick3(i == 2 ? 0 : i + 1, e.v[0], e.v[1], e.v[2]), tr.v[0],
                    tr.v[1], tr.v[2], x)) {
        best = T(0);
        break;
      }
    }
  }
  return best;
}

// Exact maximum distance^2 over the 9 vertex pairs, first strict max
// (bounds.py:309-330)
template <typename A, typename T, bool kPoints>
__device__ __forceinline__ T tri_tri_max_d2(const Tri<T>& t1, const Tri<T>& t2, V3<T>* bp, V3<T>* bq) {
  T best = T(-1);
  int bi = 0, bj = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      V3<T> w = vsub<A>(t1.v[i], t2.v[j]);
      T d2 = vdot<A>(w, w);
      if (d2 > best) {
        best = d2;
        bi = i;
        bj = j;
      }
    }
  if (kPoints) {
    *bp = t1.v[bi];
    *bq = t2.v[bj];
  }
  return best;
}

// ---------------------------------------------------------------------------
// box bounds, float32 traversal versions (bounds.py:47-101, Eqs. 5-10).
// The enhanced bounds use the closed form of the 36 face-pair min/max
// (equal to the pairwise evaluation: DESIGN.md "Enhanced bounds").
// ---------------------------------------------------------------------------
struct Box {
  float lo[3], hi[3];
};

__device__ __forceinline__ float box_min_lower_sq(const Box& a, const Box& b) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float g = fmaxf(fmaxf(a.lo[k] - b.hi[k], b.lo[k] - a.hi[k]), 0.f);
    s = fmaf(g, g, s);
  }
  return s;
}

__device__ __forceinline__ float box_max_upper_sq(const Box& a, const Box& b) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float h = fmaxf(fabsf(a.lo[k] - b.hi[k]), fabsf(a.hi[k] - b.lo[k]));
    s = fmaf(h, h, s);
  }
  return s;
}

// Eq. 9: min over face pairs of the face-rectangle max distance.
__device__ __forceinline__ float box_enhanced_min_upper_sq(const Box& a, const Box& b) {
  float H2[3], PA2[3], PB2[3], PP2[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float al = a.lo[k], ah = a.hi[k], bl = b.lo[k], bh = b.hi[k];
    float H = fmaxf(fabsf(al - bh), fabsf(ah - bl));
    float pa = fminf(fmaxf(fabsf(al - bl), fabsf(al - bh)), fmaxf(fabsf(ah - bl), fabsf(ah - bh)));
    float pb = fminf(fmaxf(fabsf(al - bl), fabsf(ah - bl)), fmaxf(fabsf(al - bh), fabsf(ah - bh)));
    float pp = fminf(fminf(fabsf(al - bl), fabsf(al - bh)), fminf(fabsf(ah - bl), fabsf(ah - bh)));
    H2[k] = H * H;
    PA2[k] = pa * pa;
    PB2[k] = pb * pb;
    PP2[k] = pp * pp;
  }
  float best = PP2[0] + H2[1] + H2[2];
  best = fminf(best, H2[0] + PP2[1] + H2[2]);
  best = fminf(best, H2[0] + H2[1] + PP2[2]);
  // alpha != beta, gamma the third axis
  best = fminf(best, PA2[0] + PB2[1] + H2[2]);
  best = fminf(best, PA2[0] + H2[1] + PB2[2]);
  best = fminf(best, PB2[0] + PA2[1] + H2[2]);
  best = fminf(best, H2[0] + PA2[1] + PB2[2]);
  best = fminf(best, PB2[0] + H2[1] + PA2[2]);
  best = fminf(best, H2[0] + PB2[1] + PA2[2]);
  return best;
}

// Eq. 10: max over face pairs of the face-rectangle min distance.
__device__ __forceinline__ float box_enhanced_max_lower_sq(const Box& a, const Box& b) {
  float G2[3], QA2[3], QB2[3], QQ2[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float al = a.lo[k], ah = a.hi[k], bl = b.lo[k], bh = b.hi[k];
    float G = fmaxf(fmaxf(al - bh, bl - ah), 0.f);
    float qa = fmaxf(fmaxf(fmaxf(bl - al, al - bh), fmaxf(bl - ah, ah - bh)), 0.f);
    float qb = fmaxf(fmaxf(fmaxf(al - bl, bl - ah), fmaxf(al - bh, bh - ah)), 0.f);
    float qq = fmaxf(fmaxf(fabsf(al - bl), fabsf(al - bh)), fmaxf(fabsf(ah - bl), fabsf(ah - bh)));
    G2[k] = G * G;
    QA2[k] = qa * qa;
    QB2[k] = qb * qb;
    QQ2[k] = qq * qq;
  }
  float best = QQ2[0] + G2[1] + G2[2];
  best = fmaxf(best, G2[0] + QQ2[1] + G2[2]);
  best = fmaxf(best, G2[0] + G2[1] + QQ2[2]);
  best = fmaxf(best, QA2[0] + QB2[1] + G2[2]);
  best = fmaxf(best, QA2[0] + G2[1] + QB2[2]);
  best = fmaxf(best, QB2[0] + QA2[1] + G2[2]);
  best = fmaxf(best, G2[0] + QA2[1] + QB2[2]);
  best = fmaxf(best, QB2[0] + G2[1] + QA2[2]);
  best = fmaxf(best, G2[0] + QB2[1] + QA2[2]);
  return best;
}

__device__ __forceinline__ float box_min_lower(const Box& a, const Box& b) { return sqrtf(box_min_lower_sq(a, b)); }
__device__ __forceinline__ float box_max_upper(const Box& a, const Box& b) { return sqrtf(box_max_upper_sq(a, b)); }

}  // namespace gd
