// narrow.cuh -- narrow phase (query.py:287-346, bounds.py:245-330):
// float32 filter over the leaf-pair list, exact pass over the band, and the
// witness record.
#pragma once

#include "traverse.cuh"

namespace gd {


// exact narrow phase for one triangle pair -> 128-bit key (distance bits,
// tri_a, tri_b): its minimum is the reference's lexicographic witness rule
// (query.py:205-220, 299)
template <bool kMax, int kOrder = -1>
__device__ __forceinline__ Key128 exact_key(const QArgs& q, unsigned ta, unsigned tb) {
  double d;
  if (q.cfg.precision == 32) {
    Tri<float> a = mesh_tri<float, kOrder>(q.ma, ta), b = mesh_tri<float, kOrder>(q.mb, tb);
    float d2 = kMax ? tri_tri_max_d2<Exact<float>, float, false>(a, b, nullptr, nullptr)
                    : tri_tri_min_d2_lean<Exact<float>, float>(a, b);
    d = (double)__fsqrt_rn(d2);
  } else {
    Tri<double> a = mesh_tri<double, kOrder>(q.ma, ta), b = mesh_tri<double, kOrder>(q.mb, tb);
    double d2 = kMax ? tri_tri_max_d2<Exact<double>, double, false>(a, b, nullptr, nullptr)
                     : tri_tri_min_d2_lean<Exact<double>, double>(a, b);
    d = __dsqrt_rn(d2);
  }
  unsigned long long bits = (unsigned long long)__double_as_longlong(d);
  Key128 k;
  k.hi = kMax ? ~bits : bits;  // d >= 0: bit order == value order
  k.lo = ((unsigned long long)ta << 32) | tb;
  return k;
}

__device__ __forceinline__ Key128 shfl_key(Key128 k, int o) {
  Key128 r;
  r.hi = __shfl_xor_sync(0xffffffffu, k.hi, o);
  r.lo = __shfl_xor_sync(0xffffffffu, k.lo, o);
  return r;
}

// Lower bound^2 of the distance between two triangles: the gap between their
// projections on the axis through the centroids (any axis separates at most
// by the distance).  float32, well inside the slack E.
__device__ __forceinline__ float axis_gap_sq(const Tri<float>& a, const Tri<float>& b) {
  const float nx = (b.v[0].x + b.v[1].x + b.v[2].x) - (a.v[0].x + a.v[1].x + a.v[2].x);
  const float ny = (b.v[0].y + b.v[1].y + b.v[2].y) - (a.v[0].y + a.v[1].y + a.v[2].y);
  const float nz = (b.v[0].z + b.v[1].z + b.v[2].z) - (a.v[0].z + a.v[1].z + a.v[2].z);
  const float n2 = fmaf(nx, nx, fmaf(ny, ny, nz * nz));
  if (!(n2 > 0.f)) return 0.f;
  float amax = -INFINITY, bmin = INFINITY;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    amax = fmaxf(amax, fmaf(a.v[i].x, nx, fmaf(a.v[i].y, ny, a.v[i].z * nz)));
    bmin = fminf(bmin, fmaf(b.v[i].x, nx, fmaf(b.v[i].y, ny, b.v[i].z * nz)));
  }
  const float g = bmin - amax;  // gap * |n|
  return g > 0.f ? g * g / n2 : 0.f;
}

// axis_gap_sq(a, b) > ub2 without the division: gap * |n| = bmin - amax along
// n = (sum of b) - (sum of a); gap^2 > ub2  <=>  (gap |n|)^2 > ub2 |n|^2.
__device__ __forceinline__ bool axis_separated(const Tri<float>& a, const Tri<float>& b, const V3<float>& sa,
                                               const V3<float>& sb, float ub2) {
  const float nx = sb.x - sa.x, ny = sb.y - sa.y, nz = sb.z - sa.z;
  float amax = -INFINITY, bmin = INFINITY;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    amax = fmaxf(amax, fmaf(a.v[i].x, nx, fmaf(a.v[i].y, ny, a.v[i].z * nz)));
    bmin = fminf(bmin, fmaf(b.v[i].x, nx, fmaf(b.v[i].y, ny, b.v[i].z * nz)));
  }
  const float g = bmin - amax;
  return g > 0.f && g * g > ub2 * fmaf(nx, nx, fmaf(ny, ny, nz * nz));
}

// ---------------------------------------------------------------------------
// Narrow phase, stage 1 (k_nfilter): one thread per leaf pair.  Re-culls the
// pair with the final traversal bound, loads its 1..2 x 1..2 triangles once (two
// 32-byte leaf records + staged vertices), and keeps the triangle pairs whose
// box bound -- and, for min queries, the centroid-axis separation bound --
// can still beat the bound.
//  * min, normal pass: survivors (leaf rank * 2 + triangle) pairs are
//    appended, warp-aggregated, to the idle front buffer; k_ntest runs the
//    full test on that dense list.
//  * max: the exact test is 9 vertex pairs -- cheaper here, on the loaded
//    triangles, than a candidate round trip.
//  * kRescan (only after a band / candidate overflow): every survivor of the
//    final bound is evaluated in the reference arithmetic right here.
// grid: GD_NFILTER_BLOCKS (min) / GD_NFILTER_BLOCKS_MAX (max) blocks per SM,
// striding over the leaf pairs.  k_nfilter<max> (92 registers, 2 resident
// blocks / SM) runs a short list in its first resident wave only -- the rings'
// max query 0.214 -> 0.199 ms -- and a long one (near-contact scenes) over
// the whole grid, whose later blocks balance the uneven per-pair work
// (nested shells max 304 ms vs 334 ms with 3 blocks / SM throughout).
#ifndef GD_NFILTER_BLOCKS
#define GD_NFILTER_BLOCKS 8
#endif
#ifndef GD_NFILTER_BLOCKS_MAX
#define GD_NFILTER_BLOCKS_MAX 6
#endif
constexpr int kNfilterMaxWave = 2;                 // blocks per SM of the short-list wave
constexpr unsigned long long kNfilterShortList = 1ull << 21;  // leaf pairs
#ifndef GD_NFILTER_THREADS
#define GD_NFILTER_THREADS 256
#endif
constexpr int kNfilterThreads = GD_NFILTER_THREADS;
template <bool kMax, bool kRescan>
__global__ __launch_bounds__(kNfilterThreads) void k_nfilter(QArgs q) {
  grid_dependency_wait();  // programmatic dependent launch (query.cu)
  QState* S = q.S;
  const unsigned long long n = S->n_leaf;
  if (n == 0) return;
  if (kRescan && *reinterpret_cast<volatile int*>(&S->band_overflow) == 0) return;
  if (kRescan && blockIdx.x == 0 && threadIdx.x == 0) S->rescanned = 1;  // read by the k_refine after it
  // this round's leaf-pair list and the candidate list (the arena's gap)
  const uint2* leaves = q.fnode + S->leaf_off;
  const float* keys = q.fkey + S->leaf_off;
  uint2* out = q.fnode + S->cand_off;
  const unsigned long long cand_cap = S->cand_cap;
  const bool culling = q.cfg.culling != 0;
  const XfF32 xa = q.xa, xb = q.xb;
  const int lane = threadIdx.x & 31;
  const float E = S->slack;
  float upd = 0.f;  // max query only
  unsigned long long tested = 0;
  Key128 rbest;  // rescan: this thread's best exact key
  rbest.hi = ~0ull;
  rbest.lo = ~0ull;
  const float fb_rescan = kRescan ? __uint_as_float(*reinterpret_cast<volatile unsigned*>(&S->fbest)) : 0.f;
  unsigned blocks = gridDim.x;
  if (kMax && !kRescan && n <= kNfilterShortList) blocks = max(1u, gridDim.x * kNfilterMaxWave / GD_NFILTER_BLOCKS_MAX);
  if (blockIdx.x >= blocks) return;
  const unsigned long long stride = (unsigned long long)blocks * blockDim.x;
  for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x; base < n; base += stride) {
    const unsigned long long i = base + threadIdx.x;
    const float ub = load_bound(S), ub2 = ub * ub;
    unsigned mask = 0;
    float dd[4] = {-1.f, -1.f, -1.f, -1.f};  // max: float32 distances of the tested pairs
    unsigned tid[4] = {0u, 0u, 0u, 0u};     // max: their (tri_a, tri_b) halves, packed below
    unsigned tib[4] = {0u, 0u, 0u, 0u};
    // the entry is loaded with its key, not after the key test: one dependent
    // round trip less per leaf pair
    const uint2 lp = i < n ? leaves[i] : make_uint2(0, 0);
    const float lkey = i < n ? keys[i] : 0.f;
    if (i < n && (!culling || survives<kMax>(lkey, ub2))) {
      // both leaves' triangles: one contiguous 80-byte load each (leaf_tri)
      const LeafTris ra = load_leaf_tris(q.A, xa, lp.x), rb = load_leaf_tris(q.B, xb, lp.y);
      const int ca = ra.count(), cb = rb.count();
      const Tri<float>* ta = ra.t;
      const Tri<float>* tb = rb.t;
      // per-triangle quantities once, not per pair
      Box ba[2], bb[2];
      V3<float> sa[2], sb[2];  // vertex sums (3 x centroid)
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        ba[t] = tri_box(ta[t]);
        bb[t] = tri_box(tb[t]);
        sa[t] = {ta[t].v[0].x + ta[t].v[1].x + ta[t].v[2].x, ta[t].v[0].y + ta[t].v[1].y + ta[t].v[2].y,
                 ta[t].v[0].z + ta[t].v[1].z + ta[t].v[2].z};
        sb[t] = {tb[t].v[0].x + tb[t].v[1].x + tb[t].v[2].x, tb[t].v[0].y + tb[t].v[1].y + tb[t].v[2].y,
                 tb[t].v[0].z + tb[t].v[1].z + tb[t].v[2].z};
      }
#pragma unroll
      for (int ia = 0; ia < 2; ++ia)
#pragma unroll
        for (int ib = 0; ib < 2; ++ib) {
          if (ia >= ca || ib >= cb) continue;
          bool keep = !culling || survives<kMax>(pair_key<kMax>(ba[ia], bb[ib]), ub2);
          if (!kMax && culling && keep) keep = !axis_separated(ta[ia], tb[ib], sa[ia], sb[ib], ub2);
          if (!keep) continue;
          if (kMax || kRescan) {
            float d, lb;
            if (kMax)
              d = lb = sqrtf(tri_tri_max_d2<Fast<float>, float, false>(ta[ia], tb[ib], nullptr, nullptr));
            else
              tri_tri_min_fast_lb(ta[ia], tb[ib], d, lb);
            if (kMax) upd = fmaxf(upd, d);
            ++tested;
            if (kRescan) {
              // within E of the best float32 distance (k_refine's window, on
              // the conditioning-aware lower bound), the thread keeps its best
              // exact key; one atomic per warp below
              if (kMax ? (d >= fb_rescan - E) : (lb <= fb_rescan + E)) {
                const Key128 k = exact_key<kMax>(q, ra.tri_id(ia), rb.tri_id(ib));
                if (key_less(k, rbest)) rbest = k;
              }
            } else {
              // max: appended below, warp-aggregated
              dd[2 * ia + ib] = d;
              tid[2 * ia + ib] = ra.tri_id(ia);
              tib[2 * ia + ib] = rb.tri_id(ib);
            }
          } else {
            mask |= 1u << (2 * ia + ib);
          }
        }
    }
    if (kMax && !kRescan) {
      // band append, one reservation per warp.  Besides the bound test, a
      // pair more than E below the warp's best float32 distance cannot be the
      // answer (fbest >= that best; k_refine skips f < fbest - E) and stays out
      const float thr = fmaxf(ub, warp_max(upd)) - E;
      unsigned m4 = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (dd[c] >= 0.f && dd[c] >= thr) m4 |= 1u << c;
      const unsigned cnt = __popc(m4);
      unsigned incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      unsigned long long wbase = 0;
      if (lane == 31 && incl) wbase = atomicAdd(&S->n_band, (unsigned long long)incl);
      wbase = __shfl_sync(0xffffffffu, wbase, 31);
      unsigned long long pos = wbase + incl - cnt;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (m4 & (1u << c)) {
          if (pos < q.band_cap) {
            q.band_ids[pos] = make_uint2(tid[c], tib[c]);
            q.band_d[pos] = dd[c];
          } else {
            S->band_overflow = 1;  // the rescan pass covers every leaf pair
          }
          ++pos;
        }
      }
    }
    if (!kMax && !kRescan) {
      // warp-aggregated append of up to 4 triangle pairs per thread
      const unsigned cnt = __popc(mask);
      unsigned incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      unsigned long long wbase = 0;
      if (lane == 31 && incl) wbase = atomicAdd(&S->n_cand, (unsigned long long)incl);
      wbase = __shfl_sync(0xffffffffu, wbase, 31);
      unsigned long long pos = wbase + incl - cnt;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (mask & (1u << c)) {
          if (pos < cand_cap)
            out[pos] = make_uint2(2 * lp.x + (c >> 1), 2 * lp.y + (c & 1));
          else
            S->band_overflow = 1;  // the rescan pass covers every leaf pair
          ++pos;
        }
      }
    }
  }
  if (kMax && !kRescan) {
    upd = warp_max(upd);
    if (lane == 0 && upd > 0.f) {
      commit_bound<kMax>(q, upd);
      atomicMax(&S->fbest, __float_as_uint(upd));
    }
  }
  if (kRescan) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const Key128 other = shfl_key(rbest, o);
      if (key_less(other, rbest)) rbest = other;
    }
    if (lane == 0 && rbest.hi != ~0ull) atomic_min_key(&S->best, rbest);
  }
  if (!kRescan) {
    tested = warp_sum_u64(tested);
    if (lane == 0 && tested) atomicAdd(&S->narrow, tested);
  }
}

// Short candidate lists (min queries) skip the float32 stage: k_refine
// evaluates every candidate in the reference arithmetic right away.  The
// band's float32 window exists to spare exact evaluations when the list is
// long (near-contact scenes: 70M candidates, 38M in the band); on a short
// list the exact pass is one latency-bound wave either way, and the float32
// test before it cost ~35 us on the rings (39K candidates, 29K of them in the
// band).  Exact either way: the candidates are a superset of the band, every
// key is an achieved exact distance, and the optimum pairs are among them.
#ifndef GD_DIRECT_EXACT
#define GD_DIRECT_EXACT (1ull << 18)
#endif
constexpr unsigned long long kDirectExact = GD_DIRECT_EXACT;
__device__ __forceinline__ bool direct_exact(const QState* S) {
  const volatile QState* V = S;
  const unsigned long long n = V->n_cand;
  return n <= kDirectExact && n <= V->cand_cap;  // (a longer list overflowed: the rescan covers it)
}

// Narrow phase, stage 2 (k_ntest, min queries): the float32 triangle-pair
// test on the dense candidate list; updates the bound and fills the band.
template <bool kMax>
__global__ __launch_bounds__(256) void k_ntest(QArgs q) {
  grid_dependency_wait();  // programmatic dependent launch (query.cu)
  QState* S = q.S;
  const unsigned long long n = min(S->n_cand, S->cand_cap);
  if (n == 0 || (!kMax && direct_exact(S))) return;  // a short list: k_refine evaluates it exactly
  if (blockIdx.x * 256ull >= n) return;
  const uint2* cand = q.fnode + S->cand_off;
  const float E = S->slack;
  const XfF32 xa = q.xa, xb = q.xb;
  __shared__ float warp_upd[8];
  float upd = kMax ? 0.f : INFINITY;
  unsigned long long tested = 0;
  const int lane = threadIdx.x & 31;
  // warp-uniform loop (the band append below is warp-aggregated)
  for (unsigned long long base = blockIdx.x * 256ull; base < n; base += gridDim.x * 256ull) {
    const unsigned long long j = base + threadIdx.x;
    float d = kMax ? -1.f : INFINITY, lb = d;
    uint2 ids = make_uint2(0, 0);
    if (j < n) {
      ++tested;
      const uint2 c = cand[j];
      const int ia = c.x & 1, ib = c.y & 1;
      const Tri<float> A = load_leaf_tri(q.A, xa, c.x >> 1, ia), B = load_leaf_tri(q.B, xb, c.y >> 1, ib);
      const float4* pa = reinterpret_cast<const float4*>(q.A.leaf_tri) + 5 * (unsigned long long)(c.x >> 1) + 4;
      const float4* pb = reinterpret_cast<const float4*>(q.B.leaf_tri) + 5 * (unsigned long long)(c.y >> 1) + 4;
      if (kMax) {
        d = lb = sqrtf(tri_tri_max_d2<Fast<float>, float, false>(A, B, nullptr, nullptr));
      } else {
        tri_tri_min_fast_lb(A, B, d, lb);  // d: the float32 estimate; lb: what the band windows on
      }
      upd = kMax ? fmaxf(upd, d) : fminf(upd, d);
      const float4 fa = __ldg(pa), fb = __ldg(pb);  // (the 5th word: tri ids; already in L1)
      ids = make_uint2((unsigned)__float_as_int(ia ? fa.w : fa.z), (unsigned)__float_as_int(ib ? fb.w : fb.z));
    }
    // band: within E of the bound, and within E of the warp's best float32
    // distance (fbest is at least as good; k_refine drops the rest anyway)
    const float ub = load_bound(S);
    const float wu = kMax ? warp_max(upd) : warp_min(upd);  // every lane: a full-warp shuffle
    const bool app = j < n && (kMax ? d >= fmaxf(ub, wu) - E : lb <= fminf(ub, wu) + E);
    const unsigned m = __ballot_sync(0xffffffffu, app);
    unsigned long long wbase = 0;
    if (lane == 0 && m) wbase = atomicAdd(&S->n_band, (unsigned long long)__popc(m));
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (app) {
      const unsigned long long slot = wbase + __popc(m & ((1u << lane) - 1));
      if (slot < q.band_cap) {
        q.band_ids[slot] = ids;
        q.band_d[slot] = lb;
      } else {
        S->band_overflow = 1;  // the rescan pass covers every leaf pair
      }
    }
  }
  upd = kMax ? warp_max(upd) : warp_min(upd);
  tested = warp_sum_u64(tested);
  if ((threadIdx.x & 31) == 0) {
    warp_upd[threadIdx.x >> 5] = upd;
    if (tested) atomicAdd(&S->narrow, tested);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float u = warp_upd[0];
    for (int w = 1; w < 8; ++w) u = kMax ? fmaxf(u, warp_upd[w]) : fminf(u, warp_upd[w]);
    if (kMax ? u > 0.f : u < INFINITY) {
      commit_bound<kMax>(q, u);
      if (kMax)
        atomicMax(&S->fbest, __float_as_uint(u));
      else
        atomicMin(&S->fbest, __float_as_uint(u));
    }
  }
}

// ---------------------------------------------------------------------------
// exact pass over the band: only pairs whose float32 distance can still be
// the answer (|d_fast - d_exact| <= E/2) are re-evaluated in the reference's
// arithmetic; the 128-bit minimum is the answer and its witness.
template <bool kMax>
__device__ void finalize(const QArgs& q);

// Exact pass (k_refine): one thread per band entry.  Entries whose float32
// distance f is more than E from the best float32 distance f_best (S->fbest,
// tracked where the band is filled) are skipped: |f - exact| <= E/2 for every
// pair, so such an entry is exactly worse than the f_best pair (min query;
// mirrored for max).  The rest are re-evaluated in the reference's
// arithmetic (exact_key) and reduced to the lexicographic 128-bit minimum;
// the last block to finish writes the witness and the result record.  The
// grid has far more threads than a band has entries, so the skipped entries
// cost one load each and no compaction pass is needed.
constexpr int kRefineThreads = 64;

// kOrder: the float64 transform's operation order of both meshes
// (GdMesh.xf_order, fixed per process), -1 = read at run time (meshes with
// different orders)
template <bool kMax, int kOrder>
// min: the lean float64 feature loop keeps ~150 registers live (no spills at
// 4 blocks / SM: 41 -> 36 us on the rings); max is short and stays at 12
#ifndef GD_REFINE_MINB
#define GD_REFINE_MINB 4
#endif
__global__ __launch_bounds__(kRefineThreads, kMax ? 12 : GD_REFINE_MINB) void k_refine(QArgs q) {
  grid_dependency_wait();  // programmatic dependent launch (query.cu)
  QState* S = q.S;
  const unsigned long long n = min(S->n_band, q.band_cap);
  // a short candidate list (min): every candidate after the band entries
  // (then only a warm pair), evaluated exactly (direct_exact)
  const bool direct = !kMax && direct_exact(S);
  const unsigned long long n_all = n + (direct ? S->n_cand : 0ull);
  const uint2* cand = q.fnode + S->cand_off;
  if (direct && blockIdx.x == 0 && threadIdx.x == 0 && S->n_cand) atomicAdd(&S->narrow, S->n_cand);
  const float E = S->slack;
  const float fb = __uint_as_float(*reinterpret_cast<volatile unsigned*>(&S->fbest));
  __shared__ Key128 wk[kRefineThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Key128 best;
  best.hi = ~0ull;
  best.lo = ~0ull;
  unsigned long long evals = 0;
  for (unsigned long long j = (unsigned long long)blockIdx.x * kRefineThreads + threadIdx.x; j < n_all;
       j += (unsigned long long)gridDim.x * kRefineThreads) {
    uint2 ids;
    if (j < n) {
      const float f = q.band_d[j];
      ids = q.band_ids[j];  // loaded with f: no second dependent round trip
      if (!(kMax ? f >= fb - E : f <= fb + E)) continue;  // +-inf (warm pair) always passes
    } else {
      // candidate (leaf rank * 2 + triangle) pair -> triangle ids (the 5th
      // word of the leaves' leaf_tri records, as k_ntest reads them)
      const uint2 c = cand[j - n];
      const float4 fa = __ldg(reinterpret_cast<const float4*>(q.A.leaf_tri) + 5 * (unsigned long long)(c.x >> 1) + 4);
      const float4 fb4 = __ldg(reinterpret_cast<const float4*>(q.B.leaf_tri) + 5 * (unsigned long long)(c.y >> 1) + 4);
      ids = make_uint2((unsigned)__float_as_int((c.x & 1) ? fa.w : fa.z),
                       (unsigned)__float_as_int((c.y & 1) ? fb4.w : fb4.z));
    }
    const Key128 k = exact_key<kMax, kOrder>(q, ids.x, ids.y);
    if (key_less(k, best)) best = k;
    ++evals;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key128 other = shfl_key(best, o);
    if (key_less(other, best)) best = other;
  }
  evals = warp_sum_u64(evals);
  if (lane == 0) {
    wk[wid] = best;
    if (evals) atomicAdd(&S->band_eval, evals);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kRefineThreads / 32; ++w)
      if (key_less(wk[w], best)) best = wk[w];
    if (best.hi != ~0ull) atomic_min_key(&S->best, best);
    __threadfence();
    last = atomicAdd(&S->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    finalize<kMax>(q);
  }
}

// ---------------------------------------------------------------------------
// Witness points of one triangle pair, one warp: lane l evaluates feature l
// of the reference's fixed order (9 edge pairs, then A_i->B / B_i->A), the
// warp keeps the first strict optimum, then the 6 pierce tests run in lanes
// 0..5 and the first hit wins -- the sequential semantics of
// bounds.py:245-330 at 1/15 of its latency.
template <typename T>
__device__ __forceinline__ void shfl_v3(V3<T>& v, int src) {
  v.x = __shfl_sync(0xffffffffu, v.x, src);
  v.y = __shfl_sync(0xffffffffu, v.y, src);
  v.z = __shfl_sync(0xffffffffu, v.z, src);
}

template <typename T, bool kMax>
__device__ void warp_witness(const Tri<T>& a, const Tri<T>& b, V3<T>& P, V3<T>& Q) {
  using A = Exact<T>;
  const int lane = threadIdx.x & 31;
  T d2 = kMax ? T(-1) : T(INFINITY);
  V3<T> p{T(0), T(0), T(0)}, qq{T(0), T(0), T(0)};
  if (kMax) {
    if (lane < 9) {
      p = a.v[lane / 3];
      qq = b.v[lane % 3];
      V3<T> w = vsub<A>(p, qq);
      d2 = vdot<A>(w, w);
    }
  } else if (lane < 9) {
    const int i = lane / 3, j = lane % 3;
    segment_pair<A>(a.v[i], vsub<A>(a.v[(i + 1) % 3], a.v[i]), b.v[j], vsub<A>(b.v[(j + 1) % 3], b.v[j]), p, qq);
    V3<T> w = vsub<A>(p, qq);
    d2 = vdot<A>(w, w);
  } else if (lane < 15) {
    const int i = (lane - 9) >> 1;
    if (((lane - 9) & 1) == 0) {
      p = a.v[i];
      qq = point_triangle<A>(a.v[i], b.v[0], b.v[1], b.v[2]);
    } else {
      qq = b.v[i];
      p = point_triangle<A>(b.v[i], a.v[0], a.v[1], a.v[2]);
    }
    V3<T> w = vsub<A>(p, qq);
    d2 = vdot<A>(w, w);
  }
  // first strict optimum in feature order == (d2, lane) lexicographic
  T bd = d2;
  int bl = lane;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T od = __shfl_xor_sync(0xffffffffu, bd, o);
    const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
    if ((kMax ? od > bd : od < bd) || (od == bd && ol < bl)) {
      bd = od;
      bl = ol;
    }
  }
  shfl_v3(p, bl);
  shfl_v3(qq, bl);
  if (!kMax && bd > T(0)) {
    bool hit = false;
    V3<T> x{T(0), T(0), T(0)};
    if (lane < 6) {
      const int i = lane >> 1;
      hit = (lane & 1) == 0 ? pierce<A>(a.v[i], a.v[(i + 1) % 3], b.v[0], b.v[1], b.v[2], x)
                            : pierce<A>(b.v[i], b.v[(i + 1) % 3], a.v[0], a.v[1], a.v[2], x);
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (m) {
      const int src = __ffs(m) - 1;
      shfl_v3(x, src);
      p = x;
      qq = x;
    }
  }
  P = p;
  Q = qq;
}

template <bool kMax>
__device__ void finalize(const QArgs& q) {
  QState* S = q.S;
  Key128 best;
  best.hi = reinterpret_cast<volatile unsigned long long*>(&S->best)[0];
  best.lo = reinterpret_cast<volatile unsigned long long*>(&S->best)[1];
  const bool found = !(best.hi == ~0ull && best.lo == ~0ull);
  const unsigned ta = (unsigned)(best.lo >> 32), tb = (unsigned)(best.lo & 0xffffffffu);
  double pa[3] = {0, 0, 0}, pb[3] = {0, 0, 0};
  if (found) {
    if (q.cfg.precision == 32) {
      Tri<float> a = mesh_tri<float>(q.ma, ta), b = mesh_tri<float>(q.mb, tb);
      V3<float> p, qq;
      warp_witness<float, kMax>(a, b, p, qq);
      pa[0] = p.x; pa[1] = p.y; pa[2] = p.z;
      pb[0] = qq.x; pb[1] = qq.y; pb[2] = qq.z;
    } else {
      Tri<double> a = mesh_tri<double>(q.ma, ta), b = mesh_tri<double>(q.mb, tb);
      V3<double> p, qq;
      warp_witness<double, kMax>(a, b, p, qq);
      pa[0] = p.x; pa[1] = p.y; pa[2] = p.z;
      pb[0] = qq.x; pb[1] = qq.y; pb[2] = qq.z;
    }
  }
  if (threadIdx.x != 0) return;
  GdResult r;
  memset(&r, 0, sizeof(r));
  r.status = S->err;
  r.iterations = min(S->iter, kMaxIters);
  r.expanded_pairs = (long long)S->expanded;
  r.narrow_pairs = (long long)S->narrow;
  r.band_pairs = (long long)S->band_eval;
  r.overflow_candidates = S->ov_cand;
  r.overflow_front_in = S->ov_in;
  r.overflow_cap = S->ov_cap;
  r.rounds = S->rounds;
  // bit 0: levels remain (another traversal round); bit 1: the band or the
  // candidate list overflowed and no rescan has covered it yet -- the record
  // is not final, query_round runs the rescan pass and this exact pass again
  r.pending = S->pending |
              (*reinterpret_cast<volatile int*>(&S->band_overflow) && !*reinterpret_cast<volatile int*>(&S->rescanned)
                   ? 2
                   : 0);
  if (!found) {
    r.tri_a = r.tri_b = -1;
    const float b = load_bound(S);
    r.distance = kMax ? (double)b + (double)S->slack : (double)b - (double)S->slack;
    r.witness_distance = r.distance;
  } else {
    const unsigned long long bits = kMax ? ~best.hi : best.hi;
    r.distance = __longlong_as_double((long long)bits);
    r.witness_distance = r.distance;
    r.tri_a = ta;
    r.tri_b = tb;
    for (int c = 0; c < 3; ++c) {
      r.point_a[c] = pa[c];
      r.point_b[c] = pb[c];
    }
  }
  S->res = r;
  if (q.result) *q.result = r;
}

}  // namespace gd
