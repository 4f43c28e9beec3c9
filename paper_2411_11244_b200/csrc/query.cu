// query.cu -- BVTT front traversal on the device (query.py:266-568).
//
// One query = a fixed launch sequence that never returns to the host:
//   k_init            root bounds, slack, root front           (query.py:454-509)
//   k_expand x D      one adaptive-depth expansion per launch   (query.py:349-451)
//                     (D = max tree depth bounds the iteration count; launches
//                      after the front empties exit immediately)
//   k_narrow          fast float32 narrow phase over the leaf-pair list,
//                     fills the exact-pass band                 (query.py:287-346)
//   k_refine          exact narrow phase (reference arithmetic, 64 or 32 bit)
//                     over the band, lexicographic 128-bit key minimum
//   k_final           witness points, result record
// The bound is a float32 cell carrying a slack E:
// culling is conservative, so every pair that can attain the reference's
// exact answer reaches the exact pass.
#include <algorithm>

#include "engine.cuh"

namespace gd {

constexpr int kExpandThreads = 256;
constexpr int kExpandItems = 4;
constexpr int kExpandTile = kExpandThreads * kExpandItems;
constexpr int kNarrowThreads = 256;

__device__ __forceinline__ float load_bound(const QState* S) {
  return __uint_as_float(*reinterpret_cast<const volatile unsigned int*>(&S->bound_bits));
}

template <bool kMax>
__device__ __forceinline__ void commit_bound(QState* S, float v) {
  if (kMax)
    atomic_max_pos(&S->bound_bits, v - S->slack);
  else
    atomic_min_pos(&S->bound_bits, v + S->slack);
}

// block-wide exclusive scan of small counts (blockDim.x == 256)
__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* warp_tot, unsigned& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  unsigned off = 0, tot = 0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) {
    unsigned t = warp_tot[w];
    if (w < wid) off += t;
    tot += t;
  }
  total = tot;
  return off + x - v;
}

// exact narrow phase for one triangle pair -> 128-bit key
template <bool kMax>
__device__ __forceinline__ Key128 exact_key(const QArgs& q, unsigned ta, unsigned tb) {
  double d;
  if (q.cfg.precision == 32) {
    Tri<float> a = mesh_tri<float>(q.ma, ta), b = mesh_tri<float>(q.mb, tb);
    float d2 = kMax ? tri_tri_max_d2<Exact<float>, float, false>(a, b, nullptr, nullptr)
                    : tri_tri_min_d2<Exact<float>, float, false>(a, b, nullptr, nullptr);
    d = (double)__fsqrt_rn(d2);
  } else {
    Tri<double> a = mesh_tri<double>(q.ma, ta), b = mesh_tri<double>(q.mb, tb);
    double d2 = kMax ? tri_tri_max_d2<Exact<double>, double, false>(a, b, nullptr, nullptr)
                     : tri_tri_min_d2<Exact<double>, double, false>(a, b, nullptr, nullptr);
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

// ---------------------------------------------------------------------------
template <bool kMax>
__global__ void k_init(QArgs q) {
  if (threadIdx.x != 0) return;
  QState* S = q.S;
  Box ra = load_box(q.A.box, 0), rb = load_box(q.B.box, 0);
  float M = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    M = fmaxf(M, fmaxf(fmaxf(fabsf(ra.lo[k]), fabsf(ra.hi[k])), fmaxf(fabsf(rb.lo[k]), fabsf(rb.hi[k]))));
  // slack: 256 float32 ulps of the largest coordinate
  const float E = M * 0x1p-15f;
  S->slack = E;
  float key0, b0;
  if (kMax) {
    key0 = box_max_upper(ra, rb);
    b0 = q.cfg.enhanced_bounds ? box_enhanced_max_lower(ra, rb) : box_min_lower(ra, rb);
    S->bound_bits = __float_as_uint(fmaxf(b0 - E, 0.f));
  } else {
    key0 = box_min_lower(ra, rb);
    b0 = q.cfg.enhanced_bounds ? box_enhanced_min_upper(ra, rb) : box_max_upper(ra, rb);
    S->bound_bits = __float_as_uint(b0 + E);
  }
  S->best.hi = ~0ull;
  S->best.lo = ~0ull;
  S->done = 0;
  S->err = 0;
  S->cur = 0;
  S->depth_a = 0;
  S->depth_b = 0;
  S->iter = 0;
  S->leaf_buf = 1;
  S->n_out = 0;
  S->n_leaf = 0;
  S->n_band = 0;
  S->expanded = 0;
  S->narrow = 0;
  S->culled = 0;
  S->band_eval = 0;
  S->band_overflow = 0;
  S->ov_cand = S->ov_in = S->ov_cap = 0;
  q.node[0][0] = make_uint2(0, 0);
  q.key[0][0] = key0;
  if (q.A.depth == 0 && q.B.depth == 0) {
    // both roots are leaves: narrow phase immediately (query.py:510-518)
    q.node[1][0] = make_uint2(0, 0);
    q.key[1][0] = key0;
    S->n_leaf = 1;
    S->n_in = 0;
    GdIterStat st;
    st.k = 0;
    st.front_in = 1;
    st.front_out = 0;
    st.culled = 0;
    st.bound_after = b0;
    st._pad = 0;
    S->stats[0] = st;
    S->iter = 1;
  } else {
    S->n_in = 1;
  }
  if (q.cfg.warm_a >= 0) {
    // warm_pair seeds the bound with one exact pair (query.py:494-502)
    unsigned ta = (unsigned)q.cfg.warm_a, tb = (unsigned)q.cfg.warm_b;
    const int32_t* ia = q.ma.tri + 3 * (long long)ta;
    const int32_t* ib = q.mb.tri + 3 * (long long)tb;
    Tri<float> a = load_tri32(q.A, make_int4(ia[0], ia[1], ia[2], 0));
    Tri<float> b = load_tri32(q.B, make_int4(ib[0], ib[1], ib[2], 0));
    float d = kMax ? sqrtf(tri_tri_max_d2<Fast<float>, float, false>(a, b, nullptr, nullptr))
                   : sqrtf(tri_tri_min_d2<Fast<float>, float, false>(a, b, nullptr, nullptr));
    commit_bound<kMax>(S, d);
    q.band_ids[0] = make_uint2(ta, tb);
    q.band_d[0] = d;
    S->n_band = 1;
  }
}

// ---------------------------------------------------------------------------
// one expansion sweep (query.py:349-451, Alg. 2).  Candidate t of the
// ncand = n_in << (ka+kb) candidates maps to entry t >> (ka+kb); the low bits
// pick the two descendants ((node+1) << k) - 1 + offset.
template <bool kMax>
__global__ __launch_bounds__(kExpandThreads) void k_expand(QArgs q) {
  QState* S = q.S;
  const unsigned long long n_in = S->n_in;
  if (n_in == 0) return;
  __shared__ unsigned warp_tot[kExpandThreads / 32];
  __shared__ unsigned long long out_base;
  __shared__ float warp_upd[kExpandThreads / 32];
  __shared__ unsigned long long red_culled[kExpandThreads / 32];

  const int ra = q.A.depth - S->depth_a, rb = q.B.depth - S->depth_b;
  const int rem = max(ra, rb);
  const int k = adaptive_k(n_in, q.cfg.front_cap, q.cfg.depth_cap, rem);
  const int ka = min(k, ra), kb = min(k, rb), sh = ka + kb;
  const bool to_leaves = (k == rem);
  const unsigned long long ncand = n_in << sh;
  const bool overflow = ncand > (unsigned long long)q.cfg.front_hard_cap;
  const int cur = S->cur;
  const uint2* __restrict__ in_node = q.node[cur];
  const float* __restrict__ in_key = q.key[cur];
  uint2* out_node = q.node[cur ^ 1];
  float* out_key = q.key[cur ^ 1];
  const unsigned long long leaf_a0 = (1ull << q.A.depth) - 1, leaf_b0 = (1ull << q.B.depth) - 1;
  const unsigned long long off_mask = (1ull << sh) - 1, mask_b = (1ull << kb) - 1;
  const bool culling = q.cfg.culling != 0, enh = q.cfg.enhanced_bounds != 0;
  unsigned long long my_culled = 0;

  if (!overflow) {
    for (unsigned long long tile = blockIdx.x; tile * kExpandTile < ncand; tile += gridDim.x) {
      const unsigned long long base = tile * kExpandTile;
      const float ub = load_bound(S);  // one bound snapshot per tile (query.py:396)
      float upd = kMax ? 0.f : INFINITY;
      uint2 on[kExpandItems];
      float ok[kExpandItems];
      unsigned keep_mask = 0;
#pragma unroll
      for (int it = 0; it < kExpandItems; ++it) {
        const unsigned long long t = base + (unsigned long long)it * kExpandThreads + threadIdx.x;
        if (t >= ncand) continue;
        const unsigned long long e = t >> sh, off = t & off_mask;
        const float pk = __ldg(in_key + e);
        // stale-entry re-cull: descendants' keys are monotone in the parent's
        if (culling && (kMax ? pk < ub : pk > ub)) {
          ++my_culled;
          continue;
        }
        const uint2 nd = __ldg(in_node + e);
        const unsigned long long na = (((unsigned long long)nd.x + 1) << ka) - 1 + (off >> kb);
        const unsigned long long nb = (((unsigned long long)nd.y + 1) << kb) - 1 + (off & mask_b);
        const Box ba = load_box(q.A.box, na), bb = load_box(q.B.box, nb);
        const float key = kMax ? box_max_upper(ba, bb) : box_min_lower(ba, bb);
        const bool keep = !culling || (kMax ? key >= ub : key <= ub);
        if (!keep) {
          ++my_culled;
          continue;
        }
        keep_mask |= 1u << it;
        on[it] = to_leaves ? make_uint2((unsigned)(na - leaf_a0), (unsigned)(nb - leaf_b0))
                           : make_uint2((unsigned)na, (unsigned)nb);
        ok[it] = key;
        // kept pairs tighten the bound (query.py:416-423); at leaf level the
        // leaf boxes are tight, so the enhanced bound is valid there too.
        if (kMax) {
          const float u = enh ? box_enhanced_max_lower(ba, bb) : box_min_lower(ba, bb);
          upd = fmaxf(upd, u);
        } else {
          const float u = enh ? box_enhanced_min_upper(ba, bb) : box_max_upper(ba, bb);
          upd = fminf(upd, u);
        }
      }
      unsigned total;
      const unsigned my_off = block_exclusive_scan(__popc(keep_mask), warp_tot, total);
      upd = kMax ? warp_max(upd) : warp_min(upd);
      if ((threadIdx.x & 31) == 0) warp_upd[threadIdx.x >> 5] = upd;
      __syncthreads();
      if (threadIdx.x == 0) {
        out_base = total ? atomicAdd(&S->n_out, (unsigned long long)total) : 0ull;
        float u = warp_upd[0];
        for (int w = 1; w < kExpandThreads / 32; ++w) u = kMax ? fmaxf(u, warp_upd[w]) : fminf(u, warp_upd[w]);
        if (kMax ? u > 0.f : u < INFINITY) commit_bound<kMax>(S, u);
      }
      __syncthreads();
      unsigned long long slot = out_base + my_off;
#pragma unroll
      for (int it = 0; it < kExpandItems; ++it) {
        if (keep_mask & (1u << it)) {
          if (slot < q.cap) {
            out_node[slot] = on[it];
            out_key[slot] = ok[it];
          }
          ++slot;
        }
      }
      __syncthreads();  // warp_tot / out_base reuse
    }
  }

  // --- per-block counters, then the last block advances the front ---------
  unsigned long long c = warp_sum_u64(my_culled);
  if ((threadIdx.x & 31) == 0) red_culled[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long bc = 0;
    for (int w = 0; w < kExpandThreads / 32; ++w) bc += red_culled[w];
    if (bc) atomicAdd(&S->culled, bc);
    __threadfence();
    const unsigned prev = atomicAdd(&S->done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      volatile QState* V = S;
      const unsigned long long n_out = V->n_out;
      const int it = V->iter;
      if (overflow || n_out > (unsigned long long)q.cfg.front_hard_cap) {
        S->err = GD_ERR_FRONT_OVERFLOW;
        S->ov_cand = overflow ? (long long)ncand : (long long)n_out;
        S->ov_in = (long long)n_in;
        S->ov_cap = q.cfg.front_hard_cap;
        S->n_in = 0;
        S->n_leaf = 0;
      } else {
        S->expanded += ncand;
        if (it < kMaxIters) {
          GdIterStat st;
          st.k = k;
          st.front_in = (long long)n_in;
          st.front_out = to_leaves ? 0 : (long long)n_out;
          st.culled = (long long)V->culled;
          const float b = __uint_as_float(V->bound_bits);
          st.bound_after = kMax ? (double)b + (double)S->slack : (double)b - (double)S->slack;
          st._pad = 0;
          S->stats[it] = st;
        }
        if (to_leaves) {
          S->n_leaf = n_out;
          S->leaf_buf = cur ^ 1;
          S->n_in = 0;
        } else {
          S->n_in = n_out;
          S->cur = cur ^ 1;
        }
        S->depth_a += ka;
        S->depth_b += kb;
      }
      S->iter = it + 1;
      S->n_out = 0;
      S->culled = 0;
      S->done = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// fast float32 narrow phase over the leaf-pair list (query.py:287-346):
// every leaf pair expands to its 1..4 triangle pairs inside the block
// (block scan), so lanes stay busy whatever the 1/2-triangle leaf mix.
template <bool kMax, bool kRescan>
__global__ __launch_bounds__(kNarrowThreads) void k_narrow(QArgs q) {
  QState* S = q.S;
  const unsigned long long n = S->n_leaf;
  if (n == 0) return;
  // rescan pass: only when the band overflowed; re-filters every pair with
  // the final bound and evaluates the survivors exactly
  if (kRescan && *reinterpret_cast<volatile int*>(&S->band_overflow) == 0) return;
  __shared__ unsigned warp_tot[kNarrowThreads / 32];
  __shared__ unsigned char owner[kNarrowThreads * 4];
  __shared__ unsigned s_off[kNarrowThreads];
  __shared__ uint2 s_first[kNarrowThreads];
  __shared__ unsigned char s_cb[kNarrowThreads];
  __shared__ float warp_upd[kNarrowThreads / 32];
  const int buf = S->leaf_buf;
  const uint2* __restrict__ leaves = q.node[buf];
  const float* __restrict__ keys = q.key[buf];
  const float E = S->slack;
  const bool culling = q.cfg.culling != 0;
  unsigned long long my_pairs = 0;
  const int4* __restrict__ lta = reinterpret_cast<const int4*>(q.A.leaf_tri);
  const int4* __restrict__ ltb = reinterpret_cast<const int4*>(q.B.leaf_tri);

  for (unsigned long long tile = blockIdx.x; tile * kNarrowThreads < n; tile += gridDim.x) {
    const unsigned long long i = tile * kNarrowThreads + threadIdx.x;
    const float ub = load_bound(S);
    unsigned cnt = 0;
    uint2 first = make_uint2(0, 0);
    unsigned cb = 1;
    if (i < n) {
      const float pk = keys[i];
      if (!culling || (kMax ? pk >= ub : pk <= ub)) {
        const uint2 lp = leaves[i];
        const unsigned fa = __ldg(q.A.leaf_first + lp.x), ca = __ldg(q.A.leaf_first + lp.x + 1) - fa;
        const unsigned fb = __ldg(q.B.leaf_first + lp.y);
        cb = __ldg(q.B.leaf_first + lp.y + 1) - fb;
        first = make_uint2(fa, fb);
        cnt = ca * cb;
      }
    }
    unsigned total;
    const unsigned off = block_exclusive_scan(cnt, warp_tot, total);
    s_off[threadIdx.x] = off;
    s_first[threadIdx.x] = first;
    s_cb[threadIdx.x] = (unsigned char)cb;
    for (unsigned j = 0; j < cnt; ++j) owner[off + j] = (unsigned char)threadIdx.x;
    __syncthreads();
    float upd = kMax ? 0.f : INFINITY;
    for (unsigned s = threadIdx.x; s < total; s += kNarrowThreads) {
      const int o = owner[s];
      const unsigned j = s - s_off[o];
      const unsigned cbo = s_cb[o];
      const uint2 f = s_first[o];
      const int4 sa = __ldg(lta + f.x + j / cbo);
      const int4 sb = __ldg(ltb + f.y + j % cbo);
      const Tri<float> A = load_tri32(q.A, sa), B = load_tri32(q.B, sb);
      const float d = kMax ? sqrtf(tri_tri_max_d2<Fast<float>, float, false>(A, B, nullptr, nullptr))
                           : sqrtf(tri_tri_min_d2<Fast<float>, float, false>(A, B, nullptr, nullptr));
      upd = kMax ? fmaxf(upd, d) : fminf(upd, d);
      const bool cand = kMax ? (d + E >= ub) : (d - E <= ub);
      if (cand) {
        if (kRescan) {
          atomic_min_key(&S->best, exact_key<kMax>(q, (unsigned)sa.w, (unsigned)sb.w));
          atomicAdd(&S->band_eval, 1ull);
        } else {
          const unsigned long long slot = atomicAdd(&S->n_band, 1ull);
          if (slot < q.band_cap) {
            q.band_ids[slot] = make_uint2((unsigned)sa.w, (unsigned)sb.w);
            q.band_d[slot] = d;
          } else {
            S->band_overflow = 1;  // k_narrow<kMax, true> re-scans the leaf list
          }
        }
      }
    }
    if (kRescan) {
      __syncthreads();
      continue;
    }
    my_pairs += total;
    upd = kMax ? warp_max(upd) : warp_min(upd);
    if ((threadIdx.x & 31) == 0) warp_upd[threadIdx.x >> 5] = upd;
    __syncthreads();
    if (threadIdx.x == 0) {
      float u = warp_upd[0];
      for (int w = 1; w < kNarrowThreads / 32; ++w) u = kMax ? fmaxf(u, warp_upd[w]) : fminf(u, warp_upd[w]);
      if (kMax ? u > 0.f : u < INFINITY) commit_bound<kMax>(S, u);
    }
    __syncthreads();
  }
  if (!kRescan && threadIdx.x == 0 && my_pairs) atomicAdd(&S->narrow, my_pairs);
}

// ---------------------------------------------------------------------------
// exact pass over the band: only pairs whose float32 distance can still be
// the answer (|d_fast - d_exact| <= E/2) are re-evaluated in the reference's
// arithmetic; the 128-bit (distance, tri_a, tri_b) minimum is the witness
// with the reference's lexicographic tie rule (query.py:205-220, 299).
template <bool kMax>
__global__ __launch_bounds__(256) void k_refine(QArgs q) {
  QState* S = q.S;
  const unsigned long long n = min(S->n_band, q.band_cap);
  const float E = S->slack;
  const float ub = load_bound(S);
  __shared__ Key128 wk[8];
  Key128 best;
  best.hi = ~0ull;
  best.lo = ~0ull;
  unsigned long long evals = 0;
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
    const float d = q.band_d[i];
    if (kMax ? (d + E >= ub) : (d - E <= ub)) {
      const uint2 ids = q.band_ids[i];
      Key128 k = exact_key<kMax>(q, ids.x, ids.y);
      if (key_less(k, best)) best = k;
      ++evals;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key128 other = shfl_key(best, o);
    if (key_less(other, best)) best = other;
  }
  evals = warp_sum_u64(evals);
  if ((threadIdx.x & 31) == 0) {
    wk[threadIdx.x >> 5] = best;
    if (evals) atomicAdd(&S->band_eval, evals);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w)
      if (key_less(wk[w], best)) best = wk[w];
    if (best.hi != ~0ull) atomic_min_key(&S->best, best);
  }
}

template <bool kMax>
__global__ void k_final(QArgs q) {
  if (threadIdx.x != 0) return;
  QState* S = q.S;
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
  const Key128 best = S->best;
  if (best.hi == ~0ull && best.lo == ~0ull) {
    r.tri_a = r.tri_b = -1;
    const float b = load_bound(S);
    r.distance = kMax ? (double)b + (double)S->slack : (double)b - (double)S->slack;
    r.witness_distance = r.distance;
  } else {
    const unsigned long long bits = kMax ? ~best.hi : best.hi;
    const double d = __longlong_as_double((long long)bits);
    const unsigned ta = (unsigned)(best.lo >> 32), tb = (unsigned)(best.lo & 0xffffffffu);
    r.distance = d;
    r.witness_distance = d;
    r.tri_a = ta;
    r.tri_b = tb;
    if (q.cfg.precision == 32) {
      Tri<float> a = mesh_tri<float>(q.ma, ta), b = mesh_tri<float>(q.mb, tb);
      V3<float> p, qq;
      if (kMax)
        tri_tri_max_d2<Exact<float>, float, true>(a, b, &p, &qq);
      else
        tri_tri_min_d2<Exact<float>, float, true>(a, b, &p, &qq);
      r.point_a[0] = p.x; r.point_a[1] = p.y; r.point_a[2] = p.z;
      r.point_b[0] = qq.x; r.point_b[1] = qq.y; r.point_b[2] = qq.z;
    } else {
      Tri<double> a = mesh_tri<double>(q.ma, ta), b = mesh_tri<double>(q.mb, tb);
      V3<double> p, qq;
      if (kMax)
        tri_tri_max_d2<Exact<double>, double, true>(a, b, &p, &qq);
      else
        tri_tri_min_d2<Exact<double>, double, true>(a, b, &p, &qq);
      r.point_a[0] = p.x; r.point_a[1] = p.y; r.point_a[2] = p.z;
      r.point_b[0] = qq.x; r.point_b[1] = qq.y; r.point_b[2] = qq.z;
    }
  }
  *q.result = r;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct WsLayout {
  size_t state, node0, key0, node1, key1, band_ids, band_d, result, total;
  unsigned long long cap, band_cap;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static WsLayout ws_layout(const GdConfig& cfg) {
  WsLayout L;
  L.cap = (unsigned long long)std::max<int64_t>(cfg.front_hard_cap, 4);
  L.band_cap = cfg.band_cap > 0 ? (unsigned long long)cfg.band_cap : (1ull << 20);
  size_t o = 0;
  L.state = o;
  o = align_up(o + sizeof(QState), 256);
  L.result = o;
  o = align_up(o + sizeof(GdResult), 256);
  L.node0 = o;
  o = align_up(o + L.cap * sizeof(uint2), 256);
  L.key0 = o;
  o = align_up(o + L.cap * sizeof(float), 256);
  L.node1 = o;
  o = align_up(o + L.cap * sizeof(uint2), 256);
  L.key1 = o;
  o = align_up(o + L.cap * sizeof(float), 256);
  L.band_ids = o;
  o = align_up(o + L.band_cap * sizeof(uint2), 256);
  L.band_d = o;
  o = align_up(o + L.band_cap * sizeof(float), 256);
  L.total = o;
  return L;
}

size_t query_workspace_size(const GdConfig& cfg) { return ws_layout(cfg).total; }

static void validate(const GdBvh& a, const GdBvh& b, const GdConfig& cfg) {
  GD_CHECK(cfg.kind == 0 || cfg.kind == 1, GD_ERR_INVALID, "kind must be 0 (min) or 1 (max)");
  GD_CHECK(cfg.precision == 32 || cfg.precision == 64, GD_ERR_CONFIG, "precision must be 32 or 64");
  GD_CHECK(cfg.front_cap >= 4, GD_ERR_CONFIG, "front_cap must be >= 4");
  GD_CHECK(cfg.depth_cap >= 1 && cfg.depth_cap <= 16, GD_ERR_CONFIG, "depth_cap must be in [1, 16]");
  GD_CHECK(cfg.front_hard_cap >= 4, GD_ERR_CONFIG, "front_hard_cap must be >= 4");
  GD_CHECK(a.depth >= 0 && a.depth <= 31 && b.depth >= 0 && b.depth <= 31, GD_ERR_INVALID,
           "tree depth out of range");
  GD_CHECK(a.box && b.box && a.leaf_tri && b.leaf_tri && a.leaf_first && b.leaf_first && a.vtx32 && b.vtx32,
           GD_ERR_INVALID, "BVH arrays must be allocated");
}

// optional phase timing for the bench: events between the query phases
static bool g_profile = false;
static cudaEvent_t g_ev[6];
static int g_ev_dev = -1;
void set_profiling(int on) {
  g_profile = on != 0;
  if (g_profile) {
    int dev = 0;
    GD_CUDA(cudaGetDevice(&dev));
    if (g_ev_dev != dev) {
      for (auto& e : g_ev) GD_CUDA(cudaEventCreate(&e));
      g_ev_dev = dev;
    }
  }
}
// [init, expand (all iterations), narrow, refine, rescan + final] in ms
int phase_ms(float* out, int n) {
  if (g_ev_dev < 0) return 0;
  GD_CUDA(cudaEventSynchronize(g_ev[5]));
  int k = 0;
  for (; k < 5 && k < n; ++k) GD_CUDA(cudaEventElapsedTime(out + k, g_ev[k], g_ev[k + 1]));
  return k;
}

template <bool kMax>
static void launch_query(const QArgs& q, int max_iters, cudaStream_t s) {
  const int sms = num_sms();
  auto mark = [&](int i) {
    if (g_profile) GD_CUDA(cudaEventRecord(g_ev[i], s));
  };
  mark(0);
  k_init<kMax><<<1, 32, 0, s>>>(q);
  mark(1);
  for (int i = 0; i < max_iters; ++i) k_expand<kMax><<<sms * 8, kExpandThreads, 0, s>>>(q);
  mark(2);
  k_narrow<kMax, false><<<sms * 4, kNarrowThreads, 0, s>>>(q);
  mark(3);
  k_refine<kMax><<<sms * 2, 256, 0, s>>>(q);
  mark(4);
  k_narrow<kMax, true><<<sms * 4, kNarrowThreads, 0, s>>>(q);
  k_final<kMax><<<1, 32, 0, s>>>(q);
  mark(5);
  GD_CUDA(cudaGetLastError());
  count_launches(5 + max_iters);
}

void query_async(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                 void* ws, size_t ws_bytes, GdResult* result_dev, cudaStream_t s) {
  validate(a, b, cfg);
  WsLayout L = ws_layout(cfg);
  GD_CHECK(ws != nullptr && ws_bytes >= L.total, GD_ERR_WORKSPACE,
           "query workspace too small: need " + std::to_string(L.total) + " bytes");
  char* base = static_cast<char*>(ws);
  QArgs q;
  q.ma = ma;
  q.mb = mb;
  q.A = a;
  q.B = b;
  q.cfg = cfg;
  q.S = reinterpret_cast<QState*>(base + L.state);
  q.node[0] = reinterpret_cast<uint2*>(base + L.node0);
  q.node[1] = reinterpret_cast<uint2*>(base + L.node1);
  q.key[0] = reinterpret_cast<float*>(base + L.key0);
  q.key[1] = reinterpret_cast<float*>(base + L.key1);
  q.band_ids = reinterpret_cast<uint2*>(base + L.band_ids);
  q.band_d = reinterpret_cast<float*>(base + L.band_d);
  q.cap = L.cap;
  q.band_cap = L.band_cap;
  q.result = result_dev ? result_dev : reinterpret_cast<GdResult*>(base + L.result);
  const int max_iters = std::max(a.depth, b.depth);
  if (cfg.kind == 1)
    launch_query<true>(q, max_iters, s);
  else
    launch_query<false>(q, max_iters, s);
}

void query_collect(const GdConfig& cfg, void* ws, const GdResult* result_dev, GdResult* out, GdIterStat* stats,
                   int max_stats, cudaStream_t s) {
  WsLayout L = ws_layout(cfg);
  char* base = static_cast<char*>(ws);
  const GdResult* src = result_dev ? result_dev : reinterpret_cast<const GdResult*>(base + L.result);
  GD_CUDA(cudaMemcpyAsync(out, src, sizeof(GdResult), cudaMemcpyDeviceToHost, s));
  if (stats && max_stats > 0) {
    const QState* S = reinterpret_cast<const QState*>(base + L.state);
    GD_CUDA(cudaMemcpyAsync(stats, S->stats, sizeof(GdIterStat) * std::min(max_stats, kMaxIters),
                            cudaMemcpyDeviceToHost, s));
  }
  GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gd
