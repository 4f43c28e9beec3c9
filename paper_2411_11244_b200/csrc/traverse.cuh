// traverse.cuh -- root setup and BVTT front expansion (query.py:266-509).
#pragma once

#include "engine.cuh"

namespace gd {

// 2 blocks / SM of 512 threads: one block's tile flush overlaps the other's
// sweep, and the grid barrier has 296 arrivals instead of 592 (measured: 256
// x 4 -> 512 x 2 cut the traversal 0.251 -> 0.240 ms; 1024 x 1: 0.256 ms)
#ifndef GD_EXPAND_THREADS
#define GD_EXPAND_THREADS 512
#endif
constexpr int kExpandThreads = GD_EXPAND_THREADS;
constexpr int kGenericItems = 1;                                   // candidates / thread / tile (k >= 2)
constexpr int kGenericTile = kExpandThreads * kGenericItems;
constexpr int kK1Rounds = 4;                                       // entries / thread / tile (k == 1)
constexpr int kK1Tile = kExpandThreads * kK1Rounds;
constexpr int kK1Stage = kK1Tile * 4;                              // staged survivors (<= 4 / entry)
constexpr size_t kExpandDynSmem = kK1Stage * (sizeof(uint2) + sizeof(float));

__device__ __forceinline__ float load_bound(const QState* S) {
  return __uint_as_float(*reinterpret_cast<const volatile unsigned int*>(&S->bound_bits));
}

template <bool kMax>
__device__ __forceinline__ bool improves(float a, float b) {
  return kMax ? a > b : a < b;
}

// a candidate survives while its key can still beat the (slack-carrying) bound
template <bool kMax>
__device__ __forceinline__ bool survives(float key, float bound) {
  return kMax ? key >= bound : key <= bound;
}

template <bool kMax>
__device__ __forceinline__ void commit_bound(QState* S, float v) {
  if (kMax)
    atomic_max_pos(&S->bound_bits, v - S->slack);
  else
    atomic_min_pos(&S->bound_bits, v + S->slack);
}
// the same, also applied to the other ranks' bound cells of a split query
// (GdConfig.peer_bounds: their workspaces mapped over NVLink).  A bound is an
// achieved distance +- the common slack, valid for every rank's sub-query.
template <bool kMax>
__device__ __forceinline__ void commit_bound(const QArgs& q, float v) {
  QState* S = q.S;
  commit_bound<kMax>(S, v);
  if (q.cfg.n_peers > 0) {
    const unsigned bits = __float_as_uint(fmaxf(kMax ? v - S->slack : v + S->slack, 0.f));
    unsigned* const* peers = static_cast<unsigned* const*>(q.cfg.peer_bounds);
    for (int i = 0; i < q.cfg.n_peers; ++i) {
      if (kMax)
        atomicMax_system(peers[i], bits);
      else
        atomicMin_system(peers[i], bits);
    }
  }
}

// Keys and bound updates are kept SQUARED inside the traversal (no sqrt per
// candidate); the bound cell itself is a distance, squared once per tile.
// key of a node pair: box min distance^2 (min query) / box max distance^2 (max)
template <bool kMax>
__device__ __forceinline__ float pair_key(const Box& a, const Box& b) {
  return kMax ? box_max_upper_sq(a, b) : box_min_lower_sq(a, b);
}

// bound contribution^2 of a kept pair (query.py:416-423): the enhanced bound
// of tight boxes, or the conventional one when enhanced bounds are off
template <bool kMax>
__device__ __forceinline__ float pair_update(const Box& a, const Box& b, bool enh) {
  if (kMax) return enh ? box_enhanced_max_lower_sq(a, b) : box_min_lower_sq(a, b);
  return enh ? box_enhanced_min_upper_sq(a, b) : box_max_upper_sq(a, b);
}

__device__ __forceinline__ float load_bound_sq(const QState* S) {
  const float b = load_bound(S);
  return b * b;
}

// block-wide exclusive scan of small counts (blockDim.x == kExpandThreads)
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

// closest (min) / farthest (max) vertex pair of two triangles
template <bool kMax>
__device__ __forceinline__ float vertex_pair_bound(const Tri<float>& a, const Tri<float>& b) {
  float best = kMax ? 0.f : INFINITY;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const float dx = a.v[i].x - b.v[j].x, dy = a.v[i].y - b.v[j].y, dz = a.v[i].z - b.v[j].z;
      const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      best = kMax ? fmaxf(best, d2) : fminf(best, d2);
    }
  return sqrtf(best);
}

// ---------------------------------------------------------------------------
// split query: owner rank of a node pair at depths (da, db) -- the hash of
// its ancestor pair at (la, lb) (gdist.h GdConfig.split_*); every descendant
// of an owned pair is owned, so the test is idempotent once da >= la, db >= lb
__device__ __forceinline__ bool owned(const GdConfig& c, unsigned na, unsigned nb, int da, int db, int la, int lb) {
  if (c.split_world <= 1 || da < la || db < lb) return true;
  const unsigned aa = ((na + 1) >> (da - la)) - 1, ab = ((nb + 1) >> (db - lb)) - 1;
  unsigned h = aa * 0x9E3779B1u ^ (ab + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 13;
  return (int)(h % (unsigned)c.split_world) == c.split_rank;
}

// query prologue (one thread; k_traverse block 0 before its first barrier):
// root key and bound, slack, root front, counters, warm_pair
template <bool kMax>
__device__ void init_query(const QArgs& q) {
  QState* S = q.S;
  Box ra = load_box(q.A.box, 0), rb = load_box(q.B.box, 0);
  float M = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    M = fmaxf(M, fmaxf(fmaxf(fabsf(ra.lo[k]), fabsf(ra.hi[k])), fmaxf(fabsf(rb.lo[k]), fabsf(rb.hi[k]))));
  // slack: 256 float32 ulps of the largest coordinate
  const float E = M * 0x1p-15f;
  S->slack = E;
  const float key0 = pair_key<kMax>(ra, rb);  // squared
  bool nan_root = false;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    nan_root = nan_root || ra.lo[k] != ra.lo[k] || ra.hi[k] != ra.hi[k] || rb.lo[k] != rb.lo[k] || rb.hi[k] != rb.hi[k];
  const float b0 = nan_root ? __int_as_float(0x7fc00000) : sqrtf(pair_update<kMax>(ra, rb, q.cfg.enhanced_bounds != 0));
  // a NaN root box (a NaN vertex, propagated by the refit) leaves a NaN
  // bound: every candidate is culled and the distance is NaN, as in the
  // reference (its np.minimum boxes and `key < bound` tests)
  S->bound_bits = __float_as_uint(kMax ? (b0 != b0 ? b0 : fmaxf(b0 - E, 0.f)) : b0 + E);
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
  S->n_cand = 0;
  S->fbest = kMax ? 0u : __float_as_uint(INFINITY);
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
  long long wa = q.cfg.warm_a, wb = q.cfg.warm_b;
  if (q.cfg.warm_from) {  // the previous frame's witness (GdConfig.warm_from)
    const GdResult* w = static_cast<const GdResult*>(q.cfg.warm_from);
    if (w->status == 0 && w->tri_a >= 0 && w->tri_a < q.ma.m && w->tri_b >= 0 && w->tri_b < q.mb.m) {
      wa = w->tri_a;
      wb = w->tri_b;
    }
  }
  if (wa >= 0) {
    // warm_pair seeds the bound with one exact pair (query.py:494-502)
    unsigned ta = (unsigned)wa, tb = (unsigned)wb;
    const int32_t* ia = q.ma.tri + 3 * (long long)ta;
    const int32_t* ib = q.mb.tri + 3 * (long long)tb;
    // the pair always reaches the exact pass (band distance -inf / +inf);
    // its vertex-pair distance is an achieved distance, hence a valid bound
    Tri<float> a = tri32(q.A, q.xa, q.A.vmap[ia[0]], q.A.vmap[ia[1]], q.A.vmap[ia[2]]);
    Tri<float> b = tri32(q.B, q.xb, q.B.vmap[ib[0]], q.B.vmap[ib[1]], q.B.vmap[ib[2]]);
    commit_bound<kMax>(S, vertex_pair_bound<kMax>(a, b));
    q.band_ids[0] = make_uint2(ta, tb);
    q.band_d[0] = kMax ? INFINITY : -INFINITY;
    S->n_band = 1;
  }
}

// ---------------------------------------------------------------------------
// Shared per-block plumbing of an expansion sweep: survivors are compacted
// with one block scan + one global atomic per tile, bound updates reduced to
// one atomic per tile (the paper's block-wise reduction).
struct ExpandShared {
  unsigned warp_tot[kExpandThreads / 32];
  unsigned long long out_base;
  float warp_upd[kExpandThreads / 32];
  unsigned long long red_culled[kExpandThreads / 32];
  unsigned stage_count;
};

// Grid-wide barrier of the persistent traversal (all blocks co-resident:
// cooperative launch).  `bar` only grows; phase p completes when it reaches
// p * gridDim.x, so no reset is needed inside a query.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// release-arrive / acquire-spin: every block's writes before the barrier are
// visible to every block after it.  Data written in the same launch (fronts,
// counters) is read with plain coherent loads, never through __ldg.
// Iteration barrier fused with the survivor count: cnt[it] holds the
// survivors (low 40 bits, reserved by the tiles with plain atomicAdd) and the
// block arrivals (high 24 bits).  Returns the final survivor count -- no
// separate load after the barrier.
constexpr int kArriveShift = 40;
__device__ __forceinline__ unsigned long long count_barrier(unsigned long long* cnt) {
  __shared__ unsigned long long total;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long target = (unsigned long long)gridDim.x << kArriveShift;
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(cnt), "l"(1ull << kArriveShift) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
    } while ((v & ~((1ull << kArriveShift) - 1)) < target);
    total = v & ((1ull << kArriveShift) - 1);
  }
  __syncthreads();
  return total;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned phase) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = phase * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// One expansion sweep (query.py:349-451, Alg. 2) over front `cur`.  Two
// mappings, chosen uniformly per iteration from the adaptive depth k:
//  k == 1 (the wide late iterations): one thread per front entry; it loads the
//          (1 or 2) child boxes of each side once (contiguous siblings) and
//          tests the <= 4 child pairs -- 14 loads per entry instead of 32.
//  k >= 2 (narrow early fronts, ncand < front_cap): one thread per candidate,
//          t -> entry t >> (ka+kb), descendants ((node+1) << k) - 1 + offset.
// Survivors are counted into S->cnt[it]; the caller synchronises the grid.
template <bool kMax>
__device__ __forceinline__ void expand_sweep(const QArgs& q, ExpandShared& sh, unsigned char* k1_stage, int it,
                                             int cur, unsigned long long n_in, int k, int ka, int kb,
                                             bool to_leaves, unsigned long long ncand, int da, int db, int la,
                                             int lb) {
  QState* S = q.S;
  const int shift = ka + kb;
  const bool k1 = (k == 1);
  const unsigned long long tiles = k1 ? (n_in + kK1Tile - 1) / kK1Tile : (ncand + kGenericTile - 1) / kGenericTile;
  const uint2* __restrict__ in_node = q.node[cur];
  const float* __restrict__ in_key = q.key[cur];
  uint2* out_node = q.node[cur ^ 1];
  float* out_key = q.key[cur ^ 1];
  unsigned long long* n_out = &S->cnt[it];
  const unsigned leaf_a0 = (unsigned)((1ull << q.A.depth) - 1), leaf_b0 = (unsigned)((1ull << q.B.depth) - 1);
  const unsigned ra0 = to_leaves ? leaf_a0 : 0u, rb0 = to_leaves ? leaf_b0 : 0u;  // output index base
  const bool culling = q.cfg.culling != 0, enh = q.cfg.enhanced_bounds != 0;
  unsigned long long my_culled = 0, my_skipped = 0;  // skipped: not owned (split query)

  if (k1) {
    // survivors are staged in shared memory (warp-aggregated appends), then
    // one global reservation per tile and a coalesced copy-out.  A tile is
    // R rounds of one entry per thread; R shrinks with the front so a small
    // front spreads over all blocks (latency, not throughput, bounds it).
    uint2* s_node = reinterpret_cast<uint2*>(k1_stage);
    float* s_key = reinterpret_cast<float*>(k1_stage + kK1Stage * sizeof(uint2));
    const int ca = 1 << ka, cb = 1 << kb;
    const int lane = threadIdx.x & 31;
    // even contiguous split of the front over the blocks (no tail
    // imbalance at the grid barrier), processed in tiles of <= kK1Rounds
    // rounds of one entry per thread
    unsigned long long per_blk = (n_in + gridDim.x - 1) / gridDim.x;
    per_blk = (per_blk + 63) & ~63ull;
    const unsigned long long blk_lo = min(n_in, blockIdx.x * per_blk);
    const unsigned long long blk_hi = min(n_in, blk_lo + per_blk);
    for (unsigned long long t0 = blk_lo; t0 < blk_hi; t0 += kK1Tile) {
      const unsigned long long t1 = min(blk_hi, t0 + kK1Tile);
      const int R = (int)((t1 - t0 + kExpandThreads - 1) / kExpandThreads);
      if (threadIdx.x == 0) sh.stage_count = 0;
      // entry loads are software-pipelined one round ahead
      const unsigned long long e0 = t0 + threadIdx.x;
      float pk_next = e0 < t1 ? in_key[e0] : 0.f;
      uint2 nd_next = e0 < t1 ? in_node[e0] : make_uint2(0, 0);
      const float ub = load_bound_sq(S);  // one bound snapshot per tile (query.py:396)
      __syncthreads();
      float upd = kMax ? 0.f : INFINITY;
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        const unsigned long long e = t0 + (unsigned long long)r * kExpandThreads + threadIdx.x;
        const float pk = pk_next;
        uint2 nd = nd_next;
        if (r + 1 < R && e + kExpandThreads < t1) {
          pk_next = in_key[e + kExpandThreads];
          nd_next = in_node[e + kExpandThreads];
        }
        unsigned keep = 0;
        float keys[4];
        const bool mine = e < t1 && owned(q.cfg, nd.x, nd.y, da, db, la, lb);
        if (e < t1 && !mine) my_skipped += (unsigned)(ca * cb);
        if (mine) {
          // stale-entry re-cull: descendants' keys are monotone in the parent's
          if (culling && !survives<kMax>(pk, ub)) {
            my_culled += (unsigned)(ca * cb);
          } else {
            const unsigned a0 = ka ? 2 * nd.x + 1 : nd.x, b0 = kb ? 2 * nd.y + 1 : nd.y;
            Box A[2], B[2];
            if (ka)
              load_children(q.A.box, nd.x, A[0], A[1]);
            else
              A[0] = load_box(q.A.box, a0);
            if (kb)
              load_children(q.B.box, nd.y, B[0], B[1]);
            else
              B[0] = load_box(q.B.box, b0);
            float best = kMax ? -INFINITY : INFINITY;
            int bc = 0;
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                if (i >= ca || j >= cb) continue;
                const int c = 2 * i + j;
                const float key = pair_key<kMax>(A[i], B[j]);
                keys[c] = key;
                if (culling && !survives<kMax>(key, ub)) {
                  ++my_culled;
                  continue;
                }
                keep |= 1u << c;
                if (improves<kMax>(key, best)) {
                  best = key;
                  bc = c;
                }
              }
            // leaf pairs go to the narrow phase and emit no bound
            // (query.py:411-415); otherwise the bound is updated from the
            // most promising kept child pair: any kept pair's enhanced bound
            // is a valid bound (query.py:416-423 takes the minimum over all
            // kept pairs -- same fixed point, a quarter of the arithmetic)
            if (keep && !to_leaves) {
              const Box ba = select_box((bc >> 1) != 0, A[1], A[0]);
              const Box bb = select_box((bc & 1) != 0, B[1], B[0]);
              const float u = pair_update<kMax>(ba, bb, enh);
              upd = kMax ? fmaxf(upd, u) : fminf(upd, u);
            }
            nd = make_uint2(a0, b0);
          }
        }
        // warp-aggregated append into the shared staging area
        const unsigned cnt = __popc(keep);
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        unsigned wbase = 0;
        if (lane == 31 && incl) wbase = atomicAdd(&sh.stage_count, incl);
        wbase = __shfl_sync(0xffffffffu, wbase, 31);
        unsigned pos = wbase + incl - cnt;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (keep & (1u << c)) {
            s_node[pos] = make_uint2(nd.x + (c >> 1) - ra0, nd.y + (c & 1) - rb0);
            s_key[pos] = keys[c];
            ++pos;
          }
        }
      }  // rounds
      upd = kMax ? warp_max(upd) : warp_min(upd);
      if (lane == 0) sh.warp_upd[threadIdx.x >> 5] = upd;
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned total = sh.stage_count;
        // low 40 bits: survivors so far (blocks that finished have added their
        // arrival in the high bits, count_barrier)
        sh.out_base = total ? (atomicAdd(n_out, (unsigned long long)total) & ((1ull << kArriveShift) - 1)) : 0ull;
        float u = sh.warp_upd[0];
        for (int w = 1; w < kExpandThreads / 32; ++w) u = kMax ? fmaxf(u, sh.warp_upd[w]) : fminf(u, sh.warp_upd[w]);
        if (kMax ? u > 0.f : u < INFINITY) commit_bound<kMax>(q, sqrtf(u));
      }
      __syncthreads();
      const unsigned total = sh.stage_count;
      const unsigned long long base = sh.out_base;
      for (unsigned i = threadIdx.x; i < total; i += kExpandThreads) {
        if (base + i < q.cap) {
          out_node[base + i] = s_node[i];
          out_key[base + i] = s_key[i];
        }
      }
      __syncthreads();  // staging reuse by the next tile
    }
  } else {
    const unsigned long long off_mask = (1ull << shift) - 1, mask_b = (1ull << kb) - 1;
    for (unsigned long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const unsigned long long base = tile * kGenericTile;
      const float ub = load_bound_sq(S);
      float upd = kMax ? 0.f : INFINITY;
      uint2 on[kGenericItems];
      float ok[kGenericItems];
      unsigned keep = 0;
#pragma unroll
      for (int itm = 0; itm < kGenericItems; ++itm) {
        const unsigned long long t = base + (unsigned long long)itm * kExpandThreads + threadIdx.x;
        if (t >= ncand) continue;
        const unsigned long long e = t >> shift, off = t & off_mask;
        const float pk = in_key[e];
        const uint2 nd = in_node[e];
        if (!owned(q.cfg, nd.x, nd.y, da, db, la, lb)) {
          ++my_skipped;
          continue;
        }
        if (culling && !survives<kMax>(pk, ub)) {
          ++my_culled;
          continue;
        }
        const unsigned na = (unsigned)(((((unsigned long long)nd.x + 1) << ka) - 1) + (off >> kb));
        const unsigned nb = (unsigned)(((((unsigned long long)nd.y + 1) << kb) - 1) + (off & mask_b));
        const Box ba = load_box(q.A.box, na), bb = load_box(q.B.box, nb);
        const float key = pair_key<kMax>(ba, bb);
        if (culling && !survives<kMax>(key, ub)) {
          ++my_culled;
          continue;
        }
        keep |= 1u << itm;
        on[itm] = make_uint2(na - ra0, nb - rb0);
        ok[itm] = key;
        if (!to_leaves) {
          const float u = pair_update<kMax>(ba, bb, enh);
          upd = kMax ? fmaxf(upd, u) : fminf(upd, u);
        }
      }
      unsigned my_off;
      unsigned total;
      my_off = block_exclusive_scan(__popc(keep), sh.warp_tot, total);
      upd = kMax ? warp_max(upd) : warp_min(upd);
      if ((threadIdx.x & 31) == 0) sh.warp_upd[threadIdx.x >> 5] = upd;
      __syncthreads();
      if (threadIdx.x == 0) {
        // low 40 bits: survivors so far (blocks that finished have added their
        // arrival in the high bits, count_barrier)
        sh.out_base = total ? (atomicAdd(n_out, (unsigned long long)total) & ((1ull << kArriveShift) - 1)) : 0ull;
        float u = sh.warp_upd[0];
        for (int w = 1; w < kExpandThreads / 32; ++w) u = kMax ? fmaxf(u, sh.warp_upd[w]) : fminf(u, sh.warp_upd[w]);
        if (kMax ? u > 0.f : u < INFINITY) commit_bound<kMax>(q, sqrtf(u));
      }
      __syncthreads();
      unsigned long long slot = sh.out_base + my_off;
#pragma unroll
      for (int itm = 0; itm < kGenericItems; ++itm) {
        if (keep & (1u << itm)) {
          if (slot < q.cap) {
            out_node[slot] = on[itm];
            out_key[slot] = ok[itm];
          }
          ++slot;
        }
      }
      __syncthreads();
    }
  }

  // --- per-block counters -----------------------------------------------------
  unsigned long long c = warp_sum_u64(my_culled);
  const unsigned long long sk = q.cfg.split_world > 1 ? warp_sum_u64(my_skipped) : 0ull;
  if ((threadIdx.x & 31) == 0) {
    sh.red_culled[threadIdx.x >> 5] = c;
    if (sk) atomicAdd(&S->skip_it[it], sk);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long bc = 0;
    for (int w = 0; w < kExpandThreads / 32; ++w) bc += sh.red_culled[w];
    if (bc) atomicAdd(&S->culled_it[it], bc);
  }
}

// Persistent traversal: one cooperative launch runs every expansion
// iteration, separated by grid barriers.  Every block derives the same
// iteration parameters from the shared counters, so no block has to publish
// the next iteration's state; block 0 records the statistics.
template <bool kMax>
__global__ __launch_bounds__(kExpandThreads, 1024 / kExpandThreads) void k_traverse(QArgs q) {
  QState* S = q.S;
  __shared__ ExpandShared sh;
  extern __shared__ unsigned char k1_stage[];
  volatile QState* V = S;
  const bool rec = blockIdx.x == 0 && threadIdx.x == 0;
  if (rec) init_query<kMax>(q);  // S->bar was zeroed by the host (memset node)
  if (blockIdx.x == 0) {
    // per-iteration counters, zeroed by block 0's threads in parallel (the
    // grid barrier below publishes them)
    for (int i = threadIdx.x; i <= kMaxIters; i += blockDim.x) {
      S->cnt[i] = 0;
      if (i < kMaxIters) {
        S->culled_it[i] = 0;
        S->skip_it[i] = 0;
        S->t_sweep[i] = 0;
      }
    }
  }
  unsigned phase = 0;
  grid_barrier(&S->bar, ++phase);
  unsigned long long n_in = V->n_in;
  int it = V->iter, cur = 0, da = 0, db = 0;
  unsigned long long expanded = 0;
  const int la = min(q.cfg.split_level, q.A.depth), lb = min(q.cfg.split_level, q.B.depth);
  if (rec) S->t_it[it] = globaltimer_ns();
  while (n_in > 0 && it < kMaxIters) {
    const int ra = q.A.depth - da, rb = q.B.depth - db;
    const int rem = max(ra, rb);
    const int k = adaptive_k(n_in, q.cfg.front_cap, q.cfg.depth_cap, rem);
    const int ka = min(k, ra), kb = min(k, rb);
    const bool to_leaves = (k == rem);
    const unsigned long long ncand = n_in << (ka + kb);
    if (ncand > (unsigned long long)q.cfg.front_hard_cap) {  // query.py:373-376
      if (rec) {
        S->err = GD_ERR_FRONT_OVERFLOW;
        S->ov_cand = (long long)ncand;
        S->ov_in = (long long)n_in;
        S->ov_cap = q.cfg.front_hard_cap;
      }
      n_in = 0;
      break;
    }
    expand_sweep<kMax>(q, sh, k1_stage, it, cur, n_in, k, ka, kb, to_leaves, ncand, da, db, la, lb);
    if (q.profile && threadIdx.x == 0) atomicMax(&S->t_sweep[it], globaltimer_ns());
    const unsigned long long n_out = count_barrier(&S->cnt[it]);
    if (n_out > (unsigned long long)q.cfg.front_hard_cap) {  // query.py:448-449
      if (rec) {
        S->err = GD_ERR_FRONT_OVERFLOW;
        S->ov_cand = (long long)n_out;
        S->ov_in = (long long)n_in;
        S->ov_cap = q.cfg.front_hard_cap;
      }
      n_in = 0;
      break;
    }
    expanded += ncand - V->skip_it[it];  // candidates of the pairs this call owns
    if (rec) {
      S->t_it[it + 1] = globaltimer_ns();
      GdIterStat st;
      st.k = k;
      st.front_in = (long long)n_in;
      st.front_out = to_leaves ? 0 : (long long)n_out;
      st.culled = (long long)V->culled_it[it];
      const float b = __uint_as_float(V->bound_bits);
      st.bound_after = kMax ? (double)b + (double)S->slack : (double)b - (double)S->slack;
      st._pad = 0;
      S->stats[it] = st;
    }
    da += ka;
    db += kb;
    ++it;
    if (to_leaves) {
      if (rec) {
        S->n_leaf = n_out;
        S->leaf_buf = cur ^ 1;
      }
      n_in = 0;
      break;
    }
    cur ^= 1;
    n_in = n_out;
  }
  if (rec) {
    S->iter = it;
    S->expanded += expanded;
    S->n_in = 0;
    S->depth_a = da;
    S->depth_b = db;
    S->cur = cur;
  }
}

}  // namespace gd
