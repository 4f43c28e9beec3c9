// traverse.cu -- the BVTT front traversal (query.py:266-509): query
// prologue, the front arena's level stack, the expansion sweeps and the
// persistent k_traverse kernels.  Its own compilation unit, built with
// -maxrregcount=64 (_build.py): the serial stack bookkeeping (plan_sweep /
// commit_sweep, thread 0 of each block) is out of line within the kernel's
// 64-register budget, so the k = 1 sweep -- the bulk of the traversal --
// keeps its registers.
#include "traverse.cuh"

namespace gd {

// Device schedule (GdConfig.schedule >= 0): k = 1 sweeps of fronts of at
// least this many entries take the bound update (the enhanced bound of each
// entry's most promising kept child pair, ~90 instructions) from the first
// round of every tile only -- a quarter of the entries.  By then the bound
// has converged (rings: it moves by < 1e-4 relative over the last five
// iterations), any kept pair's bound is valid, and the sweeps are issue /
// latency bound: rings min expand 0.252 -> 0.244 ms.  The reference schedule
// (-1) updates from every entry, as query.py:416-423.
#ifndef GD_K1_THIN_BOUND
#define GD_K1_THIN_BOUND 200000u
#endif

// ownership test compiled out of the single-GPU traversal (kSplit = false):
// the sweeps run at 64 registers, and every live value counts
template <bool kSplit>
__device__ __forceinline__ bool owns(const GdConfig& c, unsigned na, unsigned nb, int da, int db, int la, int lb) {
  return !kSplit || owned(c, na, nb, da, db, la, lb);
}

// query prologue (one thread; k_traverse block 0 before its first barrier):
// root key and bound, slack, root level of the front stack, counters,
// warm_pair
template <bool kMax>
__device__ void init_query(const QArgs& q) {
  QState* S = q.S;
  Box ra = load_box(q.A.box, 0), rb = load_box(q.B.box, 0);
  float M = 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    M = fmaxf(M, fmaxf(fmaxf(fabsf(ra.lo[k]), fabsf(ra.hi[k])), fmaxf(fabsf(rb.lo[k]), fabsf(rb.hi[k]))));
  // The float32 vertices are R v + t of the staged float32 base vertices:
  // their rounding scales with the FMA chain's partial sums |R||v| + |t|
  // (S below), not only with the result -- a mesh authored far from the
  // origin and moved back by its transform.  xf_apply's error is <= 4 ulps
  // of S per coordinate, so a distance moves by <= 14 * 2^-24 S; S / 8 in M
  // keeps that under half of E / 2 = 2^-16 M.
  M = fmaxf(M, 0.125f * fmaxf(xf_mag(q.xa, stage_mag(q.A)), xf_mag(q.xb, stage_mag(q.B))));
  if (q.cfg.frame == 1 && q.cfg.precision == 32 && q.mb.has_xf) {
    // B-local traversal at precision 32: the exact pass reproduces the
    // reference's float32 arithmetic on WORLD coordinates, whose rounding
    // scales with |Rb x + tb| <= |Rb|_inf M + |tb| (float64 needs no term)
    float rs = 0.f, tm = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rs = fmaxf(rs, (float)(fabs(q.mb.rot[3 * i]) + fabs(q.mb.rot[3 * i + 1]) + fabs(q.mb.rot[3 * i + 2])));
      tm = fmaxf(tm, (float)fabs(q.mb.trans[i]));
    }
    M = fmaxf(M, rs * M + tm);
  }
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
  S->iter = 0;
  S->sp = 0;
  S->chunked = 0;
  S->pending = 0;
  S->paused = 0;
  S->rounds = 0;
  S->lo_top = 1;  // the root entry
  S->hi_bot = q.arena;
  S->leaf_off = 0;
  S->leaf_end = 0;
  S->n_leaf = 0;
  S->n_band = 0;
  S->n_cand = 0;
  S->fbest = kMax ? 0u : __float_as_uint(INFINITY);
  S->expanded = 0;
  S->ncand_total = 0;
  S->narrow = 0;
  S->culled = 0;
  S->band_eval = 0;
  S->band_overflow = 0;
  S->rescanned = 0;
  S->ov_cand = S->ov_in = S->ov_cap = 0;
  if (q.A.depth == 0 && q.B.depth == 0) {
    q.fnode[0] = make_uint2(0, 0);
    q.fkey[0] = key0;
    // both roots are leaves: narrow phase immediately (query.py:510-518)
    S->n_leaf = 1;
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
#ifndef GD_ROOT_END
#define GD_ROOT_END 0
#endif
    Level root;
    root.end = GD_ROOT_END;
    root.off = root.end ? q.arena - 1 : 0;
    root.n = 1;
    root.cur = 0;
    root.da = root.db = 0;
    root.it = 0;
    q.fnode[root.off] = make_uint2(0, 0);
    q.fkey[root.off] = key0;
    if (root.end) {
      S->lo_top = 0;
      S->hi_bot = q.arena - 1;
    }
    S->lv[0] = root;
    S->sp = 1;
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

// a later round (the previous one ended with a leaf chunk for the narrow
// phase, which has consumed it): release the leaf list, fresh band
__device__ void resume_round(const QArgs& q) {
  QState* S = q.S;
  if (S->n_leaf) {
    if (S->leaf_end == 0)
      S->lo_top = S->leaf_off;
    else
      S->hi_bot = S->leaf_off + S->n_leaf;
    S->n_leaf = 0;
  }
  S->n_band = 0;
  S->n_cand = 0;
  S->band_overflow = 0;
  S->rescanned = 0;
  S->done = 0;
}

// ---------------------------------------------------------------------------
// Shared per-block plumbing of an expansion sweep: survivors are compacted
// with one global atomic per tile, bound updates reduced to one atomic per
// tile (the paper's block-wise reduction).
struct ExpandShared {
  unsigned long long out_base;
  unsigned warp_tot[kExpandThreads / 32];
  float warp_upd[2][kExpandThreads / 32];
  unsigned stage_count;
};

// One sweep: entries [in_off, in_off + c) of the arena (depth pair da, db)
// expanded k levels; survivors go to output slots out_base + dir * slot.
struct SweepPlan {
  unsigned long long in_off, c, out_base;
  int out_dir, out_end, k, ka, kb, da, db, it, to_leaves;
  int stop;  // 0 = sweep, 1 = stack empty, 2 = leaf chunk ready, 3 = error
};
// every block keeps an identical copy of the front stack; thread 0 of each
// block advances it deterministically from the same survivor counts
struct TravShared {
  Level lv[kMaxLevels];
  unsigned long long tot_cand[kMaxIters], tot_in[kMaxIters], tot_out[kMaxIters];
  unsigned long long lo, hi, leaf_off, leaf_n;
  int sp, chunked, leaf_end, iter;
  int stat_it, stat_k, stat_leaf, stat_pending;  // block 0: statistics of the last sweep, written during the next
  unsigned long long ncand_total;                 // candidates expanded so far (all rounds)
  SweepPlan p[2];
};

__device__ __forceinline__ unsigned long long out_slot(const SweepPlan& p, unsigned long long i) {
  return p.out_dir > 0 ? p.out_base + i : p.out_base - i;
}

template <bool kMax>
__device__ __forceinline__ void write_stat(QState* S, TravShared& t);

// A grid barrier that can never complete (a bug) must not hang the GPU:
// after ~2^26 polls (tens of seconds; a sweep's barrier takes microseconds)
// the kernel traps -- the launch fails loudly with an error instead.
__device__ __forceinline__ void spin_watchdog(unsigned polls) {
  if (polls == (1u << 26)) __trap();
}

// Grid-wide barrier of the persistent traversal (all blocks co-resident:
// cooperative launch).  `bar` only grows; phase p completes when it reaches
// p * gridDim.x, so no reset is needed inside a launch.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// release-arrive / acquire-spin: every block's writes before the barrier are
// visible to every block after it.  Data written in the same launch (fronts,
// counters) is read with plain coherent loads, never through __ldg.
// Sweep barrier fused with the survivor count: cnt holds the survivors (low
// 40 bits, reserved by the tiles with plain atomicAdd) and the block arrivals
// (high 24 bits).  Returns the final survivor count -- no separate load after
// the barrier.
constexpr int kArriveShift = 40;
// Block 0 writes the previous sweep's statistics (stat) between its arrival
// and the spin, where their loads cost nothing unless it arrives last.
template <bool kMax>
__device__ __forceinline__ unsigned long long count_barrier(unsigned long long* cnt, QState* S = nullptr,
                                                            TravShared* stat = nullptr) {
  __shared__ unsigned long long total;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long target = (unsigned long long)gridDim.x << kArriveShift;
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(cnt), "l"(1ull << kArriveShift) : "memory");
    if (stat) write_stat<kMax>(S, *stat);
    unsigned long long v;
    unsigned polls = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
      spin_watchdog(++polls);
    } while ((v & ~((1ull << kArriveShift) - 1)) < target);
    total = v & ((1ull << kArriveShift) - 1);
  }
  __syncthreads();
  return total;
}

// The launch's start: block 0 runs the prologue, then publishes the launch's
// epoch (unique per launch, from the host); every other block waits for it.
// Nothing else crosses blocks before the first sweep barrier, so no counted
// grid barrier -- and no counter to reset with a memset before the launch --
// is needed.  A workspace's stale flag is an older epoch of this process (or
// garbage), never the current one.
__device__ __forceinline__ void prologue_barrier(unsigned long long* flag, unsigned long long epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flag), "l"(epoch) : "memory");
    } else {
      unsigned long long v;
      unsigned polls = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        spin_watchdog(++polls);
      } while (v != epoch);
    }
  }
  __syncthreads();
}

// warp-aggregated append of `cnt` items into a shared-memory list; returns
// this lane's first position (all lanes of the warp must call it)
__device__ __forceinline__ unsigned warp_append(unsigned* counter, unsigned cnt) {
  const int lane = threadIdx.x & 31;
  unsigned incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  unsigned wbase = 0;
  if (lane == 31 && incl) wbase = atomicAdd(counter, incl);
  wbase = __shfl_sync(0xffffffffu, wbase, 31);
  return wbase + incl - cnt;
}

// Every candidate of a sweep is culled, survives, or (split query) belongs
// to another rank, so an iteration's reference-equivalent culled count is
// derived from its totals (write_stat): only the skipped candidates of a
// split query are counted, per warp.  (my_culled stays in the sweeps as the
// reference's accounting; the compiler drops it.)
__device__ __forceinline__ void sweep_counters(QState* S, ExpandShared&, int it, unsigned long long,
                                               unsigned long long my_skipped, bool split) {
  if (!split) return;
  const unsigned long long sk = warp_sum_u64(my_skipped);
  if ((threadIdx.x & 31) == 0 && sk) atomicAdd(&S->skip_it[it], sk);
}

// k == 1 sweep (the wide late iterations): one thread per front entry; it
// loads the (1 or 2) child boxes of each side once (contiguous siblings) and
// tests the <= 4 child pairs -- 14 loads per entry instead of 32.  Survivors
// are staged in shared memory (warp-aggregated appends), then one global
// reservation per tile and a coalesced copy-out.  A tile is R rounds of one
// entry per thread; R shrinks with the front so a small front spreads over
// all blocks (latency, not throughput, bounds it).  (expand_sweep with k = 1,
// specialised: the bulk of the traversal's bytes go through this loop.)
template <bool kMax, bool kSplit>
__device__ __forceinline__ void k1_sweep(const QArgs& q, ExpandShared& sh, unsigned char* stage, const SweepPlan& p,
                                         unsigned long long* n_out, int la, int lb) {
  QState* S = q.S;
  const int ka = p.ka, kb = p.kb;
  const unsigned n_in = (unsigned)p.c;  // chunks are < 2^31 entries (the arena is)
  const uint2* __restrict__ in_node = q.fnode + p.in_off;
  const float* __restrict__ in_key = q.fkey + p.in_off;
  const unsigned leaf_a0 = (unsigned)((1ull << q.A.depth) - 1), leaf_b0 = (unsigned)((1ull << q.B.depth) - 1);
  const unsigned ra0 = p.to_leaves ? leaf_a0 : 0u, rb0 = p.to_leaves ? leaf_b0 : 0u;  // output index base
  const bool to_leaves = p.to_leaves;
  const int da = p.da, db = p.db;
  const bool culling = q.cfg.culling != 0, enh = q.cfg.enhanced_bounds != 0;
  unsigned my_culled = 0, my_skipped = 0;  // skipped: not owned (split query); < 2^32 per thread and sweep
  uint2* s_node = reinterpret_cast<uint2*>(stage);
  float* s_key = reinterpret_cast<float*>(stage + kK1Stage * sizeof(uint2));
  const int ca = 1 << ka, cb = 1 << kb;
  const int lane = threadIdx.x & 31;
  const bool thin_bound = q.cfg.schedule >= 0 && n_in >= (unsigned)GD_K1_THIN_BOUND;
  // even contiguous split of the chunk over the blocks (no tail imbalance at
  // the grid barrier), processed in tiles of <= kK1Rounds rounds of one entry
  // per thread
  unsigned per_blk = (n_in + gridDim.x - 1) / gridDim.x;
  per_blk = (per_blk + 63) & ~63u;
  const unsigned blk_lo = min(n_in, blockIdx.x * per_blk);
  const unsigned blk_hi = min(n_in, blk_lo + per_blk);
  for (unsigned t0 = blk_lo; t0 < blk_hi; t0 += kK1Tile) {
    const unsigned t1 = min(blk_hi, t0 + kK1Tile);
    const int R = (int)((t1 - t0 + kExpandThreads - 1) / kExpandThreads);
    if (threadIdx.x == 0) sh.stage_count = 0;
    // entry loads are software-pipelined one round ahead
    const unsigned e0 = t0 + threadIdx.x;
    float pk_next = e0 < t1 ? in_key[e0] : 0.f;
    uint2 nd_next = e0 < t1 ? in_node[e0] : make_uint2(0, 0);
    const float ub = load_bound_sq(S);  // one bound snapshot per tile (query.py:396)
    __syncthreads();
    float upd = kMax ? 0.f : INFINITY;
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      const unsigned e = t0 + (unsigned)r * kExpandThreads + threadIdx.x;
      const float pk = pk_next;
      uint2 nd = nd_next;
      if (r + 1 < R && e + kExpandThreads < t1) {
        pk_next = in_key[e + kExpandThreads];
        nd_next = in_node[e + kExpandThreads];
      }
      unsigned keep = 0;
      float keys[4];
      const bool mine = e < t1 && owns<kSplit>(q.cfg, nd.x, nd.y, da, db, la, lb);
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
          if (keep && !to_leaves && (r == 0 || !thin_bound)) {
            const Box ba = select_box((bc >> 1) != 0, A[1], A[0]);
            const Box bb = select_box((bc & 1) != 0, B[1], B[0]);
            const float u = pair_update<kMax>(ba, bb, enh);
            upd = kMax ? fmaxf(upd, u) : fminf(upd, u);
          }
          nd = make_uint2(a0, b0);
        }
      }
      // warp-aggregated append into the shared staging area
      unsigned pos = warp_append(&sh.stage_count, __popc(keep));
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
    if (lane == 0) sh.warp_upd[0][threadIdx.x >> 5] = upd;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned total = sh.stage_count;
      // low 40 bits: survivors so far (blocks that finished have added their
      // arrival in the high bits, count_barrier)
      sh.out_base = total ? (atomicAdd(n_out, (unsigned long long)total) & ((1ull << kArriveShift) - 1)) : 0ull;
      float u = sh.warp_upd[0][0];
      for (int w = 1; w < kExpandThreads / 32; ++w) u = kMax ? fmaxf(u, sh.warp_upd[0][w]) : fminf(u, sh.warp_upd[0][w]);
      if (kMax ? u > 0.f : u < INFINITY) commit_bound<kMax>(q, sqrtf(u), ub);
    }
    __syncthreads();
    const unsigned total = sh.stage_count;
    const long long base = (long long)sh.out_base, dir = p.out_dir;
    uint2* const on = q.fnode + p.out_base;
    float* const ok = q.fkey + p.out_base;
    for (unsigned i = threadIdx.x; i < total; i += kExpandThreads) {
      const long long o = dir * (base + (long long)i);
      on[o] = s_node[i];
      ok[o] = s_key[i];
    }
    __syncthreads();  // staging reuse by the next tile
  }
  sweep_counters(S, sh, p.it, my_culled, my_skipped, kSplit);
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

// k == 2 sweep (two levels per iteration on both trees): one thread per
// CHILD pair of a front entry -- the k = 1 expansion of that child pair,
// without writing the intermediate front.  Thread v handles entry v / 4,
// child pair v % 4 = (i, j); its loads (the entry, then the children of A
// child i and of B child j: 3 float4 each) are independent, so one round
// trip covers both levels.  A child's box is the union of its two
// children's (the refit's fold: bitwise), so it is not loaded.  Same
// survivors as the reference's 16-candidate expansion (a grandchild pair's
// key is monotone in its child pair's); culled counts are the
// reference-equivalent ones.  Tiles, staging and the bound reduction as in
// k1_sweep.
template <bool kMax, bool kSplit>
__device__ __forceinline__ void k2_sweep(const QArgs& q, ExpandShared& sh, unsigned char* stage, const SweepPlan& p,
                                         unsigned long long* n_out, int la, int lb) {
  QState* S = q.S;
  const unsigned n_v = 4u * (unsigned)p.c;  // child pairs (k2 chunks are < 2^28 entries: rem <= schedule < 2^31 / 16)
  const uint2* __restrict__ in_node = q.fnode + p.in_off;
  const float* __restrict__ in_key = q.fkey + p.in_off;
  const unsigned ra0 = p.to_leaves ? (unsigned)((1ull << q.A.depth) - 1) : 0u;
  const unsigned rb0 = p.to_leaves ? (unsigned)((1ull << q.B.depth) - 1) : 0u;
  const bool to_leaves = p.to_leaves;
  const bool culling = q.cfg.culling != 0, enh = q.cfg.enhanced_bounds != 0;
  unsigned my_culled = 0, my_skipped = 0;
  uint2* s_node = reinterpret_cast<uint2*>(stage);
  float* s_key = reinterpret_cast<float*>(stage + kK1Stage * sizeof(uint2));
  const int lane = threadIdx.x & 31;
  unsigned per_blk = (n_v + gridDim.x - 1) / gridDim.x;
  per_blk = (per_blk + 63) & ~63u;
  const unsigned blk_lo = min(n_v, blockIdx.x * per_blk);
  const unsigned blk_hi = min(n_v, blk_lo + per_blk);
  for (unsigned t0 = blk_lo; t0 < blk_hi; t0 += kK1Tile) {
    const unsigned t1 = min(blk_hi, t0 + kK1Tile);
    const int R = (int)((t1 - t0 + kExpandThreads - 1) / kExpandThreads);
    if (threadIdx.x == 0) sh.stage_count = 0;
    const float ub = load_bound_sq(S);
    __syncthreads();
    float upd = kMax ? 0.f : INFINITY;
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      const unsigned v = t0 + (unsigned)r * kExpandThreads + threadIdx.x;
      unsigned keep = 0;
      float keys[4];
      uint2 nd = make_uint2(0, 0);
      if (v < t1) {
        const float pk = in_key[v >> 2];
        nd = in_node[v >> 2];
        if (!owns<kSplit>(q.cfg, nd.x, nd.y, p.da, p.db, la, lb)) {
          my_skipped += 4;
        } else if (culling && !survives<kMax>(pk, ub)) {
          my_culled += 4;
        } else {
          const unsigned an = 2 * nd.x + 1 + ((v >> 1) & 1), bn = 2 * nd.y + 1 + (v & 1);
          Box A[2], B[2];
          load_children(q.A.box, an, A[0], A[1]);
          load_children(q.B.box, bn, B[0], B[1]);
          const Box ca = box_union(A[0], A[1]), cb = box_union(B[0], B[1]);
          if (culling && !survives<kMax>(pair_key<kMax>(ca, cb), ub)) {
            my_culled += 4;  // the child pair: its grandchildren are culled with it
          } else {
            // bound: the kept child pair's enhanced bound when the
            // grandchildren are leaves (which emit none), else the most
            // promising kept grandchild pair's -- both kept non-leaf pairs
            if (to_leaves) {
              const float u = pair_update<kMax>(ca, cb, enh);
              upd = kMax ? fmaxf(upd, u) : fminf(upd, u);
            }
            float best = kMax ? -INFINITY : INFINITY;
            int bc = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float key = pair_key<kMax>(A[c >> 1], B[c & 1]);
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
            if (keep && !to_leaves) {
              const float u = pair_update<kMax>(select_box((bc >> 1) != 0, A[1], A[0]),
                                                select_box((bc & 1) != 0, B[1], B[0]), enh);
              upd = kMax ? fmaxf(upd, u) : fminf(upd, u);
            }
            nd = make_uint2(2 * an + 1 - ra0, 2 * bn + 1 - rb0);  // first grandchild of each side
          }
        }
      }
      unsigned pos = warp_append(&sh.stage_count, __popc(keep));
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (keep & (1u << c)) {
          s_node[pos] = make_uint2(nd.x + (c >> 1), nd.y + (c & 1));
          s_key[pos] = keys[c];
          ++pos;
        }
      }
    }  // rounds
    upd = kMax ? warp_max(upd) : warp_min(upd);
    if (lane == 0) sh.warp_upd[0][threadIdx.x >> 5] = upd;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned total = sh.stage_count;
      sh.out_base = total ? (atomicAdd(n_out, (unsigned long long)total) & ((1ull << kArriveShift) - 1)) : 0ull;
      float u = sh.warp_upd[0][0];
      for (int w = 1; w < kExpandThreads / 32; ++w) u = kMax ? fmaxf(u, sh.warp_upd[0][w]) : fminf(u, sh.warp_upd[0][w]);
      if (kMax ? u > 0.f : u < INFINITY) commit_bound<kMax>(q, sqrtf(u), ub);
    }
    __syncthreads();
    const unsigned total = sh.stage_count;
    const long long base = (long long)sh.out_base, dir = p.out_dir;
    uint2* const on = q.fnode + p.out_base;
    float* const ok = q.fkey + p.out_base;
    for (unsigned i = threadIdx.x; i < total; i += kExpandThreads) {
      const long long o = dir * (base + (long long)i);
      on[o] = s_node[i];
      ok[o] = s_key[i];
    }
    __syncthreads();
  }
  sweep_counters(S, sh, p.it, my_culled, my_skipped, kSplit);
}

// k >= 2 sweep (the narrow early fronts, candidates < front_cap): one thread
// per candidate of the reference's k-level expansion (query.py:349-451:
// candidate t -> entry t >> (ka + kb), descendants ((node + 1) << k) - 1 +
// offset, bvh.py:309-335) -- k levels for one load round trip.
template <bool kMax, bool kSplit>
__device__ __forceinline__ void generic_sweep(const QArgs& q, ExpandShared& sh, const SweepPlan& p,
                                              unsigned long long* n_out, int la, int lb) {
  QState* S = q.S;
  const int ka = p.ka, kb = p.kb, shift = ka + kb;
  const uint2* __restrict__ in_node = q.fnode + p.in_off;
  const float* __restrict__ in_key = q.fkey + p.in_off;
  const unsigned leaf_a0 = (unsigned)((1ull << q.A.depth) - 1), leaf_b0 = (unsigned)((1ull << q.B.depth) - 1);
  const unsigned ra0 = p.to_leaves ? leaf_a0 : 0u, rb0 = p.to_leaves ? leaf_b0 : 0u;
  const bool culling = q.cfg.culling != 0, enh = q.cfg.enhanced_bounds != 0;
  const unsigned long long ncand = p.c << shift;
  const unsigned long long tiles = (ncand + kExpandThreads - 1) / kExpandThreads;
  const unsigned long long off_mask = (1ull << shift) - 1, mask_b = (1ull << kb) - 1;
  uint2* const on = q.fnode + p.out_base;
  float* const ok = q.fkey + p.out_base;
  const long long dir = p.out_dir;
  unsigned long long my_culled = 0, my_skipped = 0;
  for (unsigned long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const unsigned long long t = tile * kExpandThreads + threadIdx.x;
    const float ub = load_bound_sq(S);
    float upd = kMax ? 0.f : INFINITY;
    uint2 o_node = make_uint2(0, 0);
    float o_key = 0.f;
    bool keep = false;
    if (t < ncand) {
      const unsigned long long e = t >> shift, off = t & off_mask;
      const float pk = in_key[e];
      const uint2 nd = in_node[e];
      const unsigned na = (unsigned)(((((unsigned long long)nd.x + 1) << ka) - 1) + (off >> kb));
      const unsigned nb = (unsigned)(((((unsigned long long)nd.y + 1) << kb) - 1) + (off & mask_b));
      if (!owns<kSplit>(q.cfg, nd.x, nd.y, p.da, p.db, la, lb)) {
        ++my_skipped;
      } else if (culling && !survives<kMax>(pk, ub)) {
        ++my_culled;
      } else {
        const Box ba = load_box(q.A.box, na), bb = load_box(q.B.box, nb);
        const float key = pair_key<kMax>(ba, bb);
        if (culling && !survives<kMax>(key, ub)) {
          ++my_culled;
        } else {
          keep = true;
          o_node = make_uint2(na - ra0, nb - rb0);
          o_key = key;
          if (!p.to_leaves) upd = pair_update<kMax>(ba, bb, enh);
        }
      }
    }
    unsigned total;
    const unsigned my_off = block_exclusive_scan(keep ? 1u : 0u, sh.warp_tot, total);
    upd = kMax ? warp_max(upd) : warp_min(upd);
    if ((threadIdx.x & 31) == 0) sh.warp_upd[0][threadIdx.x >> 5] = upd;
    __syncthreads();
    if (threadIdx.x == 0) {
      // low 40 bits: survivors so far (blocks that finished have added their
      // arrival in the high bits, count_barrier)
      sh.out_base = total ? (atomicAdd(n_out, (unsigned long long)total) & ((1ull << kArriveShift) - 1)) : 0ull;
      float u = sh.warp_upd[0][0];
      for (int w = 1; w < kExpandThreads / 32; ++w) u = kMax ? fmaxf(u, sh.warp_upd[0][w]) : fminf(u, sh.warp_upd[0][w]);
      if (kMax ? u > 0.f : u < INFINITY) commit_bound<kMax>(q, sqrtf(u), ub);
    }
    __syncthreads();
    if (keep) {
      const long long o = dir * (long long)(sh.out_base + my_off);
      on[o] = o_node;
      ok[o] = o_key;
    }
    __syncthreads();
  }
  sweep_counters(S, sh, p.it, my_culled, my_skipped, kSplit);
}

// pop a consumed level: it is the top of its end of the arena
__device__ __forceinline__ void release_level(TravShared& t, const Level& L) {
  if (L.end == 0)
    t.lo = L.off;
  else
    t.hi = L.off + L.n;
}

// Next sweep from the top of the stack (thread 0 of every block, identical
// results).  Schedule: the reference's adaptive_depth on the level's
// remaining entries.  Chunking: the children of c entries must fit the gap
// between the arena's two stacks with room for every deeper level (each gets
// gap / D in the worst case, D = levels still to come + 2 for the leaf list
// and its candidates); when the whole level does not fit, it is expanded in
// chunks, depth first, with k = 1 from then on (uniform depth per iteration
// index).
template <bool kMax>
__device__ __noinline__ void plan_sweep(const QArgs& q, TravShared& t, SweepPlan& p, bool rec) {
  QState* S = q.S;
  p.stop = 0;
  while (true) {
    if (t.sp == 0) {
      p.stop = 1;
      return;
    }
    const Level& L = t.lv[t.sp - 1];
    if (L.cur < L.n) break;
    release_level(t, L);
    --t.sp;
  }
  const Level& L = t.lv[t.sp - 1];
  const unsigned long long rem = L.n - L.cur;
  const int ra = q.A.depth - L.da, rb = q.B.depth - L.db, rd = max(ra, rb);
  // floor(x / y) through float64 (exact: the quotient is rounded down and
  // checked), cheaper than the 64-bit integer division in the serial path
  auto divf = [](unsigned long long x, unsigned long long y) -> unsigned long long {
    unsigned long long d = (unsigned long long)((double)x / (double)y);
    while (d > 0 && d * y > x) --d;
    while ((d + 1) * y <= x) ++d;
    return d;
  };
  // adaptive_depth (query.py:266-284): the largest k with n 4^(k+1) <
  // front_cap, clamped to depth_cap and the remaining depth -- the
  // reference's schedule, so the iteration statistics follow it
  int k = 1;
  if (!t.chunked)
    while (k < q.cfg.depth_cap && k < rd && 2 * (k + 1) < 62 && (rem >> (62 - 2 * (k + 1))) == 0 &&
           (rem << (2 * (k + 1))) < (unsigned long long)q.cfg.front_cap)
      ++k;
  // device schedule (GdConfig.schedule >= 0): where the rule above gives
  // k = 1, a front of at most the threshold's entries expands two levels in
  // one k2_sweep -- a grid barrier and a front write / re-read per level
  // saved where the iteration is latency bound.  Only while its <= 16 rem
  // candidates fit front_hard_cap: then neither of the two reference
  // iterations it replaces could raise FrontOverflowError either.
  if (k == 1 && !t.chunked && q.cfg.schedule >= 0 && q.cfg.depth_cap >= 2 && ra >= 2 && rb >= 2 &&
      rem <= (q.cfg.schedule > 0 ? (unsigned long long)q.cfg.schedule : kK2Front) &&
      (rem << 4) <= (unsigned long long)q.cfg.front_hard_cap)
    k = 2;
  const unsigned long long gap = t.hi - t.lo;
  auto fit = [&](int kk) -> unsigned long long {
    const int s = min(kk, ra) + min(kk, rb);
    const unsigned long long D = ((unsigned long long)(rd - kk) + 2) << s;
    return rem * D <= gap ? rem : divf(gap, D);  // the whole level (no division) or a chunk
  };
  unsigned long long c = fit(k);
  if (c < rem && !t.chunked) {
    t.chunked = 1;
    k = 1;
    c = fit(1);
  }
  c = min(c, rem);
  if (c == 0) {
    p.stop = 3;
    if (rec) S->err = GD_ERR_WORKSPACE;  // arena smaller than a few entries per level
    return;
  }
  p.k = k;
  p.ka = min(k, ra);
  p.kb = min(k, rb);
  p.to_leaves = k == rd;
  p.c = c;
  p.in_off = L.off + L.cur;
  p.da = L.da;
  p.db = L.db;
  p.it = L.it;
  p.out_end = L.end ^ 1;
  p.out_dir = p.out_end == 0 ? 1 : -1;
  p.out_base = p.out_end == 0 ? t.lo : t.hi - 1;
  // FrontOverflowError before the expansion (query.py:373-376), on the
  // iteration's candidates summed over its chunks
  const unsigned long long ncand = c << (p.ka + p.kb);
  if (t.tot_cand[L.it] + ncand > (unsigned long long)q.cfg.front_hard_cap || L.it + 1 >= kMaxIters) {
    p.stop = 3;
    if (rec) {
      S->err = GD_ERR_FRONT_OVERFLOW;
      S->ov_cand = (long long)(t.tot_cand[L.it] + ncand);
      S->ov_in = (long long)(t.tot_in[L.it] + c);
      S->ov_cap = q.cfg.front_hard_cap;
    }
  }
}

// account a finished sweep and push its survivors (thread 0 of every block);
// block 0 records the iteration statistics
template <bool kMax>
__device__ __noinline__ void commit_sweep(const QArgs& q, TravShared& t, const SweepPlan& p, SweepPlan& nx,
                             unsigned long long n_out, bool rec) {
  QState* S = q.S;
  nx.stop = 0;
  Level& L = t.lv[t.sp - 1];
  const int it = p.it;
  const unsigned long long ncand = p.c << (p.ka + p.kb);
  t.tot_cand[it] += ncand;
  t.tot_in[it] += p.c;
  t.tot_out[it] += n_out;  // survivors: front entries, or leaf pairs for the narrow phase
  t.iter = max(t.iter, it + 1);
  if (rec) {
    // the statistics are written during the next sweep (stat_pending): their
    // loads must not delay block 0's start of it
    t.ncand_total += ncand;
    t.stat_it = it;
    t.stat_k = p.k;
    t.stat_leaf = p.to_leaves;
    t.stat_pending = 1;
    if (q.profile) S->t_it[it + 1] = globaltimer_ns();
  }
  // FrontOverflowError after the expansion (query.py:448-449); leaf pairs
  // are not a front (the reference narrows them at once)
  if (!p.to_leaves && t.tot_out[it] > (unsigned long long)q.cfg.front_hard_cap) {
    nx.stop = 3;
    if (rec) {
      S->err = GD_ERR_FRONT_OVERFLOW;
      S->ov_cand = (long long)t.tot_out[it];
      S->ov_in = (long long)t.tot_in[it];
      S->ov_cap = q.cfg.front_hard_cap;
    }
    return;
  }
  L.cur += p.c;
  if (L.cur == L.n) {
    release_level(t, L);
    --t.sp;
  }
  if (n_out == 0) return;
  const unsigned long long off = p.out_end == 0 ? t.lo : t.hi - n_out;
  if (p.out_end == 0)
    t.lo += n_out;
  else
    t.hi -= n_out;
  if (p.to_leaves) {  // the round ends: this chunk's leaf pairs go to the narrow phase
    t.leaf_off = off;
    t.leaf_n = n_out;
    t.leaf_end = p.out_end;
    nx.stop = 2;
    return;
  }
  if (t.sp >= kMaxLevels) {
    nx.stop = 3;
    if (rec) S->err = GD_ERR_WORKSPACE;
    return;
  }
  Level& N = t.lv[t.sp++];
  N.off = off;
  N.n = n_out;
  N.cur = 0;
  N.da = p.da + p.ka;
  N.db = p.db + p.kb;
  N.it = it + 1;
  N.end = p.out_end;
}

// block 0, thread 0: IterationStat of the last committed sweep
template <bool kMax>
__device__ __forceinline__ void write_stat(QState* S, TravShared& t) {
  const volatile QState* V = S;
  const int it = t.stat_it;
  GdIterStat st;
  st.k = t.stat_k;
  st.front_in = (long long)t.tot_in[it];
  st.front_out = t.stat_leaf ? 0 : (long long)t.tot_out[it];
  // culled = candidates - survivors - (split query) candidates other ranks own
  st.culled = (long long)(t.tot_cand[it] - t.tot_out[it] - V->skip_it[it]);
  const float b = __uint_as_float(V->bound_bits);
  st.bound_after = kMax ? (double)b + (double)S->slack : (double)b - (double)S->slack;
  st._pad = 0;
  S->stats[it] = st;
  t.stat_pending = 0;
}

// Persistent traversal round: one cooperative launch runs sweeps until the
// stack is empty or a leaf chunk is ready for the narrow phase (one round
// for a front that fits the arena: breadth first, like the reference's
// iterations), separated by grid barriers.  Every block derives the same
// sweep plans from the shared counters, so no block has to publish them;
// block 0 records the statistics and writes the stack back for the next round.
template <bool kMax, bool kSplit>
__device__ __forceinline__ void traverse_round(const QArgs& q) {
  QState* S = q.S;
  __shared__ ExpandShared sh;
  __shared__ TravShared t;
  __shared__ QArgs qs;  // the out-of-line functions' view of the arguments (shared, not a local copy)
  extern __shared__ __align__(16) unsigned char stage[];
  const volatile QState* V = S;
  // mode 1 (bound-exchange rounds): a later launch continues a query its
  // sweep budget paused, and does nothing once the traversal has ended.
  // Every block reads `paused` before the first grid barrier; block 0
  // rewrites it only after its last one.
  const bool cont = q.mode == 1 && q.round > 0;
  if (cont && !V->paused) return;
  if (threadIdx.x == 0) qs = q;
  const bool rec = blockIdx.x == 0 && threadIdx.x == 0;
  if (rec && q.profile) S->t_edge[0] = globaltimer_ns();
  if (blockIdx.x == 0) {
    if (q.round == 0) {
      if (threadIdx.x == 0) init_query<kMax>(q);
      // per-iteration counters, zeroed by block 0's threads in parallel (the
      // grid barrier below publishes them)
      for (int i = threadIdx.x; i < kMaxIters; i += blockDim.x) {
        S->skip_it[i] = 0;
        S->t_sweep[i] = 0;
        S->tot_cand[i] = 0;
        S->tot_in[i] = 0;
        S->tot_out[i] = 0;
      }
    } else if (threadIdx.x == 0 && !cont) {
      resume_round(q);
    }
    if (threadIdx.x < 3) S->cnt[threadIdx.x] = 0;
  }
  prologue_barrier(&S->epoch_flag, q.epoch);
  if (rec && q.profile) S->t_edge[1] = globaltimer_ns();
  for (int i = threadIdx.x; i < kMaxIters; i += blockDim.x) {
    t.tot_cand[i] = V->tot_cand[i];
    t.tot_in[i] = V->tot_in[i];
    t.tot_out[i] = V->tot_out[i];
  }
  __syncthreads();  // thread 0's plan_sweep reads the totals other threads copied (racecheck)
  if (threadIdx.x == 0) {
    t.sp = V->sp;
    for (int i = 0; i < t.sp; ++i) {
      const volatile Level& s = V->lv[i];
      Level& d = t.lv[i];
      d.off = s.off;
      d.n = s.n;
      d.cur = s.cur;
      d.da = s.da;
      d.db = s.db;
      d.it = s.it;
      d.end = s.end;
    }
    t.lo = V->lo_top;
    t.hi = V->hi_bot;
    t.chunked = V->chunked;
    t.iter = V->iter;
    t.ncand_total = V->ncand_total;
    t.leaf_n = 0;
    t.stat_pending = 0;
    if (rec && q.profile && q.round == 0) S->t_it[0] = globaltimer_ns();
    plan_sweep<kMax>(qs, t, t.p[0], rec);
  }
  __syncthreads();
  const int la = min(q.cfg.split_level, q.A.depth), lb = min(q.cfg.split_level, q.B.depth);
  unsigned sweep = 0;
  int b = 0;
  while (true) {
    const SweepPlan& p = t.p[b];  // shared: no register copy of the plan
    if (p.stop) break;
    unsigned long long* cnt = &S->cnt[sweep % 3];
    if (p.k == 2 && p.ka == 2 && p.kb == 2)
      k2_sweep<kMax, kSplit>(q, sh, stage, p, cnt, la, lb);
    else if (p.k >= 2)
      generic_sweep<kMax, kSplit>(q, sh, p, cnt, la, lb);
    else
      k1_sweep<kMax, kSplit>(q, sh, stage, p, cnt, la, lb);
    if (q.profile && threadIdx.x == 0) atomicMax(&S->t_sweep[p.it], globaltimer_ns());
    const unsigned long long n_out = count_barrier<kMax>(cnt, S, rec && t.stat_pending ? &t : nullptr);
    // every block has left the previous sweep's barrier: its counter is free
    // for the sweep after next
    if (rec) S->cnt[(sweep + 2) % 3] = 0;
    ++sweep;
    if (threadIdx.x == 0) {
      SweepPlan& nx = t.p[b ^ 1];
      commit_sweep<kMax>(qs, t, p, nx, n_out, rec);
      if (!nx.stop) {
        if (q.sweep_budget > 0 && sweep >= (unsigned)q.sweep_budget)
          nx.stop = 4;  // paused: the stack is saved below, the next mode-1 launch continues
        else
          plan_sweep<kMax>(qs, t, nx, rec);
      }
      if (rec && q.profile) S->t_plan[p.it + 1] = globaltimer_ns();
    }
    __syncthreads();
    b ^= 1;
  }
  if (rec) {
    const int stop = t.p[b].stop;
    if (t.stat_pending) write_stat<kMax>(S, t);
    S->sp = t.sp;
    for (int i = 0; i < t.sp; ++i) S->lv[i] = t.lv[i];
    for (int i = 0; i < t.iter; ++i) {
      S->tot_cand[i] = t.tot_cand[i];
      S->tot_in[i] = t.tot_in[i];
      S->tot_out[i] = t.tot_out[i];
    }
    S->lo_top = t.lo;
    S->hi_bot = t.hi;
    S->chunked = t.chunked;
    S->iter = t.iter;
    if (stop == 2) {
      S->leaf_off = t.leaf_off;
      S->n_leaf = t.leaf_n;
      S->leaf_end = t.leaf_end;
    }
    S->pending = stop == 2 && t.sp > 0;
    S->paused = stop == 4;
    // the triangle-pair candidates of this round's narrow phase use the gap
    S->cand_off = t.lo;
    S->cand_cap = t.hi - t.lo;
    if (q.mode == 0 || q.round == 0) S->rounds = q.round + 1;
    unsigned long long skipped = 0;
    if (kSplit)
      for (int i = 0; i < t.iter; ++i) skipped += V->skip_it[i];
    S->ncand_total = t.ncand_total;
    S->expanded = t.ncand_total - skipped;  // candidates of the pairs this call owns
    if (q.profile) S->t_edge[2] = globaltimer_ns();
  }
}


__global__ __launch_bounds__(kExpandThreads, 1024 / kExpandThreads) void k_traverse_min(QArgs q) {
  traverse_round<false, false>(q);
}
__global__ __launch_bounds__(kExpandThreads, 1024 / kExpandThreads) void k_traverse_max(QArgs q) {
  traverse_round<true, false>(q);
}
__global__ __launch_bounds__(kExpandThreads, 1024 / kExpandThreads) void k_traverse_min_split(QArgs q) {
  traverse_round<false, true>(q);
}
__global__ __launch_bounds__(kExpandThreads, 1024 / kExpandThreads) void k_traverse_max_split(QArgs q) {
  traverse_round<true, true>(q);
}

}  // namespace gd
