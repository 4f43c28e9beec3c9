// refit.cu -- per-frame refit (bvh.py:242-306) fused with apply_transform
// (mesh.py:102-105).
//
//   k_stage        float64 base vertex -> float32 float4 at its staged slot
//                  (first-use order, bvh_layout), once per base buffer
//   k_leaf_vtx     per-leaf distinct vertex sets (also once per base buffer)
//   k_refit        ONE launch per refit: one thread per leaf, its vertex set
//                  streamed from three coalesced float4 planes, float32
//                  transform, leaf box; each block folds its 256-leaf subtree
//                  8 levels up (warp shuffles, staged coalesced stores); the
//                  last-arriving block of every 256 sibling subtrees folds
//                  their roots further (arrival counters), up to the root
// Every node box is written exactly once; only the 1/256 subtree roots are
// re-read (from L2) by the cascade.
#include <algorithm>
#include <vector>

#include "engine.cuh"

namespace gd {

constexpr int kFold = 256;  // nodes per block per fold (8 levels)
// gdist.h sizes the cascade counters in leaf_x for 256-leaf blocks (2 (L >> 16) + 4)
static_assert(kFold == 256, "leaf_x cascade counter capacity assumes 256-leaf blocks");

// also records max |coordinate| of the staged vertices (stage_mag_slot, the
// scale of the float32 transform's rounding; NaN coordinates are ignored)
__global__ __launch_bounds__(256) void k_stage(GdMesh m, const int32_t* __restrict__ vmap, float4* __restrict__ out,
                                               unsigned* __restrict__ mag) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  float a = 0.f;
  if (i < m.nv) {
    const double* p = m.vtx + 3 * i;
    const float4 v = make_float4((float)p[0], (float)p[1], (float)p[2], 0.f);
    out[vmap[i]] = v;
    a = fmaxf(fabsf(v.x), fmaxf(fabsf(v.y), fabsf(v.z)));
  }
  a = warp_max(a);
  if ((threadIdx.x & 31) == 0 && a > 0.f) atomicMax(mag, __float_as_uint(a));
}

// union of this lane's box with the one `o` lanes up (mask: the block's lanes
// when it is narrower than a warp; lanes whose source is outside never use it)
__device__ __forceinline__ Box shfl_union(const Box& b, int o, unsigned mask) {
  Box r;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = fmin_nan(b.lo[k], __shfl_down_sync(mask, b.lo[k], o));
    r.hi[k] = fmax_nan(b.hi[k], __shfl_down_sync(mask, b.hi[k], o));
  }
  return r;
}

// The first nb (= 2^B <= blockDim.x) threads hold the boxes of nodes
// [rank0, rank0 + nb) of level lv, one each.  Fold B levels up: warp
// shuffles for the first five, the warp roots in warp 0 for the rest.  Level
// u's nb >> u boxes are staged at sl[nb - (nb >> (u - 1)) ...]; one flat loop
// then writes every staged box (three float2 each, consecutive threads ->
// consecutive words of a level run).  All threads of the block must call it;
// thread 0 returns the folded root.
__device__ __forceinline__ Box fold_group(float* box, Box* sl, Box mine, int lv, unsigned rank0, int B) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nb = 1 << B;
  if (threadIdx.x < nb) {
    const unsigned mask = nb >= 32 ? 0xffffffffu : (1u << nb) - 1;
    const int wl = min(B, 5);
    for (int u = 1; u <= wl; ++u) {
      mine = shfl_union(mine, 1 << (u - 1), mask);
      if ((lane & ((1 << u) - 1)) == 0) sl[nb - (nb >> (u - 1)) + (threadIdx.x >> u)] = mine;
    }
  }
  if (B > 5) {
    __syncthreads();
    if (wid == 0) {
      const int nw = nb >> 5;
      mine = sl[nb - (nb >> 4) + (lane < nw ? lane : 0)];  // level-5 warp roots
      for (int u = 6; u <= B; ++u) {
        mine = shfl_union(mine, 1 << (u - 6), 0xffffffffu);
        if (lane < nw && (lane & ((1 << (u - 5)) - 1)) == 0) sl[nb - (nb >> (u - 1)) + (lane >> (u - 5))] = mine;
      }
    }
  }
  __syncthreads();
  const float2* s2 = reinterpret_cast<const float2*>(sl);
  float2* d2 = reinterpret_cast<float2*>(box);
  for (int j = threadIdx.x; j < 3 * (nb - 1); j += blockDim.x) {
    const int t = j / 3, c = j - 3 * t;
    const int u = B - (31 - __clz(nb - 1 - t));           // level of staged box t
    const int i = t - (nb - (nb >> (u - 1)));              // index inside level u
    const unsigned long long slot = (1ull << (lv - u)) + (rank0 >> u) + i;  // node (2^(lv-u) - 1) + r
    d2[slot * 3 + c] = s2[j];
  }
  return mine;  // thread 0: the root of the folded subtree
}

// box written earlier in the same launch by another block: L2 load (.cg)
__device__ __forceinline__ Box load_box_cg(const float* box, unsigned long long node) {
  const float2* p = reinterpret_cast<const float2*>(box + (node + 1) * 6);
  const float2 a = __ldcg(p), b = __ldcg(p + 1), c = __ldcg(p + 2);
  Box r;
  r.lo[0] = a.x; r.lo[1] = a.y; r.lo[2] = b.x;
  r.hi[0] = b.y; r.hi[1] = c.x; r.hi[2] = c.y;
  return r;
}

__device__ __forceinline__ void grow(Box& b, const V3<float>& p) {
  b.lo[0] = fmin_nan(b.lo[0], p.x);
  b.lo[1] = fmin_nan(b.lo[1], p.y);
  b.lo[2] = fmin_nan(b.lo[2], p.z);
  b.hi[0] = fmax_nan(b.hi[0], p.x);
  b.hi[1] = fmax_nan(b.hi[1], p.y);
  b.hi[2] = fmax_nan(b.hi[2], p.z);
}

// One launch refits the whole tree.  Each block: leaf boxes from the streamed
// per-leaf vertex sets (three coalesced float4 planes; extras only for the
// rare leaves with 5-6 distinct vertices), a coalesced leaf-box store, the
// fold of its 256-leaf subtree.  Then a cascade: the last block of every
// group of 256 (or fewer, at the top) sibling subtrees -- detected with a
// per-group arrival counter -- folds their roots 8 levels further, until the
// root.  The counters live at the end of leaf_x and are left zero.  The
// vertices are the staged ones, so every box contains exactly the float32
// vertices the narrow phase tests.
__global__ __launch_bounds__(kFold) void k_refit(GdBvh T, XfF32 x) {
  __shared__ __align__(16) Box sb[kFold], sl[kFold];
  __shared__ bool last;
  const unsigned L = (unsigned)T.leaf_count, W = (L + 31) >> 5;
  const unsigned l = blockIdx.x * blockDim.x + threadIdx.x;  // leaf rank (< L exactly)
  const float4* p = reinterpret_cast<const float4*>(T.leaf_vtx);
  const float4 a = __ldg(p + l), b4 = __ldg(p + L + l), c = __ldg(p + 2 * L + l);
  Box b;
  const V3<float> v0 = xf_apply(x, make_float4(a.x, a.y, a.z, 0.f));
  b.lo[0] = b.hi[0] = v0.x;
  b.lo[1] = b.hi[1] = v0.y;
  b.lo[2] = b.hi[2] = v0.z;
  grow(b, xf_apply(x, make_float4(a.w, b4.x, b4.y, 0.f)));
  grow(b, xf_apply(x, make_float4(b4.z, b4.w, c.x, 0.f)));
  grow(b, xf_apply(x, make_float4(c.y, c.z, c.w, 0.f)));
  const unsigned mask = __ldg(T.leaf_x + (l >> 5));
  const int lane = threadIdx.x & 31;
  if ((mask >> lane) & 1u) {
    const unsigned rank = __ldg(T.leaf_x + W + (l >> 5)) + __popc(mask & ((1u << lane) - 1));
    const float4* xv = reinterpret_cast<const float4*>(T.leaf_xvtx);
    grow(b, xf_apply(x, __ldg(xv + 2 * rank)));
    grow(b, xf_apply(x, __ldg(xv + 2 * rank + 1)));
  }
  // leaf boxes: coalesced float4 copy from shared memory (leaf slots L + l
  // start 16-byte aligned for every block of >= 2 leaves)
  sb[threadIdx.x] = b;
  __syncthreads();
  const unsigned rank0 = blockIdx.x * blockDim.x;
  {
    const int nb = blockDim.x;
    if (nb >= 2) {
      const float4* s4 = reinterpret_cast<const float4*>(sb);
      float4* d4 = reinterpret_cast<float4*>(T.box + ((unsigned long long)L + rank0) * 6);
      for (int i = threadIdx.x; i < nb * 3 / 2; i += nb) d4[i] = s4[i];
    } else {
      store_box(T.box, (unsigned long long)(L - 1) + rank0, b);
    }
  }
  int lv = T.depth;
  const int B = 31 - __clz(blockDim.x);
  if (B > 0) b = fold_group(T.box, sl, b, lv, rank0, B);
  lv -= B;
  unsigned rank = blockIdx.x;  // this block's subtree root: node rank at level lv
  unsigned* cnt = T.leaf_x + 2 * W + 1;
  while (lv > 0) {
    // group of sibling subtree roots folded by its last-arriving block
    const int g = min(lv, 8);
    const unsigned gsize = 1u << g, group = rank >> g, ngroups = (1u << lv) >> g;
    if (threadIdx.x == 0) {
      // the only box another block reads: this subtree's root, published by
      // thread 0 itself before its arrival
      store_box(T.box, ((1ull << lv) - 1) + rank, b);
      __threadfence();
      last = atomicAdd(cnt + ngroups + group, 1u) == gsize - 1;
      if (last) cnt[ngroups + group] = 0;  // ready for the next refit
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    Box mine = b;
    if (threadIdx.x < gsize)
      mine = load_box_cg(T.box, ((1ull << lv) - 1) + ((unsigned long long)group << g) + threadIdx.x);
    b = fold_group(T.box, sl, mine, lv, group << g, g);  // the first gsize threads fold g levels
    lv -= g;
    rank = group;
  }
}

// k_refit for full 256-leaf blocks (every tree of >= 256 leaves): the same
// boxes as k_refit.  128 threads, two adjacent leaves each: the thread's six
// plane loads are in flight together, it unions its two leaf boxes into
// their parent in registers, and levels 2 - 6 fold inside each warp with
// shuffles -- no block barrier until the four warp roots meet in warp 0 for
// the last two levels; warp 0 alone then publishes the subtree root and, in
// the last-arriving block of a group, folds the group (the other warps have
// exited: they do not wait on the arrival counter).  Leaf pairs go to global memory as three 16-byte
// stores (sibling slots are 16-byte aligned); every internal node is stored
// by the lane holding it, consecutive nodes of a level from consecutive
// holders.  (ncu: the 256-thread version was bound by its per-level block
// barriers and one load round trip per thread, profiles/r2*_refit.)
__device__ __forceinline__ Box leaf_box(const XfF32& x, const float4 a, const float4 b4, const float4 c) {
  Box b;
  const V3<float> v0 = xf_apply(x, make_float4(a.x, a.y, a.z, 0.f));
  b.lo[0] = b.hi[0] = v0.x;
  b.lo[1] = b.hi[1] = v0.y;
  b.lo[2] = b.hi[2] = v0.z;
  grow(b, xf_apply(x, make_float4(a.w, b4.x, b4.y, 0.f)));
  grow(b, xf_apply(x, make_float4(b4.z, b4.w, c.x, 0.f)));
  grow(b, xf_apply(x, make_float4(c.y, c.z, c.w, 0.f)));
  return b;
}

__global__ __launch_bounds__(128, 10) void k_refit256(GdBvh T, XfF32 x) {
  constexpr int NB = kFold;  // leaves per block
  __shared__ Box wroot[4];
  __shared__ __align__(16) Box stage[kFold + kFold / 2];  // the cascade's ping-pong levels
  const unsigned L = (unsigned)T.leaf_count, W = (L + 31) >> 5;
  const unsigned rank0 = blockIdx.x * NB;
  const unsigned l0 = rank0 + 2 * threadIdx.x;  // this thread's leaves l0, l0 + 1
  const float4* p = reinterpret_cast<const float4*>(T.leaf_vtx);
  const float4 a0 = __ldg(p + l0), a1 = __ldg(p + l0 + 1);
  const float4 b0 = __ldg(p + L + l0), b1 = __ldg(p + L + l0 + 1);
  const float4 c0 = __ldg(p + 2 * L + l0), c1 = __ldg(p + 2 * L + l0 + 1);
  // the extras mask and rank base of the leaves' 32-leaf word, loaded with
  // the planes: a leaf with extras waits one more round trip, not two
  const unsigned mask = __ldg(T.leaf_x + (l0 >> 5)), rank_base = __ldg(T.leaf_x + W + (l0 >> 5));
  // leaves with 5 - 6 distinct vertices (~20 % on the rings): both leaves'
  // extra vertices are requested together, one round trip for the pair
  const unsigned bit = l0 & 31;
  const bool xe = (mask >> bit) & 1u, xo = (mask >> (bit + 1)) & 1u;
  const unsigned re = rank_base + __popc(mask & ((1u << bit) - 1));
  const float4* xv = reinterpret_cast<const float4*>(T.leaf_xvtx);
  float4 ex0, ex1, ox0, ox1;
  if (xe) {
    ex0 = __ldg(xv + 2 * re);
    ex1 = __ldg(xv + 2 * re + 1);
  }
  if (xo) {
    const unsigned ro = re + (xe ? 1u : 0u);
    ox0 = __ldg(xv + 2 * ro);
    ox1 = __ldg(xv + 2 * ro + 1);
  }
  Box e = leaf_box(x, a0, b0, c0);
  Box o = leaf_box(x, a1, b1, c1);
  if (xe) {
    grow(e, xf_apply(x, ex0));
    grow(e, xf_apply(x, ex1));
  }
  if (xo) {
    grow(o, xf_apply(x, ox0));
    grow(o, xf_apply(x, ox1));
  }
  {  // the sibling leaf pair: slots L + l0, L + l0 + 1 (48 bytes, 16-byte aligned)
    float4* d = reinterpret_cast<float4*>(T.box + ((unsigned long long)L + l0) * 6);
    d[0] = make_float4(e.lo[0], e.lo[1], e.lo[2], e.hi[0]);
    d[1] = make_float4(e.hi[1], e.hi[2], o.lo[0], o.lo[1]);
    d[2] = make_float4(o.lo[2], o.hi[0], o.hi[1], o.hi[2]);
  }
  Box b = box_union(e, o);
  int lv = T.depth;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // level 1 (the leaf pairs' parents): node rank (rank0 >> 1) + threadIdx.x
  store_box(T.box, ((1ull << (lv - 1)) - 1) + (rank0 >> 1) + threadIdx.x, b);
  // levels 2 - 6 inside the warp: after step u the lanes with lane % 2^(u-1)
  // == 0 hold the level-u nodes of the warp's 64 leaves
#pragma unroll
  for (int u = 2; u <= 6; ++u) {
    b = shfl_union(b, 1 << (u - 2), 0xffffffffu);
    if ((lane & ((1 << (u - 1)) - 1)) == 0)
      store_box(T.box, ((1ull << (lv - u)) - 1) + (rank0 >> u) + (threadIdx.x >> (u - 1)), b);
  }
  if (lane == 0) wroot[wid] = b;
  __syncthreads();
  if (wid != 0) return;  // warp 0 alone finishes the block: its top levels and the cascade
  // levels 7, 8: the four warp roots (lanes 0 - 3)
  b = wroot[lane & 3];
#pragma unroll
  for (int u = 7; u <= 8; ++u) {
    b = shfl_union(b, 1 << (u - 7), 0xffffffffu);
    if (lane < 4 && (lane & ((1 << (u - 6)) - 1)) == 0)
      store_box(T.box, ((1ull << (lv - u)) - 1) + (rank0 >> u) + (lane >> (u - 6)), b);
  }
  lv -= 8;
  unsigned rank = blockIdx.x;  // this block's subtree root (lane 0): node rank at level lv
  unsigned* cnt = T.leaf_x + 2 * W + 1;
  while (lv > 0) {
    // group of sibling subtree roots folded by its last-arriving block (as in k_refit)
    const int g = min(lv, 8);
    const unsigned gsize = 1u << g, group = rank >> g, ngroups = (1u << lv) >> g;
    int is_last = 0;
    if (lane == 0) {
      // the only box another block reads: the subtree root, stored by lane 0
      // itself, then released by its arrival (acq_rel: the last arrival also
      // acquires every earlier block's root -- the RMWs on the counter form
      // a release sequence); no full fence
      store_box(T.box, ((1ull << lv) - 1) + rank, b);
      unsigned old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt + ngroups + group) : "memory");
      is_last = old == gsize - 1;
      if (is_last) cnt[ngroups + group] = 0;  // ready for the next refit
    }
    if (!__shfl_sync(0xffffffffu, is_last, 0)) return;
    // the other lanes read the roots too: order their loads after lane 0's acquire
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    // the warp folds the group's roots level by level through shared memory
    // (ping-pong buffers), each node stored by the lane that computes it
    Box* src = stage;
    Box* dst = stage + kFold;
    for (unsigned i = lane; i < gsize; i += 32)
      src[i] = load_box_cg(T.box, ((1ull << lv) - 1) + ((unsigned long long)group << g) + i);
    __syncwarp();
    for (int k = 1; k <= g; ++k) {
      const unsigned n = gsize >> k;
      for (unsigned i = lane; i < n; i += 32) {
        const Box r = box_union(src[2 * i], src[2 * i + 1]);
        dst[i] = r;
        store_box(T.box, ((1ull << (lv - k)) - 1) + ((unsigned long long)group << (g - k)) + i, r);
      }
      __syncwarp();
      Box* t = src;
      src = dst;
      dst = t;
    }
    b = src[0];
    lv -= g;
    rank = group;
  }
}

// per-leaf distinct vertex sets (gdist.h leaf_vtx / leaf_x / leaf_xvtx) from
// the leaf records and the staged vertices
__global__ __launch_bounds__(256) void k_leaf_vtx(GdBvh T) {
  const long long l = blockIdx.x * 256ll + threadIdx.x;
  const long long L = T.leaf_count, W = (L + 31) >> 5;
  const int lane = threadIdx.x & 31;
  int u[6];
  int k = 0;
  if (l < L) {
    const LeafRec r = load_leaf(T, l);
    const int s[6] = {r.r0.x, r.r0.y, r.r0.z, r.r0.w, r.r1.x, r.r1.y};
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      bool seen = false;
#pragma unroll
      for (int j = 0; j < i; ++j) seen = seen || (s[j] == s[i]);
      if (!seen) u[k++] = s[i];
    }
    for (int i = k; i < 6; ++i) u[i] = u[0];
    const float4* v = reinterpret_cast<const float4*>(T.vtx32);
    const float4 a = v[u[0]], b = v[u[1]], c = v[u[2]], d = v[u[3]];
    float4* p = reinterpret_cast<float4*>(T.leaf_vtx);
    p[l] = make_float4(a.x, a.y, a.z, b.x);
    p[L + l] = make_float4(b.y, b.z, c.x, c.y);
    p[2 * L + l] = make_float4(c.z, d.x, d.y, d.z);
  }
  const bool extra = k > 4;
  const unsigned mask = __ballot_sync(0xffffffffu, extra);
  unsigned base = 0;
  if (lane == 0) {
    base = mask ? atomicAdd(&T.leaf_x[2 * W], (unsigned)__popc(mask)) : 0u;
    if (l < L) {
      T.leaf_x[l >> 5] = mask;
      T.leaf_x[W + (l >> 5)] = base;
    }
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (extra) {
    const unsigned rank = base + __popc(mask & ((1u << lane) - 1));
    const float4* v = reinterpret_cast<const float4*>(T.vtx32);
    float4* x = reinterpret_cast<float4*>(T.leaf_xvtx);
    x[2 * rank] = v[u[4]];
    x[2 * rank + 1] = v[u[5]];
  }
}

// both triangles of every leaf as five float4 (gdist.h leaf_tri): the staged
// base vertices a0 a1 a2 b0 b1 b2, then tri0 / tri1 as float bits
__global__ __launch_bounds__(256) void k_leaf_tri(GdBvh T) {
  const long long l = blockIdx.x * 256ll + threadIdx.x;
  if (l >= T.leaf_count) return;
  const LeafRec r = load_leaf(T, l);
  const float4* v = reinterpret_cast<const float4*>(T.vtx32);
  const float4 a0 = v[r.r0.x], a1 = v[r.r0.y], a2 = v[r.r0.z], b0 = v[r.r0.w], b1 = v[r.r1.x], b2 = v[r.r1.y];
  float4* o = reinterpret_cast<float4*>(T.leaf_tri) + 5 * l;
  o[0] = make_float4(a0.x, a0.y, a0.z, a1.x);
  o[1] = make_float4(a1.y, a1.z, a2.x, a2.y);
  o[2] = make_float4(a2.z, b0.x, b0.y, b0.z);
  o[3] = make_float4(b1.x, b1.y, b1.z, b2.x);
  o[4] = make_float4(b2.y, b2.z, __int_as_float(r.r1.z), __int_as_float(r.r1.w));
}

void stage_vertices(const GdMesh& m, const GdBvh& T, cudaStream_t s) {
  GD_CHECK(m.nv == T.nv, GD_ERR_TOPOLOGY, "mesh vertex count differs from the tree's");
  GD_CHECK(T.leaf_vtx && T.leaf_x && T.leaf_xvtx && T.leaf_tri, GD_ERR_INVALID,
           "GdBvh leaf vertex sets must be allocated");
  const long long W = (T.leaf_count + 31) / 32;
  // extras counter + the refit's cascade counters + the staging magnitude
  // (gdist.h leaf_x)
  GD_CUDA(cudaMemsetAsync(T.leaf_x + 2 * W, 0, (1 + 2 * (T.leaf_count >> 16) + 4 + 1) * sizeof(uint32_t), s));
  if (m.nv > 0)
    k_stage<<<(unsigned)((m.nv + 255) / 256), 256, 0, s>>>(m, T.vmap, reinterpret_cast<float4*>(T.vtx32),
                                                           T.leaf_x + stage_mag_slot(T.leaf_count));
  k_leaf_vtx<<<(unsigned)((T.leaf_count + 255) / 256), 256, 0, s>>>(T);
  k_leaf_tri<<<(unsigned)((T.leaf_count + 255) / 256), 256, 0, s>>>(T);
  GD_CUDA(cudaGetLastError());
}

bool is_refit_kernel(const void* f) { return f == (const void*)k_refit || f == (const void*)k_refit256; }  // graph.cu

void refit(const GdMesh& m, const GdBvh& T, cudaStream_t s) {
  GD_CHECK(m.m == T.n_tris, GD_ERR_TOPOLOGY,
           "refit mesh has " + std::to_string(m.m) + " triangles, tree was built over " + std::to_string(T.n_tris));
  GD_CHECK(m.nv == T.nv, GD_ERR_TOPOLOGY, "refit mesh vertex count differs from the build");
  const long long L = T.leaf_count;
  GD_CHECK(L < (1ll << 31), GD_ERR_INVALID, "tree too large for 32-bit leaf ranks");
  const int bs = (int)std::min<long long>(L, kFold);
  if (bs == kFold)
    k_refit256<<<(unsigned)(L / bs), 128, 0, s>>>(T, xf32_host(m));
  else
    k_refit<<<(unsigned)(L / bs), bs, 0, s>>>(T, xf32_host(m));
  const long long launches = 1;
  GD_CUDA(cudaGetLastError());
  count_launches(launches);
}

// ---------------------------------------------------------------------------
// node boxes with the reference's dtype semantics (bvh.py:242-264): the
// float64 path reads the float64 vertices, the float32 path casts first.
template <typename T>
__global__ void k_export_leaf(GdMesh m, GdBvh B, T* nmin, T* nmax) {
  const long long l = blockIdx.x * 256ll + threadIdx.x;
  if (l >= B.leaf_count) return;
  const int4* rec = reinterpret_cast<const int4*>(B.leaf_rec) + 2 * l;
  const int4 r1 = rec[1];  // {b1, b2, tri0, tri1}: records hold staged slots, so use the triangle ids
  const int32_t* i0 = m.tri + 3 * (long long)r1.z;
  const int32_t* i1 = m.tri + 3 * (long long)(r1.w >= 0 ? r1.w : r1.z);
  const int v[6] = {i0[0], i0[1], i0[2], i1[0], i1[1], i1[2]};
  const int nvert = r1.w >= 0 ? 6 : 3;
  T lo[3], hi[3];
  for (int c = 0; c < nvert; ++c) {
    V3<double> p = mesh_vertex(m, v[c]);
    T x[3] = {T(p.x), T(p.y), T(p.z)};
    for (int k = 0; k < 3; ++k) {
      if (c == 0) {
        lo[k] = hi[k] = x[k];
      } else {
        lo[k] = (x[k] < lo[k] || x[k] != x[k]) ? x[k] : lo[k];  // np.min: NaN wins
        hi[k] = (x[k] > hi[k] || x[k] != x[k]) ? x[k] : hi[k];
      }
    }
  }
  const long long node = (B.leaf_count - 1) + l;
  for (int k = 0; k < 3; ++k) {
    nmin[3 * node + k] = lo[k];
    nmax[3 * node + k] = hi[k];
  }
}

template <typename T>
__global__ void k_export_level(T* nmin, T* nmax, int lv) {
  const long long r = blockIdx.x * 256ll + threadIdx.x;
  if (r >= (1ll << lv)) return;
  const long long node = ((1ll << lv) - 1) + r, c0 = 2 * node + 1, c1 = c0 + 1;
  for (int k = 0; k < 3; ++k) {
    const T a = nmin[3 * c0 + k], b = nmin[3 * c1 + k];
    nmin[3 * node + k] = (b < a || b != b) ? b : a;  // np.minimum (a NaN operand wins)
    const T c = nmax[3 * c0 + k], d = nmax[3 * c1 + k];
    nmax[3 * node + k] = (d > c || d != d) ? d : c;  // np.maximum
  }
}

void export_boxes(const GdMesh& m, const GdBvh& B, int precision, void* nmin, void* nmax, cudaStream_t s) {
  GD_CHECK(precision == 32 || precision == 64, GD_ERR_CONFIG, "precision must be 32 or 64");
  const unsigned g = (unsigned)((B.leaf_count + 255) / 256);
  if (precision == 64) {
    k_export_leaf<double><<<g, 256, 0, s>>>(m, B, (double*)nmin, (double*)nmax);
    for (int lv = B.depth - 1; lv >= 0; --lv)
      k_export_level<double><<<(unsigned)(((1ll << lv) + 255) / 256), 256, 0, s>>>((double*)nmin, (double*)nmax, lv);
  } else {
    k_export_leaf<float><<<g, 256, 0, s>>>(m, B, (float*)nmin, (float*)nmax);
    for (int lv = B.depth - 1; lv >= 0; --lv)
      k_export_level<float><<<(unsigned)(((1ll << lv) + 255) / 256), 256, 0, s>>>((float*)nmin, (float*)nmax, lv);
  }
  GD_CUDA(cudaGetLastError());
  GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gd
