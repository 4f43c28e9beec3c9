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
#ifndef GD_K1_ROUNDS
#define GD_K1_ROUNDS 4
#endif
constexpr int kK1Rounds = GD_K1_ROUNDS;                            // entries / thread / tile (k == 1)
constexpr int kK1Tile = kExpandThreads * kK1Rounds;
constexpr int kK1Stage = kK1Tile * 4;                              // staged survivors (<= 4 / entry)
// device schedule default (GdConfig.schedule == 0): fronts up to this many
// entries take k = 2 sweeps where the reference rule gives k = 1
#ifndef GD_K2_FRONT
#define GD_K2_FRONT (1u << 17)
#endif
constexpr unsigned long long kK2Front = GD_K2_FRONT;
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
// The remote atomics are sent only when the bound improves on `snap_sq`
// (the caller's tile snapshot of the cell, squared): once the bounds have
// converged, tiles send nothing over the links.
template <bool kMax>
__device__ __forceinline__ void commit_bound(const QArgs& q, float v, float snap_sq = kMax ? -1.f : INFINITY) {
  QState* S = q.S;
  commit_bound<kMax>(S, v);
  if (q.cfg.n_peers > 0) {
    const float nb = fmaxf(kMax ? v - S->slack : v + S->slack, 0.f);
    if (kMax ? !(nb * nb > snap_sq) : !(nb * nb < snap_sq)) return;
    const unsigned bits = __float_as_uint(nb);
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


// The persistent traversal kernels (traverse.cu, its own compilation unit:
// built with -maxrregcount=64 so its out-of-line sweeps share the kernel's
// 64-register budget of 2 blocks x 512 threads per SM): min / max query,
// single GPU / split query (ownership tests).
__global__ void k_traverse_min(QArgs q);
__global__ void k_traverse_max(QArgs q);
__global__ void k_traverse_min_split(QArgs q);
__global__ void k_traverse_max_split(QArgs q);

}  // namespace gd
