// primitives.cuh -- the build's data-parallel building blocks, written for
// this repo (no library sort or scan on the path): a stable LSD radix sort of
// (key, int32 value) pairs and a three-phase device scan over functors.
//
// Radix sort, one 8-bit digit per pass, three kernels per pass:
//   k_rs_hist     per tile of 4096 keys, the digit histogram (warp-aggregated
//                 shared-memory counts), stored digit-major: hist[d * G + b]
//   (scan)        exclusive scan of the 256 x G counts (device_scan below):
//                 the global offset of digit d in tile b
//   k_rs_scatter  the tile again, 16 rounds of 256 keys in input order; a
//                 key's rank among equal digits = earlier rounds + earlier
//                 warps + earlier lanes (__match_any_sync), so the pass is
//                 stable and the sort is an LSD radix sort
// Scan: k_scan_reduce (tile aggregates), k_scan_tiles (one block scans the
// aggregates), k_scan_apply (block scan of each tile seeded with its prefix).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace gd {

constexpr int kRsThreads = 256;
constexpr int kRsRounds = 16;
constexpr int kRsTile = kRsThreads * kRsRounds;  // keys per tile
constexpr int kRsWarps = kRsThreads / 32;

template <typename K>
__device__ __forceinline__ unsigned rs_digit(K k, int shift) {
  return (unsigned)(k >> shift) & 0xFFu;
}

template <typename K>
__global__ __launch_bounds__(kRsThreads) void k_rs_hist(const K* __restrict__ keys, long long n, int shift,
                                                        unsigned* __restrict__ hist, unsigned tiles) {
  __shared__ unsigned cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kRsTile;
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int r = 0; r < kRsRounds; ++r) {
    const long long i = base + r * kRsThreads + threadIdx.x;
    const bool v = i < n;
    const unsigned d = v ? rs_digit(keys[i], shift) : 256u + lane;  // invalid lanes match nobody
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (v && (peers & ((1u << lane) - 1)) == 0) atomicAdd(&cnt[d], (unsigned)__popc(peers));
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * tiles + blockIdx.x] = cnt[threadIdx.x];
}

template <typename K>
__global__ __launch_bounds__(kRsThreads) void k_rs_scatter(const K* __restrict__ kin, const int32_t* __restrict__ vin,
                                                           K* __restrict__ kout, int32_t* __restrict__ vout,
                                                           long long n, int shift, const unsigned* __restrict__ hist,
                                                           unsigned tiles) {
  __shared__ unsigned offs[256], run[256];
  __shared__ unsigned wcnt[kRsWarps][256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  offs[threadIdx.x] = hist[(size_t)threadIdx.x * tiles + blockIdx.x];
  run[threadIdx.x] = 0;
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) wcnt[w][threadIdx.x] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * kRsTile;
  for (int r = 0; r < kRsRounds; ++r) {
    const long long i = base + r * kRsThreads + threadIdx.x;
    if (base + r * kRsThreads >= n) break;  // uniform over the block
    const bool v = i < n;
    K k = 0;
    int32_t val = 0;
    if (v) {
      k = kin[i];
      val = vin[i];
    }
    const unsigned d = v ? rs_digit(k, shift) : 256u + lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned before = __popc(peers & ((1u << lane) - 1));
    if (v && before == 0) wcnt[wid][d] = (unsigned)__popc(peers);
    __syncthreads();
    if (v) {
      unsigned pos = offs[d] + run[d] + before;
      for (int w = 0; w < wid; ++w) pos += wcnt[w][d];
      kout[pos] = k;
      vout[pos] = val;
    }
    __syncthreads();
    unsigned add = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      add += wcnt[w][threadIdx.x];
      wcnt[w][threadIdx.x] = 0;
    }
    run[threadIdx.x] += add;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// device scan over functors: in(i) -> T, out(i, inclusive prefix)
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T, typename Op>
__device__ __forceinline__ T warp_inclusive(T v, Op op) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = op(v, y);
  }
  return v;
}

// inclusive block scan of one value per thread (blockDim.x == kScanThreads
// or 1024); returns the block aggregate in `total`
template <typename T, typename Op>
__device__ __forceinline__ T block_inclusive(T v, Op op, T ident, T* warp_tot, T& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = warp_inclusive(v, op);
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T t = lane < nw ? warp_tot[lane] : ident;
    t = warp_inclusive(t, op);
    if (lane < nw) warp_tot[lane] = t;
  }
  __syncthreads();
  if (wid > 0) x = op(warp_tot[wid - 1], x);
  total = warp_tot[nw - 1];
  __syncthreads();
  return x;
}

template <typename T, typename Op, typename In>
__global__ __launch_bounds__(kScanThreads) void k_scan_reduce(In in, long long n, Op op, T ident, T* aggr) {
  __shared__ T wt[32];
  const long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  T acc = ident;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j)
    if (base + j < n) acc = op(acc, in(base + j));
  T total;
  block_inclusive(acc, op, ident, wt, total);
  if (threadIdx.x == 0) aggr[blockIdx.x] = total;
}

// exclusive scan of the tile aggregates in place (one block of 1024)
template <typename T, typename Op>
__global__ __launch_bounds__(1024) void k_scan_tiles(T* aggr, long long tiles, Op op, T ident) {
  __shared__ T wt[32];
  T carry = ident;
  for (long long b0 = 0; b0 < tiles; b0 += 1024) {
    const long long i = b0 + threadIdx.x;
    const T v = i < tiles ? aggr[i] : ident;
    T total;
    const T inc = block_inclusive(v, op, ident, wt, total);
    // exclusive = carry op (inclusive without v): shift by one lane
    T exc = __shfl_up_sync(0xffffffffu, inc, 1);
    if ((threadIdx.x & 31) == 0) exc = threadIdx.x == 0 ? ident : wt[(threadIdx.x >> 5) - 1];
    if (i < tiles) aggr[i] = op(carry, exc);
    carry = op(carry, total);
    __syncthreads();
  }
}

template <typename T, typename Op, typename In, typename Out>
__global__ __launch_bounds__(kScanThreads) void k_scan_apply(In in, Out out, long long n, Op op, T ident,
                                                             const T* aggr) {
  __shared__ T wt[32];
  const long long base = (long long)blockIdx.x * kScanTile + (long long)threadIdx.x * kScanItems;
  T v[kScanItems];
  T acc = ident;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = base + j < n ? in(base + j) : ident;
    acc = op(acc, v[j]);
  }
  T total;
  T inc = block_inclusive(acc, op, ident, wt, total);
  // this thread's exclusive prefix within the tile
  T exc = __shfl_up_sync(0xffffffffu, inc, 1);
  if ((threadIdx.x & 31) == 0) exc = threadIdx.x == 0 ? ident : wt[(threadIdx.x >> 5) - 1];
  // (wt holds the inclusive prefix of the warp totals until the next call)
  T run = op(aggr[blockIdx.x], exc);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    run = op(run, v[j]);
    if (base + j < n) out(base + j, run, v[j]);  // inclusive prefix and the element (exclusive = run - v for sums)
  }
}

// inclusive scan of in(0 .. n-1) with `op`: out(i, prefix_i, in(i)); aggr:
// device scratch of scan_tiles(n) elements of T
inline long long scan_tiles(long long n) { return (n + kScanTile - 1) / kScanTile; }

template <typename T, typename Op, typename In, typename Out>
void device_scan(In in, Out out, long long n, Op op, T ident, T* aggr, cudaStream_t s) {
  if (n <= 0) return;
  const long long tiles = scan_tiles(n);
  k_scan_reduce<T, Op, In><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, op, ident, aggr);
  k_scan_tiles<T, Op><<<1, 1024, 0, s>>>(aggr, tiles, op, ident);
  k_scan_apply<T, Op, In, Out><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, out, n, op, ident, aggr);
  GD_CUDA(cudaGetLastError());
}

struct OpAdd {
  template <typename T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct OpMax {
  template <typename T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};
struct OpMin {
  template <typename T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a < b ? a : b; }
};

// host side of the radix sort (sort.cu): stable sort of (keys, vals) by the
// key bits [0, bits); the result is in *_out; *_in are clobbered
size_t radix_sort_ws_bytes(long long n);
void radix_sort_pairs(const unsigned long long* k_in, const int32_t* v_in, unsigned long long* k_tmp, int32_t* v_tmp,
                      unsigned long long* k_out,
                      int32_t* v_out, long long n, int bits, void* ws, cudaStream_t s);
void radix_sort_pairs(const uint32_t* k_in, const int32_t* v_in, uint32_t* k_tmp, int32_t* v_tmp, uint32_t* k_out,
                      int32_t* v_out, long long n, int bits, void* ws, cudaStream_t s);

}  // namespace gd
