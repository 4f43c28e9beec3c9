// build.cu -- f12-BVH construction (bvh.py:69-95, 98-181, 267-289).
//
//   k_bounds       float64 min/max over ALL vertices (bvh.py:82-83)
//   k_morton       centroid ((p0+p1)+p2)/3, 21-bit quantisation, 63-bit
//                  interleave, x at bit 0 (bvh.py:58-95)
//   radix sort     stable (code, id) sort == np.lexsort((ids, codes))
//   k_pair_sa      float64 surface area of Morton neighbours (bvh.py:117-120)
//   pair_greedy    exact greedy on the host (pairing.cpp)
//   k_leaf_rec     one 32-byte record per leaf (gdist.h)
//   bvh_layout     staged-vertex numbering by first use in leaf order
//                  (k_first_use + radix sort + k_rec_remap), staging
// then refit() fills every box.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "engine.cuh"

namespace gd {

void refit(const GdMesh& m, const GdBvh& T, cudaStream_t s);
void stage_vertices(const GdMesh& m, const GdBvh& T, cudaStream_t s);
void pair_greedy(const double* sa, int64_t n, uint8_t* is_left);

// order-preserving map of a double onto an unsigned 64-bit key
__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void k_bounds_init(unsigned long long* lohi) {
  if (threadIdx.x < 3) {
    lohi[threadIdx.x] = ~0ull;   // running min key
    lohi[3 + threadIdx.x] = 0ull;  // running max key
  }
}

__global__ __launch_bounds__(256) void k_bounds(GdMesh m, unsigned long long* lohi) {
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < m.nv; i += gridDim.x * 256ll) {
    V3<double> v = mesh_vertex(m, i);
    const double c[3] = {v.x, v.y, v.z};
    for (int k = 0; k < 3; ++k) {
      unsigned long long key = dkey(c[k]);
      lo[k] = min(lo[k], key);
      hi[k] = max(hi[k], key);
    }
  }
  for (int k = 0; k < 3; ++k) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(lohi + k, lo[k]);
      atomicMax(lohi + 3 + k, hi[k]);
    }
  }
}

__device__ __forceinline__ unsigned long long spread3(unsigned long long x) {
  x &= 0x1FFFFFull;
  x = (x | (x << 32)) & 0x1F00000000FFFFull;
  x = (x | (x << 16)) & 0x1F0000FF0000FFull;
  x = (x | (x << 8)) & 0x100F00F00F00F00Full;
  x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

__global__ __launch_bounds__(256) void k_morton(GdMesh m, const unsigned long long* lohi,
                                                unsigned long long* codes, int32_t* ids) {
  const long long t = blockIdx.x * 256ll + threadIdx.x;
  if (t >= m.m) return;
  using E = Exact<double>;
  const int32_t* ix = m.tri + 3 * t;
  V3<double> a = mesh_vertex(m, ix[0]), b = mesh_vertex(m, ix[1]), c = mesh_vertex(m, ix[2]);
  const double cen[3] = {E::div(E::add(E::add(a.x, b.x), c.x), 3.0), E::div(E::add(E::add(a.y, b.y), c.y), 3.0),
                         E::div(E::add(E::add(a.z, b.z), c.z), 3.0)};
  unsigned long long code = 0;
  for (int k = 0; k < 3; ++k) {
    const double lo = dkey_inv(lohi[k]), hi = dkey_inv(lohi[3 + k]);
    double span = E::sub(hi, lo);
    span = span > 0.0 ? span : 1.0;
    double f = E::div(E::sub(cen[k], lo), span);
    f = f > 0.0 ? f : 0.0;  // np.clip(., 0, None)
    unsigned long long q = (unsigned long long)E::mul(f, 2097152.0);
    q = q < 0x1FFFFFull ? q : 0x1FFFFFull;
    code |= spread3(q) << k;
  }
  codes[t] = code;
  ids[t] = (int32_t)t;
}

__device__ __forceinline__ void tri_box64(const GdMesh& m, int32_t t, double* lo, double* hi) {
  const int32_t* ix = m.tri + 3 * (long long)t;
  V3<double> a = mesh_vertex(m, ix[0]), b = mesh_vertex(m, ix[1]), c = mesh_vertex(m, ix[2]);
  const double xs[3][3] = {{a.x, b.x, c.x}, {a.y, b.y, c.y}, {a.z, b.z, c.z}};
  for (int k = 0; k < 3; ++k) {
    lo[k] = fmin(fmin(xs[k][0], xs[k][1]), xs[k][2]);
    hi[k] = fmax(fmax(xs[k][0], xs[k][1]), xs[k][2]);
  }
}

__global__ __launch_bounds__(256) void k_pair_sa(GdMesh m, const int32_t* order, long long n, double* sa) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= n - 1) return;
  using E = Exact<double>;
  double alo[3], ahi[3], blo[3], bhi[3], e[3];
  tri_box64(m, order[i], alo, ahi);
  tri_box64(m, order[i + 1], blo, bhi);
  for (int k = 0; k < 3; ++k) e[k] = E::sub(fmax(ahi[k], bhi[k]), fmin(alo[k], blo[k]));
  sa[i] = E::add(E::add(E::mul(e[0], e[1]), E::mul(e[1], e[2])), E::mul(e[2], e[0]));
}

// leaf records in Morton order (bvh.py:168-181): leaf l holds Morton ranks
// first[l] .. first[l + 1] - 1 (one or two triangles)
__global__ __launch_bounds__(256) void k_leaf_rec(GdMesh m, const int32_t* order, const uint32_t* first, long long L,
                                                  int4* rec) {
  const long long l = blockIdx.x * 256ll + threadIdx.x;
  if (l >= L) return;
  const uint32_t f = first[l], c = first[l + 1] - f;
  const int32_t t0 = order[f], t1 = c > 1 ? order[f + 1] : -1;
  const int32_t* i0 = m.tri + 3 * (long long)t0;
  const int32_t* i1 = m.tri + 3 * (long long)(t1 >= 0 ? t1 : t0);
  rec[2 * l] = make_int4(i0[0], i0[1], i0[2], i1[0]);
  rec[2 * l + 1] = make_int4(i1[1], i1[2], t0, t1);
}

// ---------------------------------------------------------------------------
// vertex layout: staged vertices are renumbered by first use in leaf-record
// order, so the leaves of one warp gather from a few contiguous lines
__global__ __launch_bounds__(256) void k_first_init(uint32_t* first, int32_t* ids, long long nv) {
  const long long v = blockIdx.x * 256ll + threadIdx.x;
  if (v >= nv) return;
  first[v] = 0xFFFFFFFFu;
  ids[v] = (int32_t)v;
}
__global__ __launch_bounds__(256) void k_first_use(const int32_t* rec, long long L, uint32_t* first) {
  const long long l = blockIdx.x * 256ll + threadIdx.x;
  if (l >= L) return;
#pragma unroll
  for (int c = 0; c < 6; ++c) atomicMin(first + rec[8 * l + c], (uint32_t)(6 * l + c));
}
__global__ __launch_bounds__(256) void k_vmap(const int32_t* sorted_ids, long long nv, int32_t* vmap) {
  const long long r = blockIdx.x * 256ll + threadIdx.x;
  if (r < nv) vmap[sorted_ids[r]] = (int32_t)r;
}
__global__ __launch_bounds__(256) void k_rec_remap(int32_t* rec, long long L, const int32_t* vmap) {
  const long long l = blockIdx.x * 256ll + threadIdx.x;
  if (l >= L) return;
#pragma unroll
  for (int c = 0; c < 6; ++c) rec[8 * l + c] = vmap[rec[8 * l + c]];
}

struct LayoutWs {
  size_t first, first_out, ids, ids_out, cub, cub_bytes, total;
};
static size_t al(size_t x) { return (x + 255) / 256 * 256; }
static LayoutWs layout_ws(int64_t nv) {
  LayoutWs w;
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(nv, 1), 0, 32);
  size_t o = 0;
  w.first = o;
  o = al(o + nv * sizeof(uint32_t));
  w.first_out = o;
  o = al(o + nv * sizeof(uint32_t));
  w.ids = o;
  o = al(o + nv * sizeof(int32_t));
  w.ids_out = o;
  o = al(o + nv * sizeof(int32_t));
  w.cub = o;
  w.cub_bytes = cub_bytes;
  o = al(o + cub_bytes);
  w.total = o;
  return w;
}

void bvh_layout(const GdMesh& mesh, GdBvh& T, void* ws, size_t ws_bytes, cudaStream_t s) {
  const int64_t nv = mesh.nv, L = T.leaf_count;
  GD_CHECK(nv == T.nv && nv < (1ll << 31) && T.vmap, GD_ERR_INVALID, "GdBvh does not match the mesh");
  LayoutWs w = layout_ws(nv);
  GD_CHECK(ws != nullptr && ws_bytes >= w.total, GD_ERR_WORKSPACE,
           "layout workspace too small: need " + std::to_string(w.total) + " bytes");
  char* base = static_cast<char*>(ws);
  auto* first = reinterpret_cast<uint32_t*>(base + w.first);
  auto* first_out = reinterpret_cast<uint32_t*>(base + w.first_out);
  auto* ids = reinterpret_cast<int32_t*>(base + w.ids);
  auto* ids_out = reinterpret_cast<int32_t*>(base + w.ids_out);
  const unsigned gv = (unsigned)((nv + 255) / 256), gl = (unsigned)((L + 255) / 256);
  if (nv > 0) {
    k_first_init<<<gv, 256, 0, s>>>(first, ids, nv);
    k_first_use<<<gl, 256, 0, s>>>(T.leaf_rec, L, first);
    size_t cub_bytes = w.cub_bytes;
    GD_CUDA(cub::DeviceRadixSort::SortPairs(base + w.cub, cub_bytes, first, first_out, ids, ids_out, (int)nv, 0, 32,
                                            s));
    k_vmap<<<gv, 256, 0, s>>>(ids_out, nv, T.vmap);
    k_rec_remap<<<gl, 256, 0, s>>>(T.leaf_rec, L, T.vmap);
  }
  GD_CUDA(cudaGetLastError());
  stage_vertices(mesh, T, s);
}

size_t layout_workspace_size(int64_t nv) { return layout_ws(nv).total; }

struct BuildWs {
  size_t lohi, codes_in, codes_out, ids_in, ids_out, sa, first, cub, total, cub_bytes;
};
static BuildWs build_layout(int64_t m) {
  BuildWs w;
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)std::max<int64_t>(m, 1), 0, 63);
  size_t o = 0;
  w.lohi = o;
  o = al(o + 6 * sizeof(unsigned long long));
  w.codes_in = o;
  o = al(o + m * sizeof(unsigned long long));
  w.codes_out = o;
  o = al(o + m * sizeof(unsigned long long));
  w.ids_in = o;
  o = al(o + m * sizeof(int32_t));
  w.ids_out = o;
  o = al(o + m * sizeof(int32_t));
  w.sa = o;
  o = al(o + m * sizeof(double));
  w.first = o;
  o = al(o + (m + 1) * sizeof(uint32_t));
  w.cub = o;
  w.cub_bytes = cub_bytes;
  o = al(o + cub_bytes);
  w.total = o;
  return w;
}

size_t build_workspace_size(int64_t m, int64_t nv) {
  return std::max(build_layout(m).total, layout_ws(nv).total);
}

// GD_BUILD_TIMING=1: per-phase wall clock of bvh_build on stderr (stream
// synchronised at each mark; scripts/exp_build.py)
struct PhaseClock {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t;
  explicit PhaseClock(cudaStream_t st) : on(std::getenv("GD_BUILD_TIMING") != nullptr), s(st) {
    if (on) t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  build %-22s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

void bvh_build(const GdMesh& mesh, GdBvh& T, void* ws, size_t ws_bytes, int64_t* prim_order_host,
               int64_t* leaf_tris_host, cudaStream_t s) {
  PhaseClock clk(s);
  const int64_t m = mesh.m;
  GD_CHECK(m >= 1, GD_ERR_INVALID, "cannot build a BVH over an empty mesh");
  GD_CHECK(m < (1ll << 31), GD_ERR_INVALID, "mesh too large for 32-bit triangle ids");
  int64_t L = 1;
  int depth = 0;
  while (L * 2 <= m) {
    L *= 2;
    ++depth;
  }
  GD_CHECK(T.leaf_count == L && T.depth == depth && T.n_tris == m && T.nv == mesh.nv, GD_ERR_INVALID,
           "GdBvh sizes do not match the mesh (use gd_bvh_sizes)");
  BuildWs w = build_layout(m);
  GD_CHECK(ws != nullptr && ws_bytes >= build_workspace_size(m, mesh.nv), GD_ERR_WORKSPACE,
           "build workspace too small: need " + std::to_string(w.total) + " bytes");
  char* base = static_cast<char*>(ws);
  auto* lohi = reinterpret_cast<unsigned long long*>(base + w.lohi);
  auto* codes_in = reinterpret_cast<unsigned long long*>(base + w.codes_in);
  auto* codes_out = reinterpret_cast<unsigned long long*>(base + w.codes_out);
  auto* ids_in = reinterpret_cast<int32_t*>(base + w.ids_in);
  auto* ids_out = reinterpret_cast<int32_t*>(base + w.ids_out);
  auto* sa = reinterpret_cast<double*>(base + w.sa);

  k_bounds_init<<<1, 32, 0, s>>>(lohi);
  k_bounds<<<num_sms() * 4, 256, 0, s>>>(mesh, lohi);
  const unsigned g = (unsigned)((m + 255) / 256);
  k_morton<<<g, 256, 0, s>>>(mesh, lohi, codes_in, ids_in);
  size_t cub_bytes = w.cub_bytes;
  GD_CUDA(cub::DeviceRadixSort::SortPairs(base + w.cub, cub_bytes, codes_in, codes_out, ids_in, ids_out, (int)m, 0,
                                          63, s));
  GD_CUDA(cudaGetLastError());
  clk.mark("bounds+morton+sort");

  std::vector<int32_t> order(m);
  GD_CUDA(cudaMemcpyAsync(order.data(), ids_out, m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  std::vector<uint8_t> is_left(m, 0);
  if (m > L) {
    k_pair_sa<<<g, 256, 0, s>>>(mesh, ids_out, m, sa);
    std::vector<double> sa_h(m - 1);
    GD_CUDA(cudaMemcpyAsync(sa_h.data(), sa, (m - 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
    clk.mark("sa + D2H");
    pair_greedy(sa_h.data(), m, is_left.data());
  } else {
    GD_CUDA(cudaStreamSynchronize(s));
  }
  clk.mark("pairing (host)");
  // leaf assembly in Morton order (bvh.py:168-181)
  std::vector<uint32_t> first(L + 1);
  int64_t rank = 0;
  for (int64_t i = 0; i < m;) {
    first[rank] = (uint32_t)i;
    leaf_tris_host[2 * rank] = order[i];
    if (is_left[i]) {
      leaf_tris_host[2 * rank + 1] = order[i + 1];
      i += 2;
    } else {
      leaf_tris_host[2 * rank + 1] = -1;
      i += 1;
    }
    ++rank;
  }
  GD_CHECK(rank == L, GD_ERR_INVALID, "internal: pairing produced a wrong leaf count");
  first[L] = (uint32_t)m;
  for (int64_t i = 0; i < m; ++i) prim_order_host[i] = order[i];
  auto* first_d = reinterpret_cast<uint32_t*>(base + w.first);
  GD_CUDA(cudaMemcpyAsync(first_d, first.data(), (L + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  k_leaf_rec<<<(unsigned)((L + 255) / 256), 256, 0, s>>>(mesh, ids_out, first_d, L, reinterpret_cast<int4*>(T.leaf_rec));
  GD_CUDA(cudaGetLastError());
  clk.mark("leaf assembly + records");
  bvh_layout(mesh, T, ws, ws_bytes, s);  // reuses the workspace (stream-ordered)
  clk.mark("vertex layout + staging");
  refit(mesh, T, s);
  GD_CUDA(cudaStreamSynchronize(s));
  clk.mark("refit");
}

}  // namespace gd
