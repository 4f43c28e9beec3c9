// refit.cu -- per-frame refit (bvh.py:242-306) fused with apply_transform
// (mesh.py:102-105).
//
//   k_stage        float64 base vertex -> float32 float4 (once per base buffer)
//   k_leaf_up      one thread per leaf: its 32-byte record, six staged vertex
//                  gathers, float32 transform, leaf box = union of its 1..2
//                  triangles; then the block folds its 256-leaf subtree 8
//                  levels up in shared memory
//   k_level_up     the same fold for the remaining top levels
// Every node box is written exactly once; no level is re-read from HBM
// except the <= 1/256 subtree roots handed from one fold to the next.
#include <algorithm>
#include <vector>

#include "engine.cuh"

namespace gd {

constexpr int kFold = 256;  // nodes per block per fold (8 levels)

__global__ __launch_bounds__(256) void k_stage(GdMesh m, float4* __restrict__ out) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= m.nv) return;
  const double* p = m.vtx + 3 * i;
  out[i] = make_float4((float)p[0], (float)p[1], (float)p[2], 0.f);
}

// fold `levels` levels inside the block; sb holds blockDim.x boxes of level
// `lv`, the block covering nodes [first_rank, first_rank + blockDim.x)
__device__ __forceinline__ void fold_up(float* box, Box* sb, Box mine, int lv, long long first_rank,
                                        int levels) {
  int width = blockDim.x;
  sb[threadIdx.x] = mine;
  for (int u = 0; u < levels; ++u) {
    __syncthreads();
    width >>= 1;
    Box p;
    const bool act = threadIdx.x < width;
    if (act) p = box_union(sb[2 * threadIdx.x], sb[2 * threadIdx.x + 1]);
    __syncthreads();
    --lv;
    first_rank >>= 1;
    if (act) {
      sb[threadIdx.x] = p;
      store_box(box, ((1ull << lv) - 1) + first_rank + threadIdx.x, p);
    }
  }
}

__global__ __launch_bounds__(kFold) void k_leaf_up(GdBvh T, GdMesh m, int levels) {
  __shared__ Box sb[kFold];
  const long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // leaf rank (< L exactly)
  const XfF32 x = xf32_of(m);
  const LeafRec r = load_leaf(T, l);
  // both triangles unconditionally: a single-triangle leaf repeats triangle 0
  const Box b = box_union(tri_box(leaf_tri32(T, x, r, 0)), tri_box(leaf_tri32(T, x, r, 1)));
  store_box(T.box, (T.leaf_count - 1) + l, b);
  fold_up(T.box, sb, b, T.depth, blockIdx.x * (long long)blockDim.x, levels);
}

__global__ __launch_bounds__(kFold) void k_level_up(float* box, int lv, int levels) {
  __shared__ Box sb[kFold];
  const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  Box b = load_box(box, ((1ull << lv) - 1) + r);
  fold_up(box, sb, b, lv, blockIdx.x * (long long)blockDim.x, levels);
}

void stage_vertices(const GdMesh& m, const GdBvh& T, cudaStream_t s) {
  GD_CHECK(m.nv == T.nv, GD_ERR_TOPOLOGY, "mesh vertex count differs from the tree's");
  if (m.nv > 0) k_stage<<<(unsigned)((m.nv + 255) / 256), 256, 0, s>>>(m, reinterpret_cast<float4*>(T.vtx32));
  GD_CUDA(cudaGetLastError());
}

void refit(const GdMesh& m, const GdBvh& T, cudaStream_t s) {
  GD_CHECK(m.m == T.n_tris, GD_ERR_TOPOLOGY,
           "refit mesh has " + std::to_string(m.m) + " triangles, tree was built over " + std::to_string(T.n_tris));
  GD_CHECK(m.nv == T.nv, GD_ERR_TOPOLOGY, "refit mesh vertex count differs from the build");
  long long launches = 0;
  const long long L = T.leaf_count;
  int lv = T.depth;
  const int bs = (int)std::min<long long>(L, kFold);
  const int lev = std::min(lv, __builtin_ctz((unsigned)bs));
  k_leaf_up<<<(unsigned)(L / bs), bs, 0, s>>>(T, m, lev);
  ++launches;
  lv -= lev;
  while (lv > 0) {
    const long long cnt = 1ll << lv;
    const int b2 = (int)std::min<long long>(cnt, kFold);
    const int l2 = std::min(lv, __builtin_ctz((unsigned)b2));
    k_level_up<<<(unsigned)(cnt / b2), b2, 0, s>>>(T.box, lv, l2);
    ++launches;
    lv -= l2;
  }
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
  const int4 r0 = rec[0], r1 = rec[1];
  const int v[6] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y};
  const int nvert = r1.w >= 0 ? 6 : 3;
  T lo[3], hi[3];
  for (int c = 0; c < nvert; ++c) {
    V3<double> p = mesh_vertex(m, v[c]);
    T x[3] = {T(p.x), T(p.y), T(p.z)};
    for (int k = 0; k < 3; ++k) {
      if (c == 0) {
        lo[k] = hi[k] = x[k];
      } else {
        lo[k] = x[k] < lo[k] ? x[k] : lo[k];
        hi[k] = x[k] > hi[k] ? x[k] : hi[k];
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
    nmin[3 * node + k] = b < a ? b : a;  // np.minimum
    const T c = nmax[3 * c0 + k], d = nmax[3 * c1 + k];
    nmax[3 * node + k] = d > c ? d : c;  // np.maximum
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
