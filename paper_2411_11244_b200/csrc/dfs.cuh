// dfs.cuh -- the per-triangle depth-first comparator (query.py:622-708), the
// naive traversal the paper measures the front engine against: one thread per
// triangle of A walks B's tree depth-first, nearer child first, pruning
// against ONE shared monotone bound (the float32 bound cell of the engine,
// slack E included), and counts every node it pops.  Leaves feed the same
// band / exact pass as the front engine (k_refine), so the answer
// is the reference's exact distance and lexicographic witness.
#pragma once

#include "narrow.cuh"

namespace gd {

constexpr int kDfsThreads = 128;
constexpr int kDfsStack = 64;  // 2 entries per level at most (depth <= 31)

// max |coordinate| of A's transformed vertices (the slack's scale; A has no
// tree here to read a root box from)
__global__ __launch_bounds__(256) void k_dfs_scale(GdMesh ma, QState* S) {
  float m = 0.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ma.nv;
       i += (long long)gridDim.x * blockDim.x) {
    const V3<double> v = mesh_vertex(ma, i);
    m = fmaxf(m, fmaxf(fabsf((float)v.x), fmaxf(fabsf((float)v.y), fabsf((float)v.z))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(&S->dfs_coord, __float_as_uint(m));
}

template <bool kMax>
__global__ void k_dfs_init(QArgs q) {
  QState* S = q.S;
  const Box rb = load_box(q.B.box, 0);
  float M = __uint_as_float(S->dfs_coord);
#pragma unroll
  for (int k = 0; k < 3; ++k) M = fmaxf(M, fmaxf(fabsf(rb.lo[k]), fabsf(rb.hi[k])));
  M = fmaxf(M, 0.125f * xf_mag(q.xb, stage_mag(q.B)));  // B's float32 transform rounding (init_query)
  // a little above the engine's 2^-15: A's float32 triangles here are the
  // float64-transformed ones rounded (mesh_tri), B's the staged ones
  S->slack = M * 0x1p-14f;
  S->bound_bits = __float_as_uint(kMax ? 0.f : INFINITY);  // query.py:632
  S->best.hi = ~0ull;
  S->best.lo = ~0ull;
  S->done = 0;
  S->err = 0;
  S->iter = 0;
  S->n_leaf = 0;
  S->rounds = 1;
  S->pending = 0;
  S->n_band = 0;
  S->fbest = kMax ? 0u : __float_as_uint(INFINITY);
  S->expanded = 0;
  S->narrow = 0;
  S->band_eval = 0;
  S->band_overflow = 0;
  S->rescanned = 0;
  S->n_cand = 0;  // no candidate list: k_refine reads the band only (direct_exact with 0 candidates)
  S->ov_cand = S->ov_in = S->ov_cap = 0;
  S->visited = 0;
}

template <bool kMax>
__device__ __forceinline__ void dfs_leaf(const QArgs& q, unsigned ta, const Tri<float>& A, unsigned long long leaf,
                                         unsigned long long& tested) {
  QState* S = q.S;
  const float E = S->slack;
  const LeafRec r = load_leaf(q.B, leaf);
  for (int i = 0; i < r.count(); ++i) {
    const Tri<float> B = leaf_tri32(q.B, q.xb, r, i);
    float d, lb;
    if (kMax)
      d = lb = sqrtf(tri_tri_max_d2<Fast<float>, float, false>(A, B, nullptr, nullptr));
    else
      tri_tri_min_fast_lb(A, B, d, lb);  // the band windows on the lower bound
    ++tested;
    const float ub = load_bound(S);
    if (kMax ? d + E < ub : lb - E > ub) continue;  // cannot be the answer
    const unsigned long long slot = atomicAdd(&S->n_band, 1ull);
    if (slot < q.band_cap) {
      q.band_ids[slot] = make_uint2(ta, r.tri_id(i));
      q.band_d[slot] = lb;
    } else {
      S->band_overflow = 1;
    }
    if (kMax ? d - E > ub : d + E < ub) commit_bound<kMax>(S, d);
    const unsigned fb = *reinterpret_cast<volatile unsigned*>(&S->fbest);
    if (kMax ? __float_as_uint(d) > fb : __float_as_uint(d) < fb) {
      if (kMax)
        atomicMax(&S->fbest, __float_as_uint(d));
      else
        atomicMin(&S->fbest, __float_as_uint(d));
    }
  }
}

// one thread per triangle of A; the stack holds (node, key) so a popped node
// is tested without reloading its box (keys were computed at the parent)
template <bool kMax>
__global__ __launch_bounds__(kDfsThreads) void k_dfs(QArgs q) {
  QState* S = q.S;
  const long long ta = (long long)blockIdx.x * kDfsThreads + threadIdx.x;
  unsigned long long visited = 0, tested = 0;
  if (ta < q.ma.m) {
    const Tri<float> A = mesh_tri<float>(q.ma, ta);
    const Box ab = tri_box(A);
    const unsigned long long first_leaf = (unsigned long long)q.B.leaf_count - 1;
    unsigned stack_node[kDfsStack];
    float stack_key[kDfsStack];
    int sp = 0;
    stack_node[0] = 0;
    stack_key[0] = pair_key<kMax>(ab, load_box(q.B.box, 0));
    sp = 1;
    while (sp > 0) {
      --sp;
      const unsigned node = stack_node[sp];
      const float key = stack_key[sp];
      ++visited;
      const float ub = load_bound(S);
      if (!survives<kMax>(key, ub * ub)) continue;
      if (node >= first_leaf) {
        dfs_leaf<kMax>(q, (unsigned)ta, A, node - first_leaf, tested);
        continue;
      }
      Box c0, c1;
      load_children(q.B.box, node, c0, c1);
      const float k0 = pair_key<kMax>(ab, c0), k1 = pair_key<kMax>(ab, c1);
      const bool left_first = kMax ? k0 >= k1 : k0 <= k1;  // query.py:698-705
      stack_node[sp] = left_first ? 2 * node + 2 : 2 * node + 1;
      stack_key[sp] = left_first ? k1 : k0;
      stack_node[sp + 1] = left_first ? 2 * node + 1 : 2 * node + 2;
      stack_key[sp + 1] = left_first ? k0 : k1;
      sp += 2;
    }
  }
  visited = warp_sum_u64(visited);
  tested = warp_sum_u64(tested);
  if ((threadIdx.x & 31) == 0) {
    if (visited) atomicAdd(&S->visited, visited);
    if (tested) atomicAdd(&S->narrow, tested);
  }
}

}  // namespace gd
