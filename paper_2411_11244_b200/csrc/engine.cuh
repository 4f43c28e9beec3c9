// engine.cuh -- shared definitions of the front-traversal engine.
#pragma once

#include "geometry.cuh"

namespace gd {

constexpr int kMaxIters = 64;

// Rigid transform of a mesh in float32 (from GdMesh's float64 R, t).  Every
// float32 vertex the traversal sees -- refit boxes, narrow filter --
// goes through xf_apply on the staged float32 base vertex, so the boxes
// contain exactly the vertices the narrow phase tests.
struct XfF32 {
  float r[9], t[3];
  int has;
};
// A's transform in B's local frame: R = Rb^T Ra, t = Rb^T (ta - tb)
inline GdMesh relative_mesh(const GdMesh& a, const GdMesh& b) {
  GdMesh r = a;
  double Ra[9], ta[3], Rb[9], tb[3];
  for (int i = 0; i < 9; ++i) {
    Ra[i] = a.has_xf ? a.rot[i] : (i % 4 == 0 ? 1.0 : 0.0);
    Rb[i] = b.has_xf ? b.rot[i] : (i % 4 == 0 ? 1.0 : 0.0);
  }
  for (int i = 0; i < 3; ++i) {
    ta[i] = a.has_xf ? a.trans[i] : 0.0;
    tb[i] = b.has_xf ? b.trans[i] : 0.0;
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.rot[3 * i + j] = (Rb[i] * Ra[j] + Rb[3 + i] * Ra[3 + j]) + Rb[6 + i] * Ra[6 + j];
  for (int i = 0; i < 3; ++i)
    r.trans[i] = (Rb[i] * (ta[0] - tb[0]) + Rb[3 + i] * (ta[1] - tb[1])) + Rb[6 + i] * (ta[2] - tb[2]);
  r.has_xf = 1;
  return r;
}

// computed once on the host (float64 -> float32 conversions are slow on the
// device) and passed by value in the kernel arguments
inline XfF32 xf32_host(const GdMesh& m) {
  XfF32 x;
  for (int i = 0; i < 9; ++i) x.r[i] = (float)m.rot[i];
  for (int i = 0; i < 3; ++i) x.t[i] = (float)m.trans[i];
  x.has = m.has_xf;
  return x;
}
// One level of the traversal's front stack: node pairs at one depth pair,
// entries [off, off + n) of the front arena, [off, off + cur) already expanded.
// The arena holds two stacks growing towards each other (end 0 from index 0
// up, end 1 from the arena's top down); a level's children go to the other
// end, so a sweep never writes the range it reads, and a level consumed in one
// sweep frees its space at once (breadth-first fronts ping-pong between the
// ends like a double buffer).  See DESIGN.md "Front arena".
struct Level {
  unsigned long long off, n, cur;
  int da, db;  // depth pair (query.py:116-133: one per front)
  int it;      // iteration index (IterationStat) of the sweeps expanding it
  int end;     // 0 = low stack, 1 = high stack
};
constexpr int kMaxLevels = 64;

// Device-resident query state (lives at the start of the workspace).
struct alignas(16) QState {
  Key128 best;                       // exact (distance, tri_a, tri_b) key
  unsigned int bound_bits;           // float32 bits of the slack-carrying bound
  unsigned int done;                 // last-block-done counter
  int err;
  int iter;                          // iterations (levels) recorded so far
  int sp;                            // front stack depth
  int chunked;                       // a level did not fit the arena: k = 1 from then on
  int pending;                       // a leaf chunk went to the narrow phase, levels remain
  int rounds;                        // traversal rounds (k_traverse launches) so far
  unsigned long long lo_top, hi_bot; // arena stack tops (entries); gap = [lo_top, hi_bot)
  unsigned long long leaf_off, n_leaf;   // this round's leaf-pair list (arena entries)
  int leaf_end;
  int paused;                        // the last traversal launch stopped at its sweep budget (mode 1)
  unsigned long long cand_off, cand_cap; // triangle-pair candidates (k_nfilter -> k_ntest), in the gap
  unsigned long long n_band;
  unsigned long long n_cand;         // triangle-pair candidates (k_nfilter)
  unsigned long long expanded, narrow, culled, band_eval, ncand_total;
  long long ov_cand, ov_in, ov_cap;
  float slack;
  int band_overflow;
  int rescanned;                     // the rescan pass covered this round's band overflow (query_round)
  unsigned fbest;                    // best float32 narrow distance (ordered bits)
  unsigned dfs_coord;                // per-triangle DFS: max |coordinate| of A (float bits)
  unsigned long long visited;        // per-triangle DFS: node examinations
  unsigned long long cnt[3];                   // sweep i % 3: survivors (low 40 bits) + arrivals
  unsigned long long epoch_flag;                // k_traverse: the launch epoch whose prologue is done
  unsigned long long skip_it[kMaxIters];       // candidates of pairs another split rank owns
  unsigned long long tot_cand[kMaxIters];      // candidates expanded per iteration (all chunks)
  unsigned long long tot_in[kMaxIters];        // front entries expanded per iteration
  unsigned long long tot_out[kMaxIters];       // survivors per iteration (leaf pairs for the last)
  Level lv[kMaxLevels];              // the front stack (persists across rounds)
  GdResult res;                      // the result record, then the stats: one
  GdIterStat stats[kMaxIters];       // contiguous device->host copy
  unsigned long long t_it[kMaxIters + 1];      // %globaltimer at iteration boundaries
  unsigned long long t_sweep[kMaxIters];       // last block's sweep end (profiling)
  unsigned long long t_plan[kMaxIters + 1];    // block 0: next sweep planned after iteration i's barrier
  unsigned long long t_edge[3];                // profiling: k_traverse entry, prologue barrier passed, exit (block 0)
};


struct QArgs {
  GdMesh ma, mb;
  XfF32 xa, xb;  // float32 transforms of ma, mb (xf32_host)
  int profile;    // record per-iteration sweep times (gd_set_profiling)
  int round;      // traversal round (0: the query starts)
  int mode;       // 0: a round resumes after a leaf chunk; 1: continue a query paused at its sweep budget
                  //    (a no-op once its traversal ended) -- the split query's bound-exchange rounds
  int sweep_budget;  // expansion sweeps this launch may run (0 = no limit)
  unsigned long long epoch;     // unique per k_traverse launch (query.cu next_epoch)
  GdBvh A, B;
  GdConfig cfg;
  QState* S;
  uint2* fnode;                 // front arena: node pairs ...
  float* fkey;                  // ... and their squared keys
  uint2* band_ids;
  float* band_d;
  unsigned long long arena;     // front arena capacity (entries)
  unsigned long long band_cap;  // band capacity (entries)
  GdResult* result;             // device result record
};

// 24-byte AoS node boxes (minx,miny,minz,maxx,maxy,maxz), stored at slot
// node + 1 (slot 0 is padding): the sibling pair (2i+1, 2i+2) then starts at
// byte 48 (i + 1), 16-byte aligned, and loads as three float4.
__device__ __forceinline__ Box load_box(const float* __restrict__ box, unsigned long long node) {
  const float2* p = reinterpret_cast<const float2*>(box + (node + 1) * 6);
  float2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
  Box r;
  r.lo[0] = a.x; r.lo[1] = a.y; r.lo[2] = b.x;
  r.hi[0] = b.y; r.hi[1] = c.x; r.hi[2] = c.y;
  return r;
}
// both children of `parent` (nodes 2 parent + 1, 2 parent + 2)
__device__ __forceinline__ void load_children(const float* __restrict__ box, unsigned long long parent, Box& c0,
                                              Box& c1) {
  const float4* p = reinterpret_cast<const float4*>(box + (2 * parent + 2) * 6);
  const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
  c0.lo[0] = a.x; c0.lo[1] = a.y; c0.lo[2] = a.z;
  c0.hi[0] = a.w; c0.hi[1] = b.x; c0.hi[2] = b.y;
  c1.lo[0] = b.z; c1.lo[1] = b.w; c1.lo[2] = c.x;
  c1.hi[0] = c.y; c1.hi[1] = c.z; c1.hi[2] = c.w;
}
__device__ __forceinline__ void store_box(float* box, unsigned long long node, const Box& r) {
  float2* p = reinterpret_cast<float2*>(box + (node + 1) * 6);
  p[0] = make_float2(r.lo[0], r.lo[1]);
  p[1] = make_float2(r.lo[2], r.hi[0]);
  p[2] = make_float2(r.hi[1], r.hi[2]);
}
__device__ __forceinline__ Box select_box(bool c, const Box& a, const Box& b) {
  Box r;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = c ? a.lo[k] : b.lo[k];
    r.hi[k] = c ? a.hi[k] : b.hi[k];
  }
  return r;
}
__device__ __forceinline__ Box box_union(const Box& a, const Box& b) {
  Box r;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = fmin_nan(a.lo[k], b.lo[k]);
    r.hi[k] = fmax_nan(a.hi[k], b.hi[k]);
  }
  return r;
}

__device__ __forceinline__ V3<float> xf_apply(const XfF32& x, const float4 v) {
  if (!x.has) return {v.x, v.y, v.z};
  return {fmaf(x.r[0], v.x, fmaf(x.r[1], v.y, fmaf(x.r[2], v.z, x.t[0]))),
          fmaf(x.r[3], v.x, fmaf(x.r[4], v.y, fmaf(x.r[5], v.z, x.t[1]))),
          fmaf(x.r[6], v.x, fmaf(x.r[7], v.y, fmaf(x.r[8], v.z, x.t[2])))};
}
// float32 triangle from three vertex indices of the staged base vertices
__device__ __forceinline__ Tri<float> tri32(const GdBvh& T, const XfF32& x, int i0, int i1, int i2) {
  const float4* v = reinterpret_cast<const float4*>(T.vtx32);
  const float4 a = __ldg(v + i0), b = __ldg(v + i1), c = __ldg(v + i2);
  Tri<float> t;
  t.v[0] = xf_apply(x, a);
  t.v[1] = xf_apply(x, b);
  t.v[2] = xf_apply(x, c);
  return t;
}
// leaf record (gdist.h): {a0,a1,a2, b0,b1,b2, tri0, tri1}; r0 = first int4
struct LeafRec {
  int4 r0, r1;
  __device__ __forceinline__ int count() const { return r1.w >= 0 ? 2 : 1; }
  __device__ __forceinline__ unsigned tri_id(int i) const { return (unsigned)(i ? r1.w : r1.z); }
};
__device__ __forceinline__ LeafRec load_leaf(const GdBvh& T, unsigned long long leaf) {
  const int4* p = reinterpret_cast<const int4*>(T.leaf_rec) + 2 * leaf;
  LeafRec r;
  r.r0 = __ldg(p);
  r.r1 = __ldg(p + 1);
  return r;
}
__device__ __forceinline__ Tri<float> leaf_tri32(const GdBvh& T, const XfF32& x, const LeafRec& r, int i) {
  return i ? tri32(T, x, r.r0.w, r.r1.x, r.r1.y) : tri32(T, x, r.r0.x, r.r0.y, r.r0.z);
}

// both triangles of a leaf from leaf_tri (gdist.h): one 80-byte load,
// transformed by xf_apply exactly as tri32 does (bitwise the same vertices)
struct LeafTris {
  Tri<float> t[2];
  int tri0, tri1;
  __device__ __forceinline__ int count() const { return tri1 >= 0 ? 2 : 1; }
  __device__ __forceinline__ unsigned tri_id(int i) const { return (unsigned)(i ? tri1 : tri0); }
};
__device__ __forceinline__ LeafTris load_leaf_tris(const GdBvh& T, const XfF32& x, unsigned long long leaf) {
  const float4* p = reinterpret_cast<const float4*>(T.leaf_tri) + 5 * leaf;
  const float4 f0 = __ldg(p), f1 = __ldg(p + 1), f2 = __ldg(p + 2), f3 = __ldg(p + 3), f4 = __ldg(p + 4);
  LeafTris r;
  r.t[0].v[0] = xf_apply(x, make_float4(f0.x, f0.y, f0.z, 0.f));
  r.t[0].v[1] = xf_apply(x, make_float4(f0.w, f1.x, f1.y, 0.f));
  r.t[0].v[2] = xf_apply(x, make_float4(f1.z, f1.w, f2.x, 0.f));
  r.t[1].v[0] = xf_apply(x, make_float4(f2.y, f2.z, f2.w, 0.f));
  r.t[1].v[1] = xf_apply(x, make_float4(f3.x, f3.y, f3.z, 0.f));
  r.t[1].v[2] = xf_apply(x, make_float4(f3.w, f4.x, f4.y, 0.f));
  r.tri0 = __float_as_int(f4.z);
  r.tri1 = __float_as_int(f4.w);
  return r;
}
// one triangle (i = 0, 1) of a leaf: 40 bytes of the record
__device__ __forceinline__ Tri<float> load_leaf_tri(const GdBvh& T, const XfF32& x, unsigned long long leaf, int i) {
  const float4* p = reinterpret_cast<const float4*>(T.leaf_tri) + 5 * leaf;
  Tri<float> t;
  if (i == 0) {
    const float4 f0 = __ldg(p), f1 = __ldg(p + 1), f2 = __ldg(p + 2);
    t.v[0] = xf_apply(x, make_float4(f0.x, f0.y, f0.z, 0.f));
    t.v[1] = xf_apply(x, make_float4(f0.w, f1.x, f1.y, 0.f));
    t.v[2] = xf_apply(x, make_float4(f1.z, f1.w, f2.x, 0.f));
  } else {
    const float4 f2 = __ldg(p + 2), f3 = __ldg(p + 3), f4 = __ldg(p + 4);
    t.v[0] = xf_apply(x, make_float4(f2.y, f2.z, f2.w, 0.f));
    t.v[1] = xf_apply(x, make_float4(f3.x, f3.y, f3.z, 0.f));
    t.v[2] = xf_apply(x, make_float4(f3.w, f4.x, f4.y, 0.f));
  }
  return t;
}

__device__ __forceinline__ Box tri_box(const Tri<float>& t) {
  Box b;
  b.lo[0] = fminf(fminf(t.v[0].x, t.v[1].x), t.v[2].x);
  b.lo[1] = fminf(fminf(t.v[0].y, t.v[1].y), t.v[2].y);
  b.lo[2] = fminf(fminf(t.v[0].z, t.v[1].z), t.v[2].z);
  b.hi[0] = fmaxf(fmaxf(t.v[0].x, t.v[1].x), t.v[2].x);
  b.hi[1] = fmaxf(fmaxf(t.v[0].y, t.v[1].y), t.v[2].y);
  b.hi[2] = fmaxf(fmaxf(t.v[0].z, t.v[1].z), t.v[2].z);
  return b;
}

// float64 vertex of a mesh with its rigid transform applied (mesh.py:102-105:
// `V @ R.T + t`).  numpy's matmul is OpenBLAS dgemm, whose kernels accumulate
// over k with fused multiply-adds, x' = fma(R02, z, fma(R01, y, R00 x)), and
// the translation is a separate add -- reproduced here, so a moved mesh has
// the reference's vertex bits (tests/test_gpu_parity.py).
// one row of R v in the host BLAS's order (GdMesh.xf_order)
__device__ __forceinline__ double xf_row(const double* r, double x, double y, double z, int order) {
  if (order == 1) return __dadd_rn(__dadd_rn(__dmul_rn(r[0], x), __dmul_rn(r[1], y)), __dmul_rn(r[2], z));
  if (order == 2) return __fma_rn(r[0], x, __fma_rn(r[1], y, __dmul_rn(r[2], z)));
  return __fma_rn(r[2], z, __fma_rn(r[1], y, __dmul_rn(r[0], x)));
}
// kOrder >= 0: the order fixed at compile time (the exact pass is
// instantiated per order: a runtime switch per vertex cost it ~4 us on the
// rings); -1: GdMesh.xf_order at run time
template <int kOrder = -1>
__device__ __forceinline__ V3<double> mesh_vertex(const GdMesh& m, long long i) {
  const double* p = m.vtx + 3 * i;
  double x = p[0], y = p[1], z = p[2];
  if (!m.has_xf) return {x, y, z};
  const double* R = m.rot;
  const int o = kOrder >= 0 ? kOrder : m.xf_order;
  return {__dadd_rn(xf_row(R, x, y, z, o), m.trans[0]),
          __dadd_rn(xf_row(R + 3, x, y, z, o), m.trans[1]),
          __dadd_rn(xf_row(R + 6, x, y, z, o), m.trans[2])};
}

template <typename T, int kOrder = -1>
__device__ __forceinline__ Tri<T> mesh_tri(const GdMesh& m, long long t) {
  const int32_t* ix = m.tri + 3 * t;
  Tri<T> r;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    V3<double> v = mesh_vertex<kOrder>(m, ix[c]);
    r.v[c] = {T(v.x), T(v.y), T(v.z)};  // cast-then-gather (mesh.py:64-66)
  }
  return r;
}

// leaf_x slot (gdist.h) holding the float bits of max |coordinate| of the
// staged float32 base vertices (k_stage): the scale of the float32
// transform's rounding, which the slack must cover
__host__ __device__ __forceinline__ long long stage_mag_slot(long long leaf_count) {
  return 2 * ((leaf_count + 31) / 32) + 1 + 2 * (leaf_count >> 16) + 4;
}
__device__ __forceinline__ float stage_mag(const GdBvh& T) {
  return __uint_as_float(*reinterpret_cast<const volatile unsigned*>(T.leaf_x + stage_mag_slot(T.leaf_count)));
}
// bound on |x'| for x' = R v + t with |v| <= vmax per coordinate, and on the
// partial sums of xf_apply's FMA chain
__device__ __forceinline__ float xf_mag(const XfF32& x, float vmax) {
  if (!x.has) return vmax;
  float m = 0.f;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    m = fmaxf(m, (fabsf(x.r[3 * i]) + fabsf(x.r[3 * i + 1]) + fabsf(x.r[3 * i + 2])) * vmax + fabsf(x.t[i]));
  return m;
}

}  // namespace gd
