// build.cu -- f12-BVH construction (bvh.py:69-95, 98-181, 267-289).
//
//   k_bounds       float64 min/max over ALL vertices (bvh.py:82-83)
//   k_morton       centroid ((p0+p1)+p2)/3, 21-bit quantisation, 63-bit
//                  interleave, x at bit 0 (bvh.py:58-95)
//   radix sort     stable (code, id) sort == np.lexsort((ids, codes)),
//                  the repo's own LSD sort (primitives.cuh, sort.cu)
//   k_pair_sa      float64 surface area of Morton neighbours (bvh.py:117-120)
//   k_pair_*       the greedy power-of-two pairing on the device (scans +
//                  sort, checked exact), else the exact greedy on the host
//                  (pairing.cpp)
//   leaf assembly  leaf ranks by scan, leaf_tris / prim_order, k_leaf_rec
//                  (one 32-byte record per leaf, gdist.h)
//   bvh_layout     staged-vertex numbering by first use in leaf order
//                  (k_first_use + radix sort + k_rec_remap), staging
// then refit() fills every box.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "engine.cuh"
#include "primitives.cuh"

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

static size_t al(size_t x) { return (x + 255) / 256 * 256; }

// bump allocator over a workspace (offsets only: sizing and carving share it)
struct Carve {
  size_t o = 0;
  size_t take(size_t bytes) {
    const size_t r = o;
    o = al(o + bytes);
    return r;
  }
};

struct LayoutWs {
  size_t first, first_out, ids, ids_out, ktmp, vtmp, sort, total;
};
static LayoutWs layout_ws(int64_t nv) {
  LayoutWs w;
  Carve c;
  const size_t n = (size_t)std::max<int64_t>(nv, 1);
  w.first = c.take(n * sizeof(uint32_t));
  w.first_out = c.take(n * sizeof(uint32_t));
  w.ids = c.take(n * sizeof(int32_t));
  w.ids_out = c.take(n * sizeof(int32_t));
  w.ktmp = c.take(n * sizeof(uint32_t));
  w.vtmp = c.take(n * sizeof(int32_t));
  w.sort = c.take(radix_sort_ws_bytes((long long)n));
  w.total = c.o;
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
    // stable: unused vertices (key 0xFFFFFFFF) keep their id order at the end
    radix_sort_pairs(first, ids, reinterpret_cast<uint32_t*>(base + w.ktmp), reinterpret_cast<int32_t*>(base + w.vtmp),
                     first_out, ids_out, nv, 32, base + w.sort, s);
    k_vmap<<<gv, 256, 0, s>>>(ids_out, nv, T.vmap);
    k_rec_remap<<<gl, 256, 0, s>>>(T.leaf_rec, L, T.vmap);
  }
  GD_CUDA(cudaGetLastError());
  stage_vertices(mesh, T, s);
}

size_t layout_workspace_size(int64_t nv) { return layout_ws(nv).total; }

// ---------------------------------------------------------------------------
// Device restatement of _pair_to_power_of_two (bvh.py:98-181).
//
// Without its feasibility deferrals the reference is the sequential greedy
// matching of a path by increasing key (surface area, index) -- every key is
// distinct -- stopped after `need` merges.  The complete greedy matching of a
// path has a local rule: a pair is taken iff no adjacent pair with a smaller
// key is taken, so along a run of keys increasing away from a local minimum
// the taken pairs alternate (the minimum, then every second one) and a local
// maximum is taken iff neither neighbour is.  Two scans give every pair's
// distance to the local minimum of its run (k_pair_*); the greedy takes the
// matching's pairs in key order, so the reference's merges are the `need`
// smallest keys of the matching (radix sort).  That holds exactly when the
// reference never deferred, i.e. when its slack (sum over runs of unmerged
// triangles of floor(len / 2), minus the merges still needed; it never
// increases) stayed positive -- equivalently when the final slack is >= 1,
// which the build checks on the device.  Otherwise (and for NaN keys, whose
// heap order is Python's) the exact host restatement (pairing.cpp) runs.
struct PairKeys {
  const double* sa;
  long long E;  // pairs (n - 1)
  __device__ __forceinline__ bool less(long long i, long long j) const {
    const double a = sa[i], b = sa[j];
    return a < b || (a == b && i < j);
  }
  // the left neighbour's key is smaller: i continues a run rising from the left
  __device__ __forceinline__ bool ls(long long i) const { return i > 0 && less(i - 1, i); }
  __device__ __forceinline__ bool rs(long long i) const { return i + 1 < E && less(i + 1, i); }
};
// last j <= i where a rising run starts (no smaller left neighbour)
struct RunStartIn {
  PairKeys k;
  __device__ __forceinline__ int operator()(long long i) const { return k.ls(i) ? -1 : (int)i; }
};
struct StoreInt {
  int* a;
  __device__ __forceinline__ void operator()(long long i, int v, int) const { a[i] = v; }
};
// first j >= i where a run falling to the right ends (scanned right to left)
struct RunEndIn {
  PairKeys k;
  __device__ __forceinline__ int operator()(long long r) const {
    const long long i = k.E - 1 - r;
    return k.rs(i) ? (int)k.E : (int)i;
  }
};
struct StoreIntRev {
  int* a;
  long long E;
  __device__ __forceinline__ void operator()(long long r, int v, int) const { a[E - 1 - r] = v; }
};

__global__ __launch_bounds__(256) void k_pair_nan(const double* sa, long long E, unsigned long long* flags) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  const bool bad = i < E && sa[i] != sa[i];
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1ull);
}

// matched[i]: the pair is in the complete greedy matching
__global__ __launch_bounds__(256) void k_pair_match(PairKeys k, const int* S, const int* Eend, uint8_t* matched) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= k.E) return;
  const bool l = k.ls(i), r = k.rs(i);
  bool m;
  if (!l && !r)
    m = true;  // local minimum
  else if (l && !r)
    m = ((i - S[i]) & 1) == 0;
  else if (!l && r)
    m = ((Eend[i] - i) & 1) == 0;
  else  // local maximum: taken iff neither neighbour is
    m = ((i - 1 - S[i - 1]) & 1) != 0 && ((Eend[i + 1] - (i + 1)) & 1) != 0;
  matched[i] = m ? 1 : 0;
}

struct MatchedIn {
  const uint8_t* m;
  __device__ __forceinline__ int operator()(long long i) const { return m[i]; }
};
// compaction of the matched pairs: (order-preserving key of sa, index)
struct MatchedOut {
  const uint8_t* m;
  const double* sa;
  unsigned long long* keys;
  int32_t* idx;
  unsigned long long* count;
  long long E;
  __device__ __forceinline__ void operator()(long long i, int inc, int v) const {
    if (v) {
      keys[inc - 1] = dkey(sa[i]);
      idx[inc - 1] = (int32_t)i;
    }
    if (i == E - 1) *count = (unsigned long long)inc;
  }
};

// argmin segment trees over the pairs (node v: the index of the smallest
// (sa, index) key below it, -1 = none); leaves at size + i
struct ArgminTree {
  const double* sa;
  int* t;
  long long size;
  __device__ __forceinline__ bool less(int a, int b) const {  // -1 = +infinity
    if (a < 0) return false;
    if (b < 0) return true;
    return sa[a] < sa[b] || (sa[a] == sa[b] && a < b);
  }
  __device__ __forceinline__ int pick(int a, int b) const { return less(a, b) ? a : b; }
  // nearest j < p (largest) holding a key smaller than p's
  __device__ int prev_smaller(int p) const {
    long long v = size + p;
    while (v > 1) {
      if ((v & 1) && less(t[v - 1], p)) {
        v = v - 1;
        while (v < size) v = less(t[2 * v + 1], p) ? 2 * v + 1 : 2 * v;
        return (int)(v - size);
      }
      v >>= 1;
    }
    return -1;
  }
  // nearest j > p (smallest) holding a key smaller than p's
  __device__ int next_smaller(int p) const {
    long long v = size + p;
    while (v > 1) {
      if (!(v & 1) && less(t[v + 1], p)) {
        v = v + 1;
        while (v < size) v = less(t[2 * v], p) ? 2 * v : 2 * v + 1;
        return (int)(v - size);
      }
      v >>= 1;
    }
    return -1;
  }
  // smallest key among pairs [l, r]
  __device__ int argmin(long long l, long long r) const {
    int best = -1;
    for (long long a = l + size, b = r + size + 1; a < b; a >>= 1, b >>= 1) {
      if (a & 1) best = pick(best, t[a++]);
      if (b & 1) best = pick(best, t[--b]);
    }
    return best;
  }
};

// leaves: every pair (tree A) or the matching's pairs only (tree B)
__global__ __launch_bounds__(256) void k_tree_leaves(ArgminTree T, long long E, const uint8_t* only) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= T.size) return;
  T.t[T.size + i] = (i < E && (!only || only[i])) ? (int)i : -1;
}
__global__ __launch_bounds__(256) void k_tree_level(ArgminTree T, long long lo, long long hi) {
  const long long v = lo + blockIdx.x * 256ll + threadIdx.x;
  if (v < hi) T.t[v] = T.pick(T.t[2 * v], T.t[2 * v + 1]);
}
static void build_tree(const ArgminTree& T, long long E, const uint8_t* only, cudaStream_t s) {
  k_tree_leaves<<<(unsigned)((T.size + 255) / 256), 256, 0, s>>>(T, E, only);
  for (long long lo = T.size / 2; lo >= 1; lo /= 2)
    k_tree_level<<<(unsigned)((lo + 255) / 256), 256, 0, s>>>(T, lo, 2 * lo);
}

// Phase 1 (the greedy before its slack first reaches 0): the matching's pairs
// are taken in key order; pair p is costly -- it lowers the slack -- when the
// run of unmerged triangles around it at that moment has even length and p
// sits at an odd offset.  That run is bounded by the nearest matching pairs
// with smaller keys on either side (taken before p).
__global__ __launch_bounds__(256) void k_pair_costly(ArgminTree B, const uint8_t* matched, long long E, long long n,
                                                      uint8_t* costly) {
  const long long p = blockIdx.x * 256ll + threadIdx.x;
  if (p >= E) return;
  if (!matched[p]) {
    costly[p] = 0;
    return;
  }
  const int q = B.prev_smaller((int)p), r = B.next_smaller((int)p);
  const long long s = q >= 0 ? q + 2 : 0, e = r >= 0 ? r - 1 : n - 1;
  costly[p] = (((e - s + 1) & 1) == 0 && ((p - s) & 1) == 1) ? 1 : 0;
}

// the slack after the r-th pick (key order) is slack0 - costly picks so far;
// k* = the pick that brings it to 0 (the reference defers after it)
struct CostlySortedIn {
  const int32_t* sorted;
  const uint8_t* costly;
  __device__ __forceinline__ int operator()(long long r) const { return costly[sorted[r]]; }
};
struct SlackOut {
  long long slack0;
  unsigned long long* kstar;  // ~0 = never
  __device__ __forceinline__ void operator()(long long r, int inc, int v) const {
    if (v && slack0 - inc <= 0 && slack0 - (inc - v) > 0) *kstar = (unsigned long long)r;
  }
};
__global__ __launch_bounds__(256) void k_pair_take(const int32_t* sorted_idx, long long count, uint8_t* is_left) {
  const long long r = blockIdx.x * 256ll + threadIdx.x;
  if (r < count) is_left[sorted_idx[r]] = 1;
}

// runs of unmerged triangles: the next merged position at or after t
struct NextMergedIn {
  const uint8_t* is_left;
  long long n;
  __device__ __forceinline__ int operator()(long long r) const {
    const long long t = n - 1 - r;
    const bool merged = is_left[t] || (t > 0 && is_left[t - 1]);
    return merged ? (int)t : (int)n;
  }
};

// Phase 2 (slack 0): runs evolve independently.  In an even run only pairs at
// even offsets are feasible; they are disjoint, so all are taken.  In an odd
// run every pair is feasible: the smallest key is taken, leaving an even part
// (all its even offsets taken) and an odd part that repeats.  One thread per
// run; the runs are disjoint.
__global__ __launch_bounds__(256) void k_pair_phase2(ArgminTree A, const int* next_merged, long long n,
                                                      uint8_t* is_left) {
  const long long t = blockIdx.x * 256ll + threadIdx.x;
  if (t >= n) return;
  // run starts from the phase-1 state only (next_merged[t] == t: t merged),
  // never from is_left, which the other runs' threads are writing
  if (next_merged[t] == t || (t > 0 && next_merged[t - 1] != t - 1)) return;
  long long lo = t, hi = (long long)next_merged[t] - 1;
  auto take_even = [&](long long a, long long b) {  // all even offsets of [a, b]
    for (long long i = a; i + 1 <= b; i += 2) is_left[i] = 1;
  };
  while (hi - lo + 1 >= 2) {
    if (((hi - lo + 1) & 1) == 0) {
      take_even(lo, hi);
      break;
    }
    const long long i = A.argmin(lo, hi - 1);
    is_left[i] = 1;
    if (((i - lo) & 1) == 0) {  // left part even, right part odd
      take_even(lo, i - 1);
      lo = i + 2;
    } else {
      take_even(i + 2, hi);
      hi = i - 1;
    }
  }
}

// leaf assembly (bvh.py:168-181): a leaf starts at every Morton rank that is
// not the right half of a merged pair; its rank is the count of earlier
// starts (scan)
struct LeafStartIn {
  const uint8_t* is_left;
  __device__ __forceinline__ int operator()(long long t) const { return (t > 0 && is_left[t - 1]) ? 0 : 1; }
};
struct LeafOut {
  const uint8_t* is_left;
  const int32_t* order;
  uint32_t* first;
  long long* leaf_tris;
  long long* prim;
  long long n, L;
  unsigned long long* err;
  __device__ __forceinline__ void operator()(long long t, int inc, int v) const {
    prim[t] = order[t];
    if (!v) return;
    const long long leaf = inc - 1;
    if (leaf >= L) {  // a pairing that does not give 2^k leaves (checked by the host)
      atomicOr(err, 1ull);
      return;
    }
    first[leaf] = (uint32_t)t;
    leaf_tris[2 * leaf] = order[t];
    leaf_tris[2 * leaf + 1] = is_left[t] ? order[t + 1] : -1;
    if (t == n - 1 || (t == n - 2 && is_left[t])) first[leaf + 1] = (uint32_t)n;
  }
};

struct BuildWs {
  size_t lohi, codes_in, codes_out, codes_tmp, ids_in, ids_out, ids_tmp, sa, S, Eend, flag, costly, treeA, treeB,
      leaf_tris, prim, first, counters, aggr, sort, total;
};
static BuildWs build_layout(int64_t m) {
  BuildWs w;
  Carve c;
  const size_t n = (size_t)std::max<int64_t>(m, 1);
  int64_t L = 1;
  while (L * 2 <= (int64_t)n) L *= 2;
  w.lohi = c.take(6 * sizeof(unsigned long long));
  w.codes_in = c.take(n * sizeof(unsigned long long));
  w.codes_out = c.take(n * sizeof(unsigned long long));
  w.codes_tmp = c.take(n * sizeof(unsigned long long));
  w.ids_in = c.take(n * sizeof(int32_t));
  w.ids_out = c.take(n * sizeof(int32_t));
  w.ids_tmp = c.take(n * sizeof(int32_t));
  w.sa = c.take(n * sizeof(double));
  w.S = c.take(n * sizeof(int));
  w.Eend = c.take(n * sizeof(int));
  w.flag = c.take(2 * n);  // matched, is_left
  w.costly = c.take(n);
  size_t tsz = 1;
  while (tsz < n) tsz <<= 1;
  w.treeA = c.take(2 * tsz * sizeof(int));
  w.treeB = c.take(2 * tsz * sizeof(int));
  w.leaf_tris = c.take(2 * (size_t)L * sizeof(long long));
  w.prim = c.take(n * sizeof(long long));
  w.first = c.take(((size_t)L + 1) * sizeof(uint32_t));
  w.counters = c.take(8 * sizeof(unsigned long long));
  w.aggr = c.take((size_t)scan_tiles((long long)n) * sizeof(long long));
  w.sort = c.take(radix_sort_ws_bytes((long long)n));
  w.total = c.o;
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
    std::fprintf(stderr, "  build %-24s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// which pairing the last build used (gd_build_pairing_mode): 0 none needed,
// 1 device, 2 host (a deferral was possible, or NaN keys)
static thread_local int g_pairing_mode = 0;
int build_pairing_mode() { return g_pairing_mode; }

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
  auto* codes_tmp = reinterpret_cast<unsigned long long*>(base + w.codes_tmp);
  auto* ids_in = reinterpret_cast<int32_t*>(base + w.ids_in);
  auto* ids_out = reinterpret_cast<int32_t*>(base + w.ids_out);
  auto* ids_tmp = reinterpret_cast<int32_t*>(base + w.ids_tmp);
  auto* sa = reinterpret_cast<double*>(base + w.sa);
  auto* S = reinterpret_cast<int*>(base + w.S);
  auto* Eend = reinterpret_cast<int*>(base + w.Eend);
  auto* matched = reinterpret_cast<uint8_t*>(base + w.flag);
  uint8_t* is_left = matched + m;
  auto* leaf_tris_d = reinterpret_cast<long long*>(base + w.leaf_tris);
  auto* prim_d = reinterpret_cast<long long*>(base + w.prim);
  auto* first_d = reinterpret_cast<uint32_t*>(base + w.first);
  auto* counters = reinterpret_cast<unsigned long long*>(base + w.counters);
  void* sort_ws = base + w.sort;

  k_bounds_init<<<1, 32, 0, s>>>(lohi);
  k_bounds<<<num_sms() * 4, 256, 0, s>>>(mesh, lohi);
  const unsigned g = (unsigned)((m + 255) / 256);
  k_morton<<<g, 256, 0, s>>>(mesh, lohi, codes_in, ids_in);
  // stable (code, id) order == np.lexsort((ids, codes)) (bvh.py:93-94)
  radix_sort_pairs(codes_in, ids_in, codes_tmp, ids_tmp, codes_out, ids_out, m, 63, sort_ws, s);
  GD_CUDA(cudaGetLastError());
  clk.mark("bounds+morton+sort");

  GD_CUDA(cudaMemsetAsync(is_left, 0, (size_t)m, s));
  GD_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(unsigned long long), s));
  const int64_t need = m - L;
  g_pairing_mode = 0;
  if (need > 0) {
    const long long E = m - 1;
    const unsigned ge = (unsigned)((E + 255) / 256);
    k_pair_sa<<<g, 256, 0, s>>>(mesh, ids_out, m, sa);
    k_pair_nan<<<ge, 256, 0, s>>>(sa, E, counters + 0);
    const PairKeys pk{sa, E};
    int* aggr_i = reinterpret_cast<int*>(base + w.aggr);
    device_scan<int>(RunStartIn{pk}, StoreInt{S}, E, OpMax{}, -1, aggr_i, s);
    device_scan<int>(RunEndIn{pk}, StoreIntRev{Eend, E}, E, OpMin{}, (int)E, aggr_i, s);
    k_pair_match<<<ge, 256, 0, s>>>(pk, S, Eend, matched);
    // the matching's pairs in index order, keyed by their surface area
    device_scan<int>(MatchedIn{matched}, MatchedOut{matched, sa, codes_in, ids_in, counters + 1, E}, E, OpAdd{}, 0,
                     aggr_i, s);
    unsigned long long cnt[2];
    GD_CUDA(cudaMemcpyAsync(cnt, counters, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
    // GD_FORCE_HOST_PAIRING: the host greedy regardless (tests compare both)
    bool device_ok = cnt[0] == 0 && std::getenv("GD_FORCE_HOST_PAIRING") == nullptr;
    if (device_ok) {
      const long long nm = (long long)cnt[1];
      // the matching in key order: stable sort of the index-ordered pairs by sa
      radix_sort_pairs(codes_in, ids_in, codes_tmp, ids_tmp, codes_out, S, nm, 64, sort_ws, s);
      long long size = 1;
      while (size < E) size <<= 1;
      const ArgminTree TA{sa, reinterpret_cast<int*>(base + w.treeA), size};
      const ArgminTree TB{sa, reinterpret_cast<int*>(base + w.treeB), size};
      build_tree(TB, E, matched, s);
      uint8_t* costly = reinterpret_cast<uint8_t*>(base + w.costly);
      k_pair_costly<<<ge, 256, 0, s>>>(TB, matched, E, m, costly);
      GD_CUDA(cudaMemsetAsync(counters + 4, 0xFF, sizeof(unsigned long long), s));
      const long long slack0 = m / 2 - need;
      const long long upto = std::min<long long>(need, nm);
      unsigned long long kstar = ~0ull;
      if (slack0 > 0) {
        device_scan<int>(CostlySortedIn{S, costly}, SlackOut{slack0, counters + 4}, upto, OpAdd{}, 0, aggr_i, s);
        GD_CUDA(cudaMemcpyAsync(&kstar, counters + 4, sizeof kstar, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
      }
      const long long picks1 = slack0 <= 0 ? 0 : (kstar == ~0ull ? -1 : (long long)kstar + 1);  // -1: no zero slack
      if (picks1 < 0) {
        // the slack never reached 0: the `need` smallest pairs of the matching
        GD_CHECK(nm >= need, GD_ERR_INVALID, "internal: greedy matching smaller than the merges needed");
        k_pair_take<<<(unsigned)((need + 255) / 256), 256, 0, s>>>(S, need, is_left);
      } else {
        // phase 1 up to the pick that zeroes the slack (none if it starts at 0)
        if (picks1 > 0) k_pair_take<<<(unsigned)((picks1 + 255) / 256), 256, 0, s>>>(S, picks1, is_left);
        build_tree(TA, E, nullptr, s);
        device_scan<int>(NextMergedIn{is_left, m}, StoreIntRev{Eend, m}, m, OpMin{}, (int)m, aggr_i, s);
        k_pair_phase2<<<g, 256, 0, s>>>(TA, Eend, m, is_left);
      }
      GD_CUDA(cudaGetLastError());
    }
    if (device_ok) {
      g_pairing_mode = 1;
      count_launches(9);
      clk.mark("pairing (device)");
    } else {
      // exact host restatement of the greedy with its deferrals
      g_pairing_mode = 2;
      std::vector<double> sa_h(m - 1);
      GD_CUDA(cudaMemcpyAsync(sa_h.data(), sa, (m - 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
      GD_CUDA(cudaStreamSynchronize(s));
      std::vector<uint8_t> left(m, 0);
      pair_greedy(sa_h.data(), m, left.data());
      GD_CUDA(cudaMemcpyAsync(is_left, left.data(), (size_t)m, cudaMemcpyHostToDevice, s));
      GD_CUDA(cudaStreamSynchronize(s));
      clk.mark("pairing (host)");
    }
  }
  // leaf assembly in Morton order (bvh.py:168-181), records, host copies
  // (codes_in reused as the ids' order is ids_out)
  device_scan<int>(LeafStartIn{is_left}, LeafOut{is_left, ids_out, first_d, leaf_tris_d, prim_d, m, L, counters + 3},
                   m, OpAdd{}, 0, reinterpret_cast<int*>(base + w.aggr), s);
  {
    unsigned long long bad = 0;
    uint32_t last = 0;
    GD_CUDA(cudaMemcpyAsync(&bad, counters + 3, sizeof bad, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaMemcpyAsync(&last, first_d + L, sizeof last, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
    GD_CHECK(bad == 0 && last == (uint32_t)m, GD_ERR_INVALID, "internal: pairing produced a wrong leaf count");
  }
  k_leaf_rec<<<(unsigned)((L + 255) / 256), 256, 0, s>>>(mesh, ids_out, first_d, L, reinterpret_cast<int4*>(T.leaf_rec));
  GD_CUDA(cudaMemcpyAsync(prim_order_host, prim_d, m * sizeof(long long), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(leaf_tris_host, leaf_tris_d, 2 * L * sizeof(long long), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaGetLastError());
  clk.mark("leaf assembly + records");
  bvh_layout(mesh, T, ws, ws_bytes, s);  // reuses the workspace (stream-ordered)
  clk.mark("vertex layout + staging");
  refit(mesh, T, s);
  GD_CUDA(cudaStreamSynchronize(s));
  clk.mark("refit");
}

}  // namespace gd
