// batch.cu -- batch entry points of bounds.py and the device brute force
// (query.py:571-619).  Exact kernels use the reference's arithmetic order.
#include "engine.cuh"

namespace gd {

template <typename T>
__device__ __forceinline__ Tri<T> load_tri_aos(const T* p, long long i) {
  const T* q = p + 9 * i;
  Tri<T> t;
#pragma unroll
  for (int c = 0; c < 3; ++c) t.v[c] = {q[3 * c], q[3 * c + 1], q[3 * c + 2]};
  return t;
}

template <typename T, bool kMax>
__global__ void k_tri_tri_exact(const T* t1, const T* t2, long long n, T* d, T* p, T* q) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= n) return;
  Tri<T> a = load_tri_aos(t1, i), b = load_tri_aos(t2, i);
  V3<T> P, Q;
  T d2 = kMax ? tri_tri_max_d2<Exact<T>, T, true>(a, b, &P, &Q) : tri_tri_min_d2<Exact<T>, T, true>(a, b, &P, &Q);
  d[i] = Exact<T>::sqrt(d2);
  p[3 * i] = P.x; p[3 * i + 1] = P.y; p[3 * i + 2] = P.z;
  q[3 * i] = Q.x; q[3 * i + 1] = Q.y; q[3 * i + 2] = Q.z;
}

template <bool kMax>
__global__ void k_tri_tri_fast(const float* t1, const float* t2, long long n, float* d) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= n) return;
  Tri<float> a = load_tri_aos(t1, i), b = load_tri_aos(t2, i);
  d[i] = sqrtf(kMax ? tri_tri_max_d2<Fast<float>, float, false>(a, b, nullptr, nullptr)
                    : tri_tri_min_d2<Fast<float>, float, false>(a, b, nullptr, nullptr));
}

// exact closed forms of bounds.py:47-101 (see DESIGN.md "Enhanced bounds":
// equal to the 36 face-pair evaluation because every per-axis term of a
// face pair depends on at most one face side and rounding is monotone)
template <typename T>
__device__ __forceinline__ T sum3(T a, T b, T c) {
  using E = Exact<T>;
  return E::add(E::add(a, b), c);
}
template <typename T>
__device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }
template <typename T>
__device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <typename T>
__device__ __forceinline__ T tabs(T a) { return a < T(0) ? -a : a; }

template <typename T>
__global__ void k_box_bounds(int which, const T* amin, const T* amax, const T* bmin, const T* bmax, long long n,
                             T* out) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= n) return;
  using E = Exact<T>;
  T al[3], ah[3], bl[3], bh[3];
  for (int k = 0; k < 3; ++k) {
    al[k] = amin[3 * i + k];
    ah[k] = amax[3 * i + k];
    bl[k] = bmin[3 * i + k];
    bh[k] = bmax[3 * i + k];
  }
  T r;
  if (which == 0) {  // batch_min_lower
    T g[3];
    for (int k = 0; k < 3; ++k) {
      g[k] = tmax(E::sub(al[k], bh[k]), E::sub(bl[k], ah[k]));
      g[k] = tmax(g[k], T(0));
      g[k] = E::mul(g[k], g[k]);
    }
    r = E::sqrt(sum3(g[0], g[1], g[2]));
  } else if (which == 1) {  // batch_max_upper
    T h[3];
    for (int k = 0; k < 3; ++k) {
      h[k] = tmax(tabs(E::sub(al[k], bh[k])), tabs(E::sub(ah[k], bl[k])));
      h[k] = E::mul(h[k], h[k]);
    }
    r = E::sqrt(sum3(h[0], h[1], h[2]));
  } else if (which == 2) {  // batch_enhanced_min_upper
    T H[3], PA[3], PB[3], PP[3];
    for (int k = 0; k < 3; ++k) {
      const T ll = tabs(E::sub(al[k], bl[k])), lh = tabs(E::sub(al[k], bh[k]));
      const T hl = tabs(E::sub(ah[k], bl[k])), hh = tabs(E::sub(ah[k], bh[k]));
      const T h = tmax(lh, tabs(E::sub(ah[k], bl[k])));
      H[k] = E::mul(h, h);
      const T pa = tmin(tmax(ll, lh), tmax(hl, hh));
      const T pb = tmin(tmax(ll, hl), tmax(lh, hh));
      const T pp = tmin(tmin(ll, lh), tmin(hl, hh));
      PA[k] = E::mul(pa, pa);
      PB[k] = E::mul(pb, pb);
      PP[k] = E::mul(pp, pp);
    }
    T b = sum3(PP[0], H[1], H[2]);
    b = tmin(b, sum3(H[0], PP[1], H[2]));
    b = tmin(b, sum3(H[0], H[1], PP[2]));
    b = tmin(b, sum3(PA[0], PB[1], H[2]));
    b = tmin(b, sum3(PA[0], H[1], PB[2]));
    b = tmin(b, sum3(PB[0], PA[1], H[2]));
    b = tmin(b, sum3(H[0], PA[1], PB[2]));
    b = tmin(b, sum3(PB[0], H[1], PA[2]));
    b = tmin(b, sum3(H[0], PB[1], PA[2]));
    r = E::sqrt(b);
  } else {  // batch_enhanced_max_lower
    T G[3], QA[3], QB[3], QQ[3];
    for (int k = 0; k < 3; ++k) {
      T g = tmax(tmax(E::sub(al[k], bh[k]), E::sub(bl[k], ah[k])), T(0));
      G[k] = E::mul(g, g);
      // point a_s against interval B: max(bmin - a, a - bmax, 0); best side
      const T qa0 = tmax(tmax(E::sub(bl[k], al[k]), E::sub(al[k], bh[k])), T(0));
      const T qa1 = tmax(tmax(E::sub(bl[k], ah[k]), E::sub(ah[k], bh[k])), T(0));
      const T qb0 = tmax(tmax(E::sub(al[k], bl[k]), E::sub(bl[k], ah[k])), T(0));
      const T qb1 = tmax(tmax(E::sub(al[k], bh[k]), E::sub(bh[k], ah[k])), T(0));
      const T qa = tmax(qa0, qa1), qb = tmax(qb0, qb1);
      const T qq = tmax(tmax(tabs(E::sub(al[k], bl[k])), tabs(E::sub(al[k], bh[k]))),
                        tmax(tabs(E::sub(ah[k], bl[k])), tabs(E::sub(ah[k], bh[k]))));
      QA[k] = E::mul(qa, qa);
      QB[k] = E::mul(qb, qb);
      QQ[k] = E::mul(qq, qq);
    }
    T b = sum3(QQ[0], G[1], G[2]);
    b = tmax(b, sum3(G[0], QQ[1], G[2]));
    b = tmax(b, sum3(G[0], G[1], QQ[2]));
    b = tmax(b, sum3(QA[0], QB[1], G[2]));
    b = tmax(b, sum3(QA[0], G[1], QB[2]));
    b = tmax(b, sum3(QB[0], QA[1], G[2]));
    b = tmax(b, sum3(G[0], QA[1], QB[2]));
    b = tmax(b, sum3(QB[0], G[1], QA[2]));
    b = tmax(b, sum3(G[0], QB[1], QA[2]));
    r = E::sqrt(b);
  }
  out[i] = r;
}

// all-pairs exact oracle on the device, lexicographic (d, i, j) key
template <typename T, bool kMax>
__global__ __launch_bounds__(256) void k_brute(const T* pa, long long ma, const T* pb, long long mb, Key128* best) {
  __shared__ Key128 wk[8];
  Key128 mine;
  mine.hi = ~0ull;
  mine.lo = ~0ull;
  const long long total = ma * mb;
  for (long long t = blockIdx.x * 256ll + threadIdx.x; t < total; t += gridDim.x * 256ll) {
    const long long i = t / mb, j = t % mb;
    Tri<T> a = load_tri_aos(pa, i), b = load_tri_aos(pb, j);
    T d2 = kMax ? tri_tri_max_d2<Exact<T>, T, false>(a, b, nullptr, nullptr)
                : tri_tri_min_d2<Exact<T>, T, false>(a, b, nullptr, nullptr);
    const double d = (double)Exact<T>::sqrt(d2);
    const unsigned long long bits = (unsigned long long)__double_as_longlong(d);
    Key128 k;
    k.hi = kMax ? ~bits : bits;
    k.lo = ((unsigned long long)i << 32) | (unsigned long long)j;
    if (key_less(k, mine)) mine = k;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key128 other;
    other.hi = __shfl_xor_sync(0xffffffffu, mine.hi, o);
    other.lo = __shfl_xor_sync(0xffffffffu, mine.lo, o);
    if (key_less(other, mine)) mine = other;
  }
  if ((threadIdx.x & 31) == 0) wk[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w)
      if (key_less(wk[w], mine)) mine = wk[w];
    atomic_min_key(best, mine);
  }
}

template <typename T, bool kMax>
__global__ void k_brute_final(const T* pa, const T* pb, const Key128* best, GdResult* out) {
  if (threadIdx.x != 0) return;
  GdResult r;
  memset(&r, 0, sizeof(r));
  const unsigned long long bits = kMax ? ~best->hi : best->hi;
  r.distance = __longlong_as_double((long long)bits);
  r.witness_distance = r.distance;
  r.tri_a = (long long)(best->lo >> 32);
  r.tri_b = (long long)(best->lo & 0xffffffffu);
  Tri<T> a = load_tri_aos(pa, r.tri_a), b = load_tri_aos(pb, r.tri_b);
  V3<T> P, Q;
  if (kMax)
    tri_tri_max_d2<Exact<T>, T, true>(a, b, &P, &Q);
  else
    tri_tri_min_d2<Exact<T>, T, true>(a, b, &P, &Q);
  r.point_a[0] = P.x; r.point_a[1] = P.y; r.point_a[2] = P.z;
  r.point_b[0] = Q.x; r.point_b[1] = Q.y; r.point_b[2] = Q.z;
  *out = r;
}

__global__ void k_key_init(Key128* k) {
  k->hi = ~0ull;
  k->lo = ~0ull;
}

// ---------------------------------------------------------------------------
static unsigned blocks_for(long long n) { return (unsigned)((n + 255) / 256); }

void tri_tri_batch(int kind, int precision, const void* t1, const void* t2, int64_t n, void* d, void* p, void* q,
                   cudaStream_t s) {
  GD_CHECK(kind == 0 || kind == 1, GD_ERR_INVALID, "kind must be 0 (min) or 1 (max)");
  GD_CHECK(precision == 32 || precision == 64, GD_ERR_CONFIG, "precision must be 32 or 64");
  if (n <= 0) return;
  if (precision == 64) {
    if (kind)
      k_tri_tri_exact<double, true><<<blocks_for(n), 256, 0, s>>>((const double*)t1, (const double*)t2, n,
                                                                 (double*)d, (double*)p, (double*)q);
    else
      k_tri_tri_exact<double, false><<<blocks_for(n), 256, 0, s>>>((const double*)t1, (const double*)t2, n,
                                                                  (double*)d, (double*)p, (double*)q);
  } else {
    if (kind)
      k_tri_tri_exact<float, true><<<blocks_for(n), 256, 0, s>>>((const float*)t1, (const float*)t2, n, (float*)d,
                                                                (float*)p, (float*)q);
    else
      k_tri_tri_exact<float, false><<<blocks_for(n), 256, 0, s>>>((const float*)t1, (const float*)t2, n, (float*)d,
                                                                 (float*)p, (float*)q);
  }
  GD_CUDA(cudaGetLastError());
}

// the conditioning-aware lower bound of the float32 min distance
// (geometry.cuh tri_tri_min_fast_lb): kind 2 of gd_tri_tri_fast
__global__ void k_tri_tri_fast_lb(const float* t1, const float* t2, long long n, float* d) {
  const long long i = blockIdx.x * 256ll + threadIdx.x;
  if (i >= n) return;
  Tri<float> a = load_tri_aos(t1, i), b = load_tri_aos(t2, i);
  float dd, lb;
  tri_tri_min_fast_lb(a, b, dd, lb);
  d[i] = lb;
}

void tri_tri_fast(int kind, const float* t1, const float* t2, int64_t n, float* d, cudaStream_t s) {
  GD_CHECK(kind >= 0 && kind <= 2, GD_ERR_INVALID, "kind must be 0 (min), 1 (max) or 2 (min lower bound)");
  if (n <= 0) return;
  if (kind == 2)
    k_tri_tri_fast_lb<<<blocks_for(n), 256, 0, s>>>(t1, t2, n, d);
  else if (kind)
    k_tri_tri_fast<true><<<blocks_for(n), 256, 0, s>>>(t1, t2, n, d);
  else
    k_tri_tri_fast<false><<<blocks_for(n), 256, 0, s>>>(t1, t2, n, d);
  GD_CUDA(cudaGetLastError());
}

void box_bounds_batch(int which, int precision, const void* amin, const void* amax, const void* bmin,
                      const void* bmax, int64_t n, void* out, cudaStream_t s) {
  GD_CHECK(which >= 0 && which <= 3, GD_ERR_INVALID, "which must be 0..3");
  GD_CHECK(precision == 32 || precision == 64, GD_ERR_CONFIG, "precision must be 32 or 64");
  if (n <= 0) return;
  if (precision == 64)
    k_box_bounds<double><<<blocks_for(n), 256, 0, s>>>(which, (const double*)amin, (const double*)amax,
                                                       (const double*)bmin, (const double*)bmax, n, (double*)out);
  else
    k_box_bounds<float><<<blocks_for(n), 256, 0, s>>>(which, (const float*)amin, (const float*)amax,
                                                      (const float*)bmin, (const float*)bmax, n, (float*)out);
  GD_CUDA(cudaGetLastError());
}

void brute_force(int kind, int precision, const void* pa, int64_t ma, const void* pb, int64_t mb, GdResult* out,
                 cudaStream_t s) {
  GD_CHECK(ma > 0 && mb > 0, GD_ERR_INVALID, "both meshes need at least one triangle");
  GD_CHECK(ma < (1ll << 31) && mb < (1ll << 31), GD_ERR_INVALID, "mesh too large");
  Key128* key = nullptr;
  GdResult* dres = nullptr;
  GD_CUDA(cudaMallocAsync((void**)&key, sizeof(Key128), s));
  GD_CUDA(cudaMallocAsync((void**)&dres, sizeof(GdResult), s));
  k_key_init<<<1, 1, 0, s>>>(key);
  const unsigned g = (unsigned)(num_sms() * 8);
#define GD_BRUTE(T, M)                                                                     \
  k_brute<T, M><<<g, 256, 0, s>>>((const T*)pa, ma, (const T*)pb, mb, key);               \
  k_brute_final<T, M><<<1, 32, 0, s>>>((const T*)pa, (const T*)pb, key, dres);
  if (precision == 64) {
    if (kind) {
      GD_BRUTE(double, true)
    } else {
      GD_BRUTE(double, false)
    }
  } else {
    if (kind) {
      GD_BRUTE(float, true)
    } else {
      GD_BRUTE(float, false)
    }
  }
#undef GD_BRUTE
  GD_CUDA(cudaGetLastError());
  GD_CUDA(cudaMemcpyAsync(out, dres, sizeof(GdResult), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaFreeAsync(key, s));
  GD_CUDA(cudaFreeAsync(dres, s));
  GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gd
