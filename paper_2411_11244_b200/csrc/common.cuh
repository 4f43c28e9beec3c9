// common.cuh -- shared device helpers for libgdist (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/gdist.h"

namespace gd {

// ---------------------------------------------------------------------------
// error plumbing (host)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
void count_launches(long long n);  // hot-path kernel launches (bench evidence)
struct Failure {
  int status;
  std::string msg;
};
#define GD_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw ::gd::Failure{GD_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)}; \
  } while (0)
#define GD_CHECK(cond, code, msg)                 \
  do {                                            \
    if (!(cond)) throw ::gd::Failure{code, msg}; \
  } while (0)

// per-device launch caches (one host process may drive several GPUs)
constexpr int kMaxDevices = 64;
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < kMaxDevices ? dev : kMaxDevices - 1;
}
inline int num_sms() {
  static int sms[kMaxDevices] = {0};
  const int dev = current_device();
  if (sms[dev] <= 0 && cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    sms[dev] = 148;
  return sms[dev];
}

// ---------------------------------------------------------------------------
// IEEE round-to-nearest arithmetic without FMA contraction.  Used wherever the
// result must equal numpy's elementwise float32/float64 arithmetic bit for bit.
// ---------------------------------------------------------------------------
template <typename T> struct Exact;
template <> struct Exact<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt(double a) { return __dsqrt_rn(a); }
};
template <> struct Exact<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float sqrt(float a) { return __fsqrt_rn(a); }
};
// Fast arithmetic: plain operators, the compiler may contract to FMA.
template <typename T> struct Fast {
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
  static __device__ __forceinline__ T sub(T a, T b) { return a - b; }
  static __device__ __forceinline__ T mul(T a, T b) { return a * b; }
  // approximate division (MUFU.RCP based): the float32 filter's error budget
  // absorbs its 2-ulp error on clamped parameters
  static __device__ __forceinline__ T div(T a, T b) { return fast_div(a, b); }
  static __device__ __forceinline__ float fast_div(float a, float b) { return __fdividef(a, b); }
  static __device__ __forceinline__ double fast_div(double a, double b) { return a / b; }
  static __device__ __forceinline__ T sqrt(T a) { return ::sqrt(a); }
};

template <typename T> struct V3 {
  T x, y, z;
};

template <typename A, typename T>
__device__ __forceinline__ V3<T> vsub(V3<T> a, V3<T> b) {
  return {A::sub(a.x, b.x), A::sub(a.y, b.y), A::sub(a.z, b.z)};
}
// ((ax*bx + ay*by) + az*bz): numpy's length-3 reduction order
template <typename A, typename T>
__device__ __forceinline__ T vdot(V3<T> a, V3<T> b) {
  return A::add(A::add(A::mul(a.x, b.x), A::mul(a.y, b.y)), A::mul(a.z, b.z));
}
// p + t*u
template <typename A, typename T>
__device__ __forceinline__ V3<T> vmadd(V3<T> p, T t, V3<T> u) {
  return {A::add(p.x, A::mul(t, u.x)), A::add(p.y, A::mul(t, u.y)), A::add(p.z, A::mul(t, u.z))};
}
// numpy.cross order
template <typename A, typename T>
__device__ __forceinline__ V3<T> vcross(V3<T> a, V3<T> b) {
  return {A::sub(A::mul(a.y, b.z), A::mul(a.z, b.y)), A::sub(A::mul(a.z, b.x), A::mul(a.x, b.z)),
          A::sub(A::mul(a.x, b.y), A::mul(a.y, b.x))};
}
template <typename T>
__device__ __forceinline__ V3<T> vsel(bool c, V3<T> a, V3<T> b) {
  return {c ? a.x : b.x, c ? a.y : b.y, c ? a.z : b.z};
}

// ---------------------------------------------------------------------------
// ordered-bit atomics for non-negative floats: for x >= 0 the IEEE bit
// pattern is monotone, so unsigned min/max on the bits is float min/max.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void atomic_min_pos(unsigned int* cell, float v) {
  atomicMin(cell, __float_as_uint(fmaxf(v, 0.0f)));
}
__device__ __forceinline__ void atomic_max_pos(unsigned int* cell, float v) {
  atomicMax(cell, __float_as_uint(fmaxf(v, 0.0f)));
}

// NaN-propagating float32 min / max (PTX min.NaN / max.NaN): the box
// unions of numpy's np.minimum / np.maximum, which the reference's boxes use
// (bvh.py:242-264) -- a NaN coordinate poisons every box above it, up to the
// root, so a query over it culls everything and returns NaN as the
// reference's does.  fminf / fmaxf would silently drop the NaN.
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float d;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may be scheduled while
// its predecessor in the stream drains; it waits here, before touching the
// predecessor's results, until that grid has completed and its writes are
// visible.  A no-op for a normal launch.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 128-bit lexicographic key (hi, lo) and an atomic minimum on it.
struct alignas(16) Key128 {
  unsigned long long hi, lo;
};
__device__ __forceinline__ bool key_less(const Key128& a, const Key128& b) {
  return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
__device__ __forceinline__ void atomic_min_key(Key128* cell, Key128 v) {
  Key128 cur;
  cur.hi = reinterpret_cast<volatile unsigned long long*>(cell)[0];
  cur.lo = reinterpret_cast<volatile unsigned long long*>(cell)[1];
  while (key_less(v, cur)) {
    Key128 prev = atomicCAS(cell, cur, v);
    if (prev.hi == cur.hi && prev.lo == cur.lo) break;
    cur = prev;
  }
}

// warp / block reductions ----------------------------------------------------
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace gd
