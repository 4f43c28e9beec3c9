// sort.cu -- the repo's stable LSD radix sort (primitives.cuh): Morton codes
// (63-bit keys) and the build's other (key, index) sorts.
#include "primitives.cuh"

namespace gd {

namespace {

struct HistIn {
  const unsigned* h;
  __device__ __forceinline__ unsigned operator()(long long i) const { return h[i]; }
};
struct HistExclusiveOut {
  unsigned* h;
  __device__ __forceinline__ void operator()(long long i, unsigned inc, unsigned v) const { h[i] = inc - v; }
};

long long rs_tiles(long long n) { return (n + kRsTile - 1) / kRsTile; }

template <typename K>
void sort_impl(const K* k_in, const int32_t* v_in, K* k_tmp, int32_t* v_tmp, K* k_out, int32_t* v_out, long long n,
               int bits, void* ws, cudaStream_t s) {
  GD_CHECK(n >= 0 && n < (1ll << 31), GD_ERR_INVALID, "radix sort: n out of range");
  GD_CHECK(bits >= 1 && bits <= (int)(8 * sizeof(K)), GD_ERR_INVALID, "radix sort: bad key width");
  const int passes = (bits + 7) / 8;
  if (n == 0) return;
  const long long tiles = rs_tiles(n);
  unsigned* hist = static_cast<unsigned*>(ws);
  unsigned* aggr = hist + 256 * tiles;
  // ping-pong so that the last pass lands in k_out: pass p reads src, writes dst
  const K* src_k = k_in;
  const int32_t* src_v = v_in;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    K* dk = to_out ? k_out : k_tmp;
    int32_t* dv = to_out ? v_out : v_tmp;
    k_rs_hist<K><<<(unsigned)tiles, kRsThreads, 0, s>>>(src_k, n, 8 * p, hist, (unsigned)tiles);
    device_scan<unsigned>(HistIn{hist}, HistExclusiveOut{hist}, 256 * tiles, OpAdd{}, 0u, aggr, s);
    k_rs_scatter<K><<<(unsigned)tiles, kRsThreads, 0, s>>>(src_k, src_v, dk, dv, n, 8 * p, hist, (unsigned)tiles);
    GD_CUDA(cudaGetLastError());
    src_k = dk;
    src_v = dv;
  }
  count_launches(4ll * passes);
}

}  // namespace

size_t radix_sort_ws_bytes(long long n) {
  const long long tiles = rs_tiles(std::max(n, 1ll));
  return (size_t)(256 * tiles + scan_tiles(256 * tiles)) * sizeof(unsigned) + 256;
}

void radix_sort_pairs(const unsigned long long* k_in, const int32_t* v_in, unsigned long long* k_tmp, int32_t* v_tmp,
                      unsigned long long* k_out,
                      int32_t* v_out, long long n, int bits, void* ws, cudaStream_t s) {
  sort_impl<unsigned long long>(k_in, v_in, k_tmp, v_tmp, k_out, v_out, n, bits, ws, s);
}

void radix_sort_pairs(const uint32_t* k_in, const int32_t* v_in, uint32_t* k_tmp, int32_t* v_tmp, uint32_t* k_out,
                      int32_t* v_out, long long n, int bits, void* ws, cudaStream_t s) {
  sort_impl<unsigned>(k_in, v_in, k_tmp, v_tmp, k_out, v_out, n, bits, ws, s);
}

}  // namespace gd
