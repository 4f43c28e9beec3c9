// abi.cpp -- extern "C" boundary of libgdist.so (include/gdist.h).
// Every entry point converts exceptions into a GdStatus + thread-local
// message; nothing C++ crosses the ABI.
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <string>

#include "engine.cuh"

namespace gd {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
static std::atomic<long long> g_launches{0};
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void set_profiling(int on);
int phase_ms(float* out, int n);

size_t build_workspace_size(int64_t m, int64_t nv);
int build_pairing_mode();
void bvh_layout(const GdMesh& mesh, GdBvh& T, void* ws, size_t ws_bytes, cudaStream_t s);
void bvh_build(const GdMesh& mesh, GdBvh& T, void* ws, size_t ws_bytes, int64_t* prim_order_host,
               int64_t* leaf_tris_host, cudaStream_t s);
void refit(const GdMesh& m, const GdBvh& T, cudaStream_t s);
void stage_vertices(const GdMesh& m, const GdBvh& T, cudaStream_t s);
void export_boxes(const GdMesh& m, const GdBvh& B, int precision, void* nmin, void* nmax, cudaStream_t s);
void pair_greedy(const double* sa, int64_t n, uint8_t* is_left);
size_t query_workspace_size(const GdConfig& cfg);
void query_async(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                 void* ws, size_t ws_bytes, GdResult* result_dev, cudaStream_t s, cudaEvent_t traversal_done,
                 int round = 0);
void query_traverse(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                    void* ws, size_t ws_bytes, int round, int budget, cudaStream_t s);
void query_finish(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                  void* ws, size_t ws_bytes, GdResult* result_dev, cudaStream_t s);
void query_round(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg, void* ws,
                 size_t ws_bytes, GdResult* result_dev, cudaStream_t s, int round);
void query_group_async(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, int n,
                       const GdConfig* cfgs, void* const* wss, const size_t* ws_bytes, void* const* host_dst,
                       int max_stats, cudaStream_t s, cudaEvent_t traversal_done, bool external_record);
void* frame_graph_create(const GdMesh& ma, const GdMesh& mb, const GdBvh& A, const GdBvh& B, int n_queries,
                         const GdConfig* cfgs, void* const* wss, const size_t* ws_bytes, void* const* host_dst,
                         int max_stats, int refit_a, int refit_b, cudaEvent_t wait_before,
                         cudaEvent_t traversal_done);
void frame_graph_launch(void* h, const GdMesh& ma, const GdMesh& mb, cudaStream_t s);
void frame_graph_destroy(void* h);
const void* query_result_device(const GdConfig& cfg, void* ws);
void* query_bound_device(const GdConfig& cfg, void* ws);
void query_result_async(const GdConfig& cfg, void* ws, void* host_dst, int max_stats, cudaStream_t s);
void query_collect(const GdConfig& cfg, void* ws, const GdResult* result_dev, GdResult* out, GdIterStat* stats,
                   int max_stats, cudaStream_t s);
void dfs_query(const GdMesh& ma, const GdMesh& mb, const GdBvh& b, const GdConfig& cfg, void* ws, size_t ws_bytes,
               GdResult* out, int64_t* visited, cudaStream_t s);
void tri_tri_batch(int kind, int precision, const void* t1, const void* t2, int64_t n, void* d, void* p, void* q,
                   cudaStream_t s);
void tri_tri_fast(int kind, const float* t1, const float* t2, int64_t n, float* d, cudaStream_t s);
void box_bounds_batch(int which, int precision, const void* amin, const void* amax, const void* bmin,
                      const void* bmax, int64_t n, void* out, cudaStream_t s);
void brute_force(int kind, int precision, const void* pa, int64_t ma, const void* pb, int64_t mb, GdResult* out,
                 cudaStream_t s);

template <typename F>
static int guarded(F&& f) {
  try {
    f();
    return GD_OK;
  } catch (const Failure& e) {
    set_error(e.msg);
    return e.status;
  } catch (const std::exception& e) {
    set_error(std::string("internal error: ") + e.what());
    return GD_ERR_INVALID;
  } catch (...) {
    set_error("internal error");
    return GD_ERR_INVALID;
  }
}

static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace gd

using namespace gd;

extern "C" {

const char* gd_version(void) { return "gdist-b200 0.1.0 (sm_100a)"; }
const char* gd_last_error(void) { return g_last_error.c_str(); }
int gd_abi_version(void) { return GDIST_ABI_VERSION; }

long long gd_launch_count(void) { return g_launches.load(); }

int gd_set_profiling(int enable) {
  return guarded([&] { set_profiling(enable); });
}

int gd_query_phase_ms(float* out, int n) {
  int got = 0;
  int st = guarded([&] {
    GD_CHECK(out && n > 0, GD_ERR_INVALID, "bad arguments");
    got = phase_ms(out, n);
  });
  return st == GD_OK ? got : -st;
}

int gd_device_count(int* count) {
  return guarded([&] {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

int gd_bvh_sizes(int64_t m, int64_t nv, GdBvhSizes* out) {
  return guarded([&] {
    GD_CHECK(m >= 1, GD_ERR_INVALID, "cannot build a BVH over an empty mesh");
    GD_CHECK(nv >= 0, GD_ERR_INVALID, "negative vertex count");
    int64_t L = 1;
    int d = 0;
    while (L * 2 <= m) {
      L *= 2;
      ++d;
    }
    out->leaf_count = L;
    out->n_nodes = 2 * L - 1;
    out->depth = d;
    out->_pad = 0;
    out->build_workspace_bytes = build_workspace_size(m, nv);
  });
}

int gd_bvh_build(const GdMesh* mesh, GdBvh* bvh, void* workspace, size_t workspace_bytes, int64_t* prim_order_host,
                 int64_t* leaf_tris_host, void* stream) {
  return guarded([&] {
    GD_CHECK(mesh && bvh && prim_order_host && leaf_tris_host, GD_ERR_INVALID, "null argument");
    bvh_build(*mesh, *bvh, workspace, workspace_bytes, prim_order_host, leaf_tris_host, S(stream));
  });
}

int gd_build_pairing_mode(void) { return gd::build_pairing_mode(); }

int gd_bvh_layout(const GdMesh* mesh, GdBvh* bvh, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    GD_CHECK(mesh && bvh, GD_ERR_INVALID, "null argument");
    bvh_layout(*mesh, *bvh, workspace, workspace_bytes, S(stream));
  });
}

int gd_mesh_relative(const GdMesh* a, const GdMesh* b, GdMesh* out) {
  return guarded([&] {
    GD_CHECK(a && b && out, GD_ERR_INVALID, "null argument");
    *out = relative_mesh(*a, *b);
  });
}

int gd_stage_vertices(const GdMesh* mesh, GdBvh* bvh, void* stream) {
  return guarded([&] {
    GD_CHECK(mesh && bvh, GD_ERR_INVALID, "null argument");
    stage_vertices(*mesh, *bvh, S(stream));
  });
}

int gd_refit(const GdMesh* mesh, GdBvh* bvh, void* stream) {
  return guarded([&] {
    GD_CHECK(mesh && bvh, GD_ERR_INVALID, "null argument");
    refit(*mesh, *bvh, S(stream));
  });
}

int gd_export_boxes(const GdMesh* mesh, const GdBvh* bvh, int precision, void* node_min, void* node_max,
                    void* stream) {
  return guarded([&] {
    GD_CHECK(mesh && bvh && node_min && node_max, GD_ERR_INVALID, "null argument");
    export_boxes(*mesh, *bvh, precision, node_min, node_max, S(stream));
  });
}

int gd_pair_greedy(const double* sa_host, int64_t n, uint8_t* is_left_host) {
  return guarded([&] {
    GD_CHECK(n >= 0 && (n < 2 || sa_host) && is_left_host, GD_ERR_INVALID, "bad arguments");
    pair_greedy(sa_host, n, is_left_host);
  });
}

int gd_query_workspace_size(const GdBvh* a, const GdBvh* b, const GdConfig* cfg, size_t* bytes) {
  return guarded([&] {
    GD_CHECK(cfg && bytes, GD_ERR_INVALID, "null argument");
    (void)a;
    (void)b;
    *bytes = query_workspace_size(*cfg);
  });
}

int gd_query(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b, const GdConfig* cfg,
             void* workspace, size_t workspace_bytes, GdResult* out, GdIterStat* stats, int max_stats,
             void* stream) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && a && b && cfg && out, GD_ERR_INVALID, "null argument");
    query_async(*mesh_a, *mesh_b, *a, *b, *cfg, workspace, workspace_bytes, nullptr, S(stream), nullptr);
    query_collect(*cfg, workspace, nullptr, out, stats, max_stats, S(stream));
    // a front larger than the arena: one more round per leaf chunk; a band
    // overflow: the rescan pass (query_round decides)
    while (out->pending && out->status == 0) {
      query_round(*mesh_a, *mesh_b, *a, *b, *cfg, workspace, workspace_bytes, nullptr, S(stream),
                  out->rounds > 0 ? out->rounds : 1);
      query_collect(*cfg, workspace, nullptr, out, stats, max_stats, S(stream));
    }
    if (out->status == GD_ERR_WORKSPACE)
      throw Failure{GD_ERR_WORKSPACE, "front arena too small (GdConfig.arena_entries)"};
    if (out->status == GD_ERR_FRONT_OVERFLOW)
      throw Failure{GD_ERR_FRONT_OVERFLOW, "front expansion would create " + std::to_string(out->overflow_candidates) +
                                               " candidate pairs from " + std::to_string(out->overflow_front_in) +
                                               " entries, exceeding the hard cap of " +
                                               std::to_string(out->overflow_cap)};
  });
}

int gd_query_async(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b, const GdConfig* cfg,
                   void* workspace, size_t workspace_bytes, GdResult* result_dev, void* stream) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && a && b && cfg, GD_ERR_INVALID, "null argument");
    query_async(*mesh_a, *mesh_b, *a, *b, *cfg, workspace, workspace_bytes, result_dev, S(stream), nullptr);
  });
}

int gd_query_round(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b, const GdConfig* cfg,
                   void* workspace, size_t workspace_bytes, int round, void* stream) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && a && b && cfg, GD_ERR_INVALID, "null argument");
    GD_CHECK(round >= 1, GD_ERR_INVALID, "gd_query_round resumes a query: round must be >= 1");
    query_round(*mesh_a, *mesh_b, *a, *b, *cfg, workspace, workspace_bytes, nullptr, S(stream), round);
  });
}

int gd_query_async_ev(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                      const GdConfig* cfg, void* workspace, size_t workspace_bytes, GdResult* result_dev,
                      void* stream, void* traversal_done) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && a && b && cfg, GD_ERR_INVALID, "null argument");
    query_async(*mesh_a, *mesh_b, *a, *b, *cfg, workspace, workspace_bytes, result_dev, S(stream),
                static_cast<cudaEvent_t>(traversal_done));
  });
}

int gd_query_traverse(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                      const GdConfig* cfg, void* workspace, size_t workspace_bytes, int round, int sweep_budget,
                      void* stream) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && a && b && cfg, GD_ERR_INVALID, "null argument");
    query_traverse(*mesh_a, *mesh_b, *a, *b, *cfg, workspace, workspace_bytes, round, sweep_budget, S(stream));
  });
}

int gd_query_finish(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                    const GdConfig* cfg, void* workspace, size_t workspace_bytes, GdResult* result_dev,
                    void* stream) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && a && b && cfg, GD_ERR_INVALID, "null argument");
    query_finish(*mesh_a, *mesh_b, *a, *b, *cfg, workspace, workspace_bytes, result_dev, S(stream));
  });
}

int gd_query_group_async(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b, int n,
                         const GdConfig* cfgs, void* const* workspaces, const size_t* workspace_bytes,
                         void* const* host_dst, int max_stats, void* stream, void* traversal_done) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && a && b && cfgs && workspaces && workspace_bytes, GD_ERR_INVALID, "null argument");
    query_group_async(*mesh_a, *mesh_b, *a, *b, n, cfgs, workspaces, workspace_bytes, host_dst, max_stats,
                      S(stream), static_cast<cudaEvent_t>(traversal_done), false);
  });
}

int gd_frame_graph_create(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                          int n_queries, const GdConfig* cfgs, void* const* workspaces,
                          const size_t* workspace_bytes, void* const* host_dst, int max_stats, int refit_a,
                          int refit_b, void* wait_before, void* traversal_done, void** graph_out) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && a && b && graph_out && (n_queries == 0 || (cfgs && workspaces && workspace_bytes)),
             GD_ERR_INVALID, "null argument");
    *graph_out = frame_graph_create(*mesh_a, *mesh_b, *a, *b, n_queries, cfgs, workspaces, workspace_bytes,
                                    host_dst, max_stats, refit_a, refit_b, static_cast<cudaEvent_t>(wait_before),
                                    static_cast<cudaEvent_t>(traversal_done));
  });
}

int gd_frame_graph_launch(void* graph, const GdMesh* mesh_a, const GdMesh* mesh_b, void* stream) {
  return guarded([&] {
    GD_CHECK(graph && mesh_a && mesh_b, GD_ERR_INVALID, "null argument");
    frame_graph_launch(graph, *mesh_a, *mesh_b, S(stream));
  });
}

int gd_frame_graph_destroy(void* graph) {
  return guarded([&] { frame_graph_destroy(graph); });
}

int gd_query_result_async(const GdConfig* cfg, void* workspace, void* host_dst, int max_stats, void* stream) {
  return guarded([&] {
    GD_CHECK(cfg && workspace && host_dst, GD_ERR_INVALID, "null argument");
    query_result_async(*cfg, workspace, host_dst, max_stats, S(stream));
  });
}

int gd_query_result_device(const GdConfig* cfg, void* workspace, const void** out) {
  return guarded([&] {
    GD_CHECK(cfg && workspace && out, GD_ERR_INVALID, "null argument");
    *out = query_result_device(*cfg, workspace);
  });
}

int gd_query_bound_device(const GdConfig* cfg, void* workspace, void** out) {
  return guarded([&] {
    GD_CHECK(cfg && workspace && out, GD_ERR_INVALID, "null argument");
    *out = query_bound_device(*cfg, workspace);
  });
}

// cuMemGetAddressRange through the runtime's driver entry point (no libcuda
// link dependency): the base of the allocation a pointer lies in
typedef int (*AddressRangeFn)(unsigned long long*, size_t*, unsigned long long);

int gd_ipc_handle(const void* ptr, void* handle_out, uint64_t* offset) {
  return guarded([&] {
    GD_CHECK(ptr && handle_out && offset, GD_ERR_INVALID, "null argument");
    static AddressRangeFn range = nullptr;
    if (!range) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      GD_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
      GD_CHECK(fn && q == cudaDriverEntryPointSuccess, GD_ERR_CUDA, "cuMemGetAddressRange unavailable");
      range = reinterpret_cast<AddressRangeFn>(fn);
    }
    unsigned long long base = 0;
    size_t size = 0;
    GD_CHECK(range(&base, &size, reinterpret_cast<unsigned long long>(ptr)) == 0, GD_ERR_CUDA,
             "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    GD_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    memcpy(handle_out, &h, sizeof h);
    *offset = reinterpret_cast<unsigned long long>(ptr) - base;
  });
}

int gd_ipc_open(const void* handle, uint64_t offset, void** ptr_out) {
  return guarded([&] {
    GD_CHECK(handle && ptr_out, GD_ERR_INVALID, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void* base = nullptr;
    GD_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *ptr_out = static_cast<char*>(base) + offset;
  });
}

int gd_ipc_close(void* base) {
  return guarded([&] { GD_CUDA(cudaIpcCloseMemHandle(base)); });
}

int gd_query_collect(const GdBvh* a, const GdBvh* b, const GdConfig* cfg, void* workspace, const GdResult* result_dev,
                     GdResult* out, GdIterStat* stats, int max_stats, void* stream) {
  return guarded([&] {
    GD_CHECK(cfg && out, GD_ERR_INVALID, "null argument");
    (void)a;
    (void)b;
    query_collect(*cfg, workspace, result_dev, out, stats, max_stats, S(stream));
  });
}

int gd_dfs_query(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* b, const GdConfig* cfg, void* workspace,
                 size_t workspace_bytes, GdResult* out, int64_t* visited_nodes, void* stream) {
  return guarded([&] {
    GD_CHECK(mesh_a && mesh_b && b && cfg && out, GD_ERR_INVALID, "null argument");
    dfs_query(*mesh_a, *mesh_b, *b, *cfg, workspace, workspace_bytes, out, visited_nodes, S(stream));
    if (out->status == GD_ERR_WORKSPACE)
      throw Failure{GD_ERR_WORKSPACE, "DFS band overflow: raise GdConfig.band_cap"};
  });
}

int gd_tri_tri_batch(int kind, int precision, const void* t1, const void* t2, int64_t n, void* d, void* p, void* q,
                     void* stream) {
  return guarded([&] { tri_tri_batch(kind, precision, t1, t2, n, d, p, q, S(stream)); });
}

int gd_tri_tri_fast(int kind, const float* t1, const float* t2, int64_t n, float* d, void* stream) {
  return guarded([&] { tri_tri_fast(kind, t1, t2, n, d, S(stream)); });
}

int gd_box_bounds_batch(int which, int precision, const void* amin, const void* amax, const void* bmin,
                        const void* bmax, int64_t n, void* out, void* stream) {
  return guarded([&] { box_bounds_batch(which, precision, amin, amax, bmin, bmax, n, out, S(stream)); });
}

int gd_brute_force(int kind, int precision, const void* pts_a, int64_t ma, const void* pts_b, int64_t mb,
                   GdResult* out, void* stream) {
  return guarded([&] {
    GD_CHECK(out, GD_ERR_INVALID, "null argument");
    brute_force(kind, precision, pts_a, ma, pts_b, mb, out, S(stream));
  });
}

}  // extern "C"
