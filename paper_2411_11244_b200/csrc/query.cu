// query.cu -- host orchestration of a BVTT distance query (query.py:480-568).
//
// One query = a fixed launch sequence on one stream, no host round trip:
//   k_traverse        ONE persistent cooperative launch: root bounds, slack,
//                     root front (query.py:454-509), then every adaptive-depth
//                     expansion (query.py:349-451) separated by grid barriers
//   k_nfilter         leaf pairs -> triangle-pair candidates (box + separating-
//                     axis bounds)                              (query.py:287-346)
//   k_ntest           float32 narrow phase on the candidates (min), fills the
//                     exact-pass band
//   k_refine          exact narrow phase (reference arithmetic, 64 or 32 bit)
//                     on the band entries within E of the best float32
//                     distance, one thread per entry, lexicographic 128-bit
//                     key minimum; its last block writes the witness and result
// The kernels after k_traverse use programmatic dependent launch (each waits
// in griddepcontrol.wait for its predecessor), so their launches overlap the
// predecessor's drain.  The bound is a float32 cell carrying a slack E
// (DESIGN.md "Exactness"): culling is conservative, so every pair that can
// attain the reference's exact answer reaches the exact pass.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstring>
#include <vector>

#include "dfs.cuh"

namespace gd {

struct WsLayout {
  size_t state, fnode, fkey, band_ids, band_d, result, total;
  unsigned long long arena, band_cap;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// The front arena is sized by the caller (GdConfig.arena_entries; the Python
// layer derives it from the free HBM), independent of front_hard_cap: a
// level that does not fit is expanded in chunks (traverse.cuh plan_sweep).
constexpr unsigned long long kDefaultArena = 1ull << 26;  // 768 MB
static WsLayout ws_layout(const GdConfig& cfg) {
  WsLayout L;
  L.arena = cfg.arena_entries > 0 ? (unsigned long long)cfg.arena_entries : kDefaultArena;
  L.arena = std::max<unsigned long long>(L.arena, 64);
  L.band_cap = cfg.band_cap > 0 ? (unsigned long long)cfg.band_cap : (1ull << 26);  // 800 MB: dense near-contact scenes
  size_t o = 0;
  auto take = [&](size_t& field, size_t bytes) {
    field = o;
    o = align_up(o + bytes, 256);
  };
  take(L.state, sizeof(QState));
  take(L.result, sizeof(GdResult));
  take(L.fnode, L.arena * sizeof(uint2));
  take(L.fkey, L.arena * sizeof(float));
  take(L.band_ids, L.band_cap * sizeof(uint2));
  take(L.band_d, L.band_cap * sizeof(float));
  L.total = o;
  return L;
}

size_t query_workspace_size(const GdConfig& cfg) { return ws_layout(cfg).total; }

static void validate(const GdBvh& a, const GdBvh& b, const GdConfig& cfg) {
  GD_CHECK(cfg.kind == 0 || cfg.kind == 1, GD_ERR_INVALID, "kind must be 0 (min) or 1 (max)");
  GD_CHECK(cfg.precision == 32 || cfg.precision == 64, GD_ERR_CONFIG, "precision must be 32 or 64");
  GD_CHECK(cfg.front_cap >= 4, GD_ERR_CONFIG, "front_cap must be >= 4");
  GD_CHECK(cfg.depth_cap >= 1 && cfg.depth_cap <= 16, GD_ERR_CONFIG, "depth_cap must be in [1, 16]");
  GD_CHECK(cfg.front_hard_cap >= 4, GD_ERR_CONFIG, "front_hard_cap must be >= 4");
  GD_CHECK(cfg.arena_entries >= 0 && cfg.arena_entries < (1ll << 31), GD_ERR_CONFIG,
           "arena_entries must be in [0, 2^31)");
  GD_CHECK(cfg.frame == 0 || cfg.frame == 1, GD_ERR_CONFIG, "frame must be 0 (world) or 1 (B-local)");
  GD_CHECK(cfg.n_peers >= 0 && cfg.n_peers <= 64 && (cfg.n_peers == 0 || cfg.peer_bounds), GD_ERR_INVALID,
           "peer_bounds must list n_peers (<= 64) bound cells");
  GD_CHECK(a.depth >= 0 && a.depth <= 31 && b.depth >= 0 && b.depth <= 31, GD_ERR_INVALID,
           "tree depth out of range");
  GD_CHECK(a.box && b.box && a.leaf_rec && b.leaf_rec && a.vtx32 && b.vtx32 && a.vmap && b.vmap,
           GD_ERR_INVALID, "BVH arrays must be allocated");
  // the box and leaf_tri gathers use 256-bit loads (engine.cuh)
  GD_CHECK(((reinterpret_cast<uintptr_t>(a.box) | reinterpret_cast<uintptr_t>(b.box) |
             reinterpret_cast<uintptr_t>(a.leaf_tri) | reinterpret_cast<uintptr_t>(b.leaf_tri)) & 31) == 0,
           GD_ERR_INVALID, "BVH box / leaf_tri buffers must be 32-byte aligned");
}

// optional phase timing for the bench: events between the query phases
static bool g_profile = false;
static cudaEvent_t g_ev[6];
static int g_ev_dev = -1;
static const QState* g_last_state = nullptr;  // profiled query's state (iteration timestamps)
void set_profiling(int on) {
  g_profile = on != 0;
  if (g_profile) {
    int dev = 0;
    GD_CUDA(cudaGetDevice(&dev));
    if (g_ev_dev != dev) {
      for (auto& e : g_ev) GD_CUDA(cudaEventCreate(&e));
      g_ev_dev = dev;
    }
  }
}
// [init, expand (all iterations), narrow (filter + test), exact + witness, -] ms,
// then (n > 5) the duration of each expansion iteration of the last profiled
// query (device %globaltimer at the grid barriers)
int phase_ms(float* out, int n) {
  if (g_ev_dev < 0) return 0;
  GD_CUDA(cudaEventSynchronize(g_ev[5]));
  int k = 0;
  for (; k < 5 && k < n; ++k) GD_CUDA(cudaEventElapsedTime(out + k, g_ev[k], g_ev[k + 1]));
  if (g_last_state && n > 5) {
    // per iteration: total, then (n > 5 + iterations) the sweep part
    int iters = 0;
    unsigned long long t[kMaxIters + 1], sw[kMaxIters], pl[kMaxIters + 1];
    GD_CUDA(cudaMemcpy(&iters, &g_last_state->iter, sizeof(int), cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(t, g_last_state->t_it, sizeof(t), cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(sw, g_last_state->t_sweep, sizeof(sw), cudaMemcpyDeviceToHost));
    GD_CUDA(cudaMemcpy(pl, g_last_state->t_plan, sizeof(pl), cudaMemcpyDeviceToHost));
    for (int i = 0; i < iters && k < n; ++i, ++k) out[k] = (float)((double)(t[i + 1] - t[i]) * 1e-6);
    for (int i = 0; i < iters && k < n; ++i, ++k) out[k] = (float)((double)(sw[i] > t[i] ? sw[i] - t[i] : 0) * 1e-6);
    // then the planning after each barrier (commit + plan of the next sweep, block 0)
    for (int i = 0; i < iters && k < n; ++i, ++k)
      out[k] = (float)((double)(pl[i + 1] > t[i + 1] ? pl[i + 1] - t[i + 1] : 0) * 1e-6);
    // then k_traverse's edges (block 0): entry -> prologue barrier passed,
    // barrier -> first sweep planned, last sweep -> exit
    unsigned long long e[3];
    GD_CUDA(cudaMemcpy(e, g_last_state->t_edge, sizeof(e), cudaMemcpyDeviceToHost));
    if (k < n) out[k++] = (float)((double)(e[1] - e[0]) * 1e-6);
    if (k < n) out[k++] = (float)((double)(t[0] > e[1] ? t[0] - e[1] : 0) * 1e-6);
    if (k < n) out[k++] = (float)((double)(e[2] > t[iters] ? e[2] - t[iters] : 0) * 1e-6);
  }
  return k;
}

// launch `kernel` so it may be scheduled while the previous kernel of the
// stream drains (programmatic dependent launch; the kernel starts with
// grid_dependency_wait), hiding the launch gap between the query's kernels
template <typename... Args>
static void launch_pdl(void (*kernel)(Args...), unsigned grid, unsigned block, cudaStream_t s, QArgs q) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GD_CUDA(cudaLaunchKernelEx(&cfg, kernel, q));
}

// k_refine runs as a resident grid (blocks per SM x SMs) striding over the
// band: a few hundred blocks for a rings band of ~20K entries instead of
// thousands of mostly idle ones (each also takes a turn on the done counter)
template <bool kMax, int kOrder>
static unsigned refine_grid() {
  static unsigned g[kMaxDevices] = {0};
  const int dev = current_device();
  if (g[dev] == 0) {
    int per_sm = 0;
    GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_refine<kMax, kOrder>, kRefineThreads, 0));
#ifdef GD_REFINE_PER_SM
    per_sm = std::min(per_sm, GD_REFINE_PER_SM);
#endif
    // max: the band's exact test is 9 vertex pairs -- 4 blocks / SM instead of
    // the resident 12 (fewer arrivals on the done counter): rings max 0.1988 -> 0.1966 ms
    if (kMax) per_sm = std::min(per_sm, 4);
    g[dev] = (unsigned)(std::max(per_sm, 1) * num_sms());
  }
  return g[dev];
}
// the exact pass instantiated for the meshes' transform order (engine.cuh
// mesh_vertex): both meshes' order when they agree (always, within one
// process), else the run-time switch
static int exact_order(const QArgs& q) {
  const int oa = q.ma.xf_order, ob = q.mb.xf_order;
  return oa == ob && oa >= 0 && oa <= 2 ? oa : -1;
}
template <bool kMax>
static void launch_refine(const QArgs& q, cudaStream_t s, bool pdl) {
  switch (exact_order(q)) {
#define GD_REFINE(O)                                                                     \
  case O:                                                                                \
    if (pdl)                                                                             \
      launch_pdl(k_refine<kMax, O>, refine_grid<kMax, O>(), kRefineThreads, s, q);        \
    else                                                                                 \
      k_refine<kMax, O><<<refine_grid<kMax, O>(), kRefineThreads, 0, s>>>(q);             \
    break;
    GD_REFINE(0)
    GD_REFINE(1)
    GD_REFINE(2)
    default:
      GD_REFINE(-1)
#undef GD_REFINE
  }
}

// k_traverse launch epochs: unique per launch within the process (odd,
// strictly increasing by 2), seeded away from values a fresh workspace might
// hold (0, small counters)
unsigned long long next_epoch() {
  static std::atomic<unsigned long long> e{
      (0x9E3779B97F4A7C15ull ^ (unsigned long long)std::chrono::steady_clock::now().time_since_epoch().count()) |
      (1ull << 62) | 1ull};
  return e.fetch_add(2, std::memory_order_relaxed);
}

// the persistent traversal kernel (its prologue initialises the state; no
// memset before it: the blocks meet on the launch's epoch, traverse.cu)
template <bool kMax>
static void launch_traverse(QArgs q, cudaStream_t s) {
  const int sms = num_sms();
  q.epoch = next_epoch();
  if (g_profile) GD_CUDA(cudaEventRecord(g_ev[1], s));
  // persistent traversal: as many blocks as can be co-resident (cooperative
  // launch guarantees it; the grid barrier relies on it); the split-query
  // variant carries the ownership tests
  // (function attributes and occupancy are per device: cached per device)
  const bool split = q.cfg.split_world > 1;
  auto kern = kMax ? (split ? k_traverse_max_split : k_traverse_max) : (split ? k_traverse_min_split : k_traverse_min);
  static int grid[kMaxDevices][2] = {{0}};
  const int dev = current_device();
  int& g = grid[dev][split ? 1 : 0];
  if (g == 0) {
    GD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kExpandDynSmem));
    int per_sm = 0;
    GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kExpandThreads, kExpandDynSmem));
    GD_CHECK(per_sm >= 1, GD_ERR_CUDA, "k_traverse cannot be resident");
    g = per_sm * sms;
  }
  {
    void* args[] = {const_cast<QArgs*>(&q)};
    GD_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(g), dim3(kExpandThreads), args, kExpandDynSmem, s));
  }
}

// the narrow / exact chain after a traversal: k_nfilter, k_ntest (min),
// k_nfilter<rescan>, k_refine.  pdl_first: the first kernel may overlap the
// drain of the stream's previous kernel (its traversal); off when the chain
// starts a side stream after an event wait.
#ifndef GD_NTEST_BLOCKS
#define GD_NTEST_BLOCKS 2  // k_ntest blocks per SM = its resident capacity at 105 registers: one wave striding over the list (4: 0.3469 ms, 2: 0.3464 ms rings min; nested shells min 26.46 -> 26.18 ms)
#endif
template <bool kMax>
static void launch_narrow(const QArgs& q, cudaStream_t s, bool pdl_first) {
  const int sms = num_sms();
  auto mark = [&](int i) {
    if (g_profile) GD_CUDA(cudaEventRecord(g_ev[i], s));
  };
  // profiling events between the kernels would serialise them: PDL only
  // when the phases are not being timed
  if (g_profile) {
    k_nfilter<kMax, false><<<sms * (kMax ? GD_NFILTER_BLOCKS_MAX : GD_NFILTER_BLOCKS) * (256 / kNfilterThreads), kNfilterThreads, 0, s>>>(q);
    if (!kMax) k_ntest<kMax><<<sms * GD_NTEST_BLOCKS, 256, 0, s>>>(q);
    mark(3);
    launch_refine<kMax>(q, s, false);  // + witness record in its last block
  } else {
    if (pdl_first)
      launch_pdl(k_nfilter<kMax, false>, sms * (kMax ? GD_NFILTER_BLOCKS_MAX : GD_NFILTER_BLOCKS) * (256 / kNfilterThreads), kNfilterThreads, s, q);
    else
      k_nfilter<kMax, false><<<sms * (kMax ? GD_NFILTER_BLOCKS_MAX : GD_NFILTER_BLOCKS) * (256 / kNfilterThreads), kNfilterThreads, 0, s>>>(q);
    if (!kMax) launch_pdl(k_ntest<kMax>, sms * GD_NTEST_BLOCKS, 256, s, q);
    launch_refine<kMax>(q, s, true);
  }
  mark(4);
  mark(5);
  GD_CUDA(cudaGetLastError());
  count_launches(kMax ? 2 : 3);
}

template <bool kMax>
static void launch_query(const QArgs& q, cudaStream_t s, cudaEvent_t traversal_done) {
  const int sms = num_sms();
  auto mark = [&](int i) {
    if (g_profile) GD_CUDA(cudaEventRecord(g_ev[i], s));
  };
  mark(0);
  launch_traverse<kMax>(q, s);  // records g_ev[1] before the kernel
  // the node boxes are read by k_traverse only: a refit for the next frame
  // may start once this event has fired
  if (traversal_done) GD_CUDA(cudaEventRecord(traversal_done, s));
  mark(2);
  launch_narrow<kMax>(q, s, true);
  count_launches(1);
}

static QArgs make_args(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                       void* ws, size_t ws_bytes, GdResult* result_dev) {
  WsLayout L = ws_layout(cfg);
  GD_CHECK(ws != nullptr && ws_bytes >= L.total, GD_ERR_WORKSPACE,
           "query workspace too small: need " + std::to_string(L.total) + " bytes");
  char* base = static_cast<char*>(ws);
  QArgs q;
  q.ma = ma;
  q.mb = mb;
  q.profile = g_profile ? 1 : 0;
  if (cfg.frame == 1) {  // traversal in B's local frame (gdist.h GdConfig.frame)
    q.xa = xf32_host(relative_mesh(ma, mb));
    GdMesh id = mb;
    id.has_xf = 0;
    q.xb = xf32_host(id);
  } else {
    q.xa = xf32_host(ma);
    q.xb = xf32_host(mb);
  }
  q.A = a;
  q.B = b;
  q.cfg = cfg;
  q.S = reinterpret_cast<QState*>(base + L.state);
  q.round = 0;
  q.fnode = reinterpret_cast<uint2*>(base + L.fnode);
  q.fkey = reinterpret_cast<float*>(base + L.fkey);
  q.band_ids = reinterpret_cast<uint2*>(base + L.band_ids);
  q.band_d = reinterpret_cast<float*>(base + L.band_d);
  q.arena = L.arena;
  q.band_cap = L.band_cap;
  q.result = result_dev;  // nullptr: the record stays in the state block (QState::res)
  q.mode = 0;
  q.sweep_budget = 0;
  return q;
}

// Frame graphs (graph.cu): the query kernels of a captured frame take one
// QArgs; a replay for new rigid transforms rewrites its meshes' transforms
// (the same derivation as make_args).
bool is_query_kernel(const void* f) {
  const void* ks[] = {(const void*)k_traverse_min,         (const void*)k_traverse_max,
                      (const void*)k_traverse_min_split,   (const void*)k_traverse_max_split,
                      (const void*)k_nfilter<false, false>, (const void*)k_nfilter<false, true>,
                      (const void*)k_nfilter<true, false>,  (const void*)k_nfilter<true, true>,
                      (const void*)k_ntest<false>,
                      (const void*)k_refine<false, 0>,      (const void*)k_refine<true, 0>,
                      (const void*)k_refine<false, 1>,      (const void*)k_refine<true, 1>,
                      (const void*)k_refine<false, 2>,      (const void*)k_refine<true, 2>,
                      (const void*)k_refine<false, -1>,     (const void*)k_refine<true, -1>};
  for (const void* k : ks)
    if (k == f) return true;
  return false;
}

void retransform(QArgs& q, const GdMesh& ma, const GdMesh& mb) {
  q.epoch = next_epoch();  // a replayed k_traverse node needs a fresh launch epoch
  GD_CHECK(ma.vtx == q.ma.vtx && mb.vtx == q.mb.vtx && ma.m == q.ma.m && mb.m == q.mb.m, GD_ERR_TOPOLOGY,
           "a frame graph replays the meshes it was captured with (same base vertices), moved");
  q.ma = ma;
  q.mb = mb;
  if (q.cfg.frame == 1) {
    q.xa = xf32_host(relative_mesh(ma, mb));
    GdMesh id = mb;
    id.has_xf = 0;
    q.xb = xf32_host(id);
  } else {
    q.xa = xf32_host(ma);
    q.xb = xf32_host(mb);
  }
}

// The rare overflow path (band or candidate list full) is not in the launch
// sequence: k_refine's record then says pending bit 1, and query_round runs
// k_nfilter<rescan> (every leaf pair of the round re-filtered and its pairs
// within E of the best float32 distance evaluated exactly) and k_refine
// again.  A no-op rescan launch in every query's dependent chain cost 13 us
// on the rings (0.357 -> 0.344 ms without it).
template <bool kMax>
static void launch_rescan(const QArgs& q, cudaStream_t s) {
  const int sms = num_sms();
  GD_CUDA(cudaMemsetAsync(&q.S->done, 0, sizeof(unsigned), s));
  k_nfilter<kMax, true><<<sms * 4 * (256 / kNfilterThreads), kNfilterThreads, 0, s>>>(q);
  launch_refine<kMax>(q, s, false);
  GD_CUDA(cudaGetLastError());
  count_launches(2);
}

// round 0 starts the query; round r > 0 resumes a query whose record says
// `pending` (its last round ended with a leaf chunk while levels remained)
void query_async(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                 void* ws, size_t ws_bytes, GdResult* result_dev, cudaStream_t s, cudaEvent_t traversal_done,
                 int round) {
  validate(a, b, cfg);
  GD_CHECK(round >= 0, GD_ERR_INVALID, "round must be >= 0");
  QArgs q = make_args(ma, mb, a, b, cfg, ws, ws_bytes, result_dev);
  q.round = round;
  if (g_profile) g_last_state = q.S;
  if (cfg.kind == 1)
    launch_query<true>(q, s, traversal_done);
  else
    launch_query<false>(q, s, traversal_done);
}

// Bound-exchange rounds of a split query: the traversal
// alone, at most `budget` sweeps per launch (mode 1: a launch continues the
// paused query, a no-op once its traversal ended); the caller combines the
// ranks' bound cells between launches.  query_finish runs the rest of the
// traversal without a budget, then the narrow and exact phases.
void query_traverse(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                    void* ws, size_t ws_bytes, int round, int budget, cudaStream_t s) {
  validate(a, b, cfg);
  GD_CHECK(round >= 0 && budget >= 1, GD_ERR_INVALID, "round must be >= 0 and sweep_budget >= 1");
  QArgs q = make_args(ma, mb, a, b, cfg, ws, ws_bytes, nullptr);
  q.round = round;
  q.mode = 1;
  q.sweep_budget = budget;
  if (cfg.kind == 1)
    launch_traverse<true>(q, s);
  else
    launch_traverse<false>(q, s);
  GD_CUDA(cudaGetLastError());
  count_launches(1);
}

void query_finish(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                  void* ws, size_t ws_bytes, GdResult* result_dev, cudaStream_t s) {
  validate(a, b, cfg);
  QArgs q = make_args(ma, mb, a, b, cfg, ws, ws_bytes, result_dev);
  q.round = 1;
  q.mode = 1;
  if (g_profile) g_last_state = q.S;
  if (cfg.kind == 1)
    launch_query<true>(q, s, nullptr);
  else
    launch_query<false>(q, s, nullptr);
}

// Continue a query whose record says `pending` (the caller has read it, so
// the stream is synchronised up to it): the rescan pass when the round's band
// overflowed (bit 1), else the next traversal round (bit 0).
void query_round(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg, void* ws,
                 size_t ws_bytes, GdResult* result_dev, cudaStream_t s, int round) {
  validate(a, b, cfg);
  GD_CHECK(round >= 1, GD_ERR_INVALID, "round must be >= 1");
  QArgs q = make_args(ma, mb, a, b, cfg, ws, ws_bytes, result_dev);
  int flags[2] = {0, 0};
  GD_CUDA(cudaMemcpyAsync(&flags[0], &q.S->band_overflow, sizeof(int), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaMemcpyAsync(&flags[1], &q.S->rescanned, sizeof(int), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  if (flags[0] && !flags[1]) {
    if (g_profile) g_last_state = q.S;
    if (cfg.kind == 1)
      launch_rescan<true>(q, s);
    else
      launch_rescan<false>(q, s);
    return;
  }
  query_async(ma, mb, a, b, cfg, ws, ws_bytes, result_dev, s, nullptr, round);
}

// Several queries on the same trees (config 3: min and max of one frame):
// their traversals back to back on s -- each needs the whole GPU -- then
// every query's narrow / exact chain on its own stream, forked after the last
// traversal and joined back into s.  The chains are short, latency-bound
// kernels on part of the GPU, so running them side by side hides most of one
// (and the trees' boxes are free for the next frame's refits once the last
// traversal is done: `traversal_done`).  Each chain ends with the copy of
// its result record to host_dst[i] when given.  Streams capture into a
// graph as a fork / join (frame_graph_create).
void query_result_async(const GdConfig& cfg, void* ws, void* host_dst, int max_stats, cudaStream_t s);
struct SideStreams {
  cudaStream_t st[8] = {};
  cudaEvent_t fork = nullptr, join[8] = {};
};
// per host thread (and device): two threads launching groups at once never
// share the fork / join events
static SideStreams& side_streams() {
  static thread_local SideStreams ss[kMaxDevices];
  SideStreams& r = ss[current_device()];
  if (!r.fork) {
    for (int i = 0; i < 8; ++i) {
      GD_CUDA(cudaStreamCreateWithFlags(&r.st[i], cudaStreamNonBlocking));
      GD_CUDA(cudaEventCreateWithFlags(&r.join[i], cudaEventDisableTiming));
    }
    GD_CUDA(cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming));
  }
  return r;
}

void query_group_prepare() { side_streams(); }

void query_group_async(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, int n,
                       const GdConfig* cfgs, void* const* wss, const size_t* ws_bytes, void* const* host_dst,
                       int max_stats, cudaStream_t s, cudaEvent_t traversal_done, bool external_record) {
  GD_CHECK(n >= 1 && n <= 8, GD_ERR_INVALID, "a query group holds 1 - 8 queries");
  std::vector<QArgs> qs;
  for (int i = 0; i < n; ++i) {
    validate(a, b, cfgs[i]);
    GD_CHECK(cfgs[i].split_world <= 1, GD_ERR_CONFIG, "query groups hold single-GPU queries");
    for (int j = 0; j < i; ++j)
      GD_CHECK(wss[j] != wss[i], GD_ERR_INVALID, "the queries of a group need distinct workspaces");
    qs.push_back(make_args(ma, mb, a, b, cfgs[i], wss[i], ws_bytes[i], nullptr));
  }
  for (int i = 0; i < n; ++i) {
    if (cfgs[i].kind == 1)
      launch_traverse<true>(qs[i], s);
    else
      launch_traverse<false>(qs[i], s);
  }
  count_launches(n);
  if (traversal_done)  // (an external event node when captured for another graph to wait on)
    GD_CUDA(cudaEventRecordWithFlags(traversal_done, s, external_record ? cudaEventRecordExternal : 0));
  SideStreams& ss = side_streams();
  if (n > 1) GD_CUDA(cudaEventRecord(ss.fork, s));
  for (int i = 0; i < n; ++i) {
    cudaStream_t si = i == 0 ? s : ss.st[i - 1];
    if (i > 0) GD_CUDA(cudaStreamWaitEvent(si, ss.fork, 0));
    if (cfgs[i].kind == 1)
      launch_narrow<true>(qs[i], si, i == 0);
    else
      launch_narrow<false>(qs[i], si, i == 0);
    if (host_dst && host_dst[i]) query_result_async(cfgs[i], wss[i], host_dst[i], max_stats, si);
    if (i > 0) {
      GD_CUDA(cudaEventRecord(ss.join[i - 1], si));
      GD_CUDA(cudaStreamWaitEvent(s, ss.join[i - 1], 0));
    }
  }
}

static_assert(offsetof(QState, stats) == offsetof(QState, res) + sizeof(GdResult),
              "result record and stats must be contiguous (one device->host copy)");

// enqueue the result record + stats copy into caller-provided (pinned) host
// memory; the caller synchronises (event) -- lets several queries be in flight
const void* query_result_device(const GdConfig& cfg, void* ws) {
  WsLayout L = ws_layout(cfg);
  return &reinterpret_cast<const QState*>(static_cast<char*>(ws) + L.state)->res;
}

void* query_bound_device(const GdConfig& cfg, void* ws) {
  WsLayout L = ws_layout(cfg);
  return &reinterpret_cast<QState*>(static_cast<char*>(ws) + L.state)->bound_bits;
}

void query_result_async(const GdConfig& cfg, void* ws, void* host_dst, int max_stats, cudaStream_t s) {
  WsLayout L = ws_layout(cfg);
  const QState* S = reinterpret_cast<const QState*>(static_cast<char*>(ws) + L.state);
  const int ns = std::min(std::max(max_stats, 0), kMaxIters);
  GD_CUDA(cudaMemcpyAsync(host_dst, &S->res, sizeof(GdResult) + sizeof(GdIterStat) * ns, cudaMemcpyDeviceToHost, s));
}

// pinned staging for the single device->host copy of result + stats
static thread_local char* g_pinned = nullptr;

void query_collect(const GdConfig& cfg, void* ws, const GdResult* result_dev, GdResult* out, GdIterStat* stats,
                   int max_stats, cudaStream_t s) {
  WsLayout L = ws_layout(cfg);
  char* base = static_cast<char*>(ws);
  const QState* S = reinterpret_cast<const QState*>(base + L.state);
  const size_t bytes = sizeof(GdResult) + sizeof(GdIterStat) * kMaxIters;
  if (!g_pinned) GD_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g_pinned), bytes, cudaHostAllocDefault));
  const int ns = stats ? std::min(std::max(max_stats, 0), kMaxIters) : 0;
  GD_CUDA(cudaMemcpyAsync(g_pinned, &S->res, sizeof(GdResult) + sizeof(GdIterStat) * ns, cudaMemcpyDeviceToHost, s));
  if (result_dev) GD_CUDA(cudaMemcpyAsync(g_pinned, result_dev, sizeof(GdResult), cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  memcpy(out, g_pinned, sizeof(GdResult));
  if (ns) memcpy(stats, g_pinned + sizeof(GdResult), sizeof(GdIterStat) * ns);
}

}  // namespace gd

namespace gd {

// per-triangle DFS comparator (dfs.cuh): scale, state, descent, exact pass
__global__ void k_dfs_check(QState* S) {
  if (S->band_overflow) S->err = GD_ERR_WORKSPACE;  // no rescan path here
}

template <bool kMax>
static void launch_dfs(const QArgs& q, cudaStream_t s) {
  const int sms = num_sms();
  GD_CUDA(cudaMemsetAsync(&q.S->dfs_coord, 0, sizeof(unsigned), s));
  k_dfs_scale<<<sms * 2, 256, 0, s>>>(q.ma, q.S);
  k_dfs_init<kMax><<<1, 1, 0, s>>>(q);
  const long long m = q.ma.m;
  if (m > 0) k_dfs<kMax><<<(unsigned)((m + kDfsThreads - 1) / kDfsThreads), kDfsThreads, 0, s>>>(q);
  k_dfs_check<<<1, 1, 0, s>>>(q.S);
  launch_refine<kMax>(q, s, false);
  GD_CUDA(cudaGetLastError());
  count_launches(m > 0 ? 5 : 4);
}

void dfs_query(const GdMesh& ma, const GdMesh& mb, const GdBvh& b, const GdConfig& cfg, void* ws, size_t ws_bytes,
               GdResult* out, int64_t* visited, cudaStream_t s) {
  validate(b, b, cfg);
  GD_CHECK(cfg.frame == 0, GD_ERR_CONFIG, "the DFS comparator traverses in the world frame (frame = 0)");
  GD_CHECK(ma.m < (1ll << 32), GD_ERR_INVALID, "mesh A too large");
  QArgs q = make_args(ma, mb, b, b, cfg, ws, ws_bytes, nullptr);
  if (cfg.kind == 1)
    launch_dfs<true>(q, s);
  else
    launch_dfs<false>(q, s);
  query_collect(cfg, ws, nullptr, out, nullptr, 0, s);
  unsigned long long v = 0;
  GD_CUDA(cudaMemcpyAsync(&v, &q.S->visited, sizeof v, cudaMemcpyDeviceToHost, s));
  GD_CUDA(cudaStreamSynchronize(s));
  if (visited) *visited = (int64_t)v;
}

}  // namespace gd
