/*
 * gdist.h -- C ABI of libgdist.so, the B200 (sm_100a) implementation of the
 * gDist hot path (arXiv 2411.11244): f12-BVH build / refit, BVTT front
 * traversal with AABB bounds, exact triangle-triangle narrow phase.
 *
 * Plain C: no torch / CUDA types in the signatures.  Device memory is owned
 * by the caller (the Python package allocates it as torch tensors); every
 * pointer documented "device" must point to CUDA device memory of the current
 * device, every "host" pointer to host memory.  `stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream).
 *
 * Every entry point returns a GdStatus; on failure a human-readable message is
 * available from gd_last_error() (thread-local).  No C++ exception crosses the
 * boundary.  The reference interface each entry point replaces is cited as
 * file:line under /root/reference/pkg/src/meshdist/.
 */
#ifndef GDIST_H
#define GDIST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GDIST_ABI_VERSION 15

/* Status codes; the Python layer maps them onto errors.py (errors.py:8-69). */
typedef enum GdStatus {
  GD_OK = 0,
  GD_ERR_INVALID = 1,        /* ValueError: bad shapes / arguments            */
  GD_ERR_CONFIG = 2,         /* ConfigError (query.py:77-92, 471-477)          */
  GD_ERR_TOPOLOGY = 3,       /* TopologyMismatchError (bvh.py:300-304)         */
  GD_ERR_FRONT_OVERFLOW = 4, /* FrontOverflowError (query.py:373-376, 448-449) */
  GD_ERR_WORKSPACE = 5,      /* caller workspace too small                     */
  GD_ERR_CUDA = 6,           /* CUDA runtime failure                           */
  GD_ERR_NO_DEVICE = 7       /* no CUDA device visible                         */
} GdStatus;

/* One mesh as seen by the device (mesh.py:21-66 TriangleMesh).  Vertices are
 * the float64 "base" positions; when has_xf != 0 every vertex is mapped to
 * R*v + t on the fly (mesh.py:102-105 apply_transform, row-major R). */
typedef struct GdMesh {
  const double* vtx;   /* device, (nv, 3) float64                        */
  const int32_t* tri;  /* device, (m, 3) vertex indices                  */
  int64_t nv;
  int64_t m;
  double rot[9];
  double trans[3];
  int32_t has_xf;
  /* operation order of the float64 transform, matching the host BLAS that
   * the reference's `V @ R.T + t` (mesh.py:104) runs on, so moved vertices
   * are bitwise the reference's: 0 = fma(R2, z, fma(R1, y, R0 x)) (OpenBLAS
   * dgemm, this image), 1 = (R0 x + R1 y) + R2 z without FMA, 2 =
   * fma(R0, x, fma(R1, y, R2 z)); then + t.  Probed once per process. */
  int32_t xf_order;
} GdMesh;

/* Sizes of an f12-BVH over m triangles (bvh.py:98-111, 184-211). */
typedef struct GdBvhSizes {
  int64_t leaf_count; /* L = largest power of two <= m */
  int64_t n_nodes;    /* 2L - 1                        */
  int32_t depth;      /* log2(L)                       */
  int32_t _pad;
  size_t build_workspace_bytes; /* scratch needed by gd_bvh_build */
} GdBvhSizes;

/* Device-resident f12-BVH (bvh.py:184-239).  Storage is implicit BFS: node
 * i has children 2i+1, 2i+2; leaves are the last L nodes.  All arrays are
 * caller-allocated device memory:
 *   box      : (n_nodes + 1) * 6 float32 (minx,miny,minz,maxx,maxy,maxz);
 *              node i at slot i + 1 (slot 0 is padding, so each sibling
 *              pair starts 16-byte aligned); traversal boxes of the
 *              float32-transformed vertices (refit output)
 *   leaf_rec : L * 8 int32, one 32-byte record per leaf in leaf (Morton)
 *              order: {a0, a1, a2, b0, b1, b2, tri0, tri1} = the staged
 *              vertex slots (vtx32 indices) of the leaf's two triangles and
 *              their triangle ids; a single-triangle leaf repeats triangle 0
 *              and has tri1 = -1
 *   vtx32    : nv * 4 float32, float32 copy of the mesh's BASE vertices in
 *              first-use order of the leaf records (gd_stage_vertices;
 *              gd_bvh_build / gd_bvh_layout stage them).  Refit and queries
 *              apply the mesh's (R, t) on the fly, so only a change of the
 *              base vertex buffer needs a new gd_stage_vertices.
 *   vmap     : nv int32, vtx32 slot of each mesh vertex
 *   leaf_vtx : 3 * L float4 = three planes of L float4 holding the first
 *              four distinct staged vertices of every leaf (x0 y0 z0 x1 |
 *              y1 z1 x2 y2 | z2 x3 y3 z3; repeats pad leaves with fewer):
 *              the refit streams these instead of gathering vertices
 *   leaf_x   : 2 * ceil(L / 32) + 1 + 2 * (L >> 16) + 5 uint32: per 32
 *              leaves a mask of the leaves with 5-6 distinct vertices, then
 *              per 32 leaves the rank of their first extra record, then a
 *              counter, then the refit's subtree arrival counters, then the
 *              float bits of max |coordinate| of the staged vertices (the
 *              scale of the float32 transform's rounding, read by queries)
 *   leaf_xvtx: 2 * L float4 (capacity): the 5th and 6th distinct vertex
 *              (repeated when only five) of each masked leaf, by rank
 *   leaf_tri : L * 20 float32 = five float4 per leaf: the two triangles'
 *              staged (base) vertices a0 a1 a2 b0 b1 b2 as 18 floats, then
 *              the float bits of tri0, tri1 (a single-triangle leaf repeats
 *              triangle 0 and has tri1 = -1): the narrow phase's one
 *              contiguous load per leaf instead of a record + six gathers
 * leaf_vtx, leaf_x, leaf_xvtx and leaf_tri are written by
 * gd_stage_vertices; the refit streams the first three. */
typedef struct GdBvh {
  float* box;
  int32_t* leaf_rec;
  float* vtx32;
  int32_t* vmap;
  float* leaf_vtx;
  uint32_t* leaf_x;
  float* leaf_xvtx;
  int64_t leaf_count;
  int64_t n_tris;
  int64_t nv;
  int32_t depth;
  int32_t _pad;
  float* leaf_tri;
} GdBvh;

/* EngineConfig (query.py:51-102).  `threads` and `batch_size` have no device
 * meaning and are not carried. */
typedef struct GdConfig {
  int32_t kind;              /* 0 = min query, 1 = max query               */
  int32_t precision;         /* 32 or 64: arithmetic of the exact pass      */
  int64_t front_cap;         /* C of the adaptive depth rule               */
  int32_t depth_cap;
  int32_t enhanced_bounds;
  int32_t culling;
  int32_t guarantee_witness; /* accepted; the engine always keeps ties      */
  int64_t front_hard_cap;
  int64_t warm_a;            /* warm_pair triangle ids, -1 = none          */
  int64_t warm_b;
  int64_t band_cap;          /* exact-pass candidate buffer entries, 0 = default */
  /* split query (multi-GPU): with split_world > 1 this call
   * expands only the node pairs whose ancestor pair at tree level
   * split_level (clamped to each tree's depth) hashes to split_rank; the
   * exact answers of the split_world calls combine lexicographically. */
  int32_t split_rank;
  int32_t split_world;       /* 0 or 1 = no split                            */
  int32_t split_level;
  /* traversal frame: 0 = world; 1 = B's local frame -- tree B's boxes are
   * those of B's untransformed vertices and tree A's those of A under
   * gd_mesh_relative(A, B), so a sequence where both meshes move refits one
   * tree per frame.  The exact pass always works in world coordinates, so
   * the answer is bitwise the world-frame one. */
  int32_t frame;
  /* temporal warm start: a DEVICE GdResult -- e.g.
   * the previous frame's record, gd_query_result_device -- read when the
   * query starts; if its status is 0 and tri_a >= 0, that pair seeds the
   * bound exactly as warm_a / warm_b do.  NULL = none.  Stream order makes
   * it safe: the producing query ran earlier on the same stream. */
  const void* warm_from;
  /* bound sharing across the ranks of a split query: a
   * DEVICE array of n_peers pointers to the other ranks' bound cells
   * (gd_query_bound_device of their workspaces, mapped here through CUDA IPC
   * -- NVLink peer memory).  Every bound this query commits is also applied
   * to those cells with a system-scope atomicMin / atomicMax, so every rank
   * culls with the best bound found anywhere.  0 / NULL = rank-local. */
  const void* peer_bounds;
  int32_t n_peers;
  /* expansion schedule: -1 = the reference's adaptive_depth exactly
   * (query.py:266-284; IterationStat.k follows it); 0 = the device schedule
   * with its default threshold; > 0 = the device schedule with this
   * threshold -- fronts of at most that many entries with >= 2 levels left
   * on both trees expand two levels per iteration (k = 2) in ONE sweep that
   * culls child pairs before their grandchildren, where the reference rule
   * would pick k = 1.  Same survivors and answers; fewer grid barriers. */
  int32_t schedule;
  /* front arena capacity in entries (12 bytes each; 0 = 2^26).  Independent
   * of front_hard_cap, which keeps the reference's FrontOverflowError
   * semantics on the candidates / survivors of each iteration (summed over
   * the chunks of an iteration).  A level whose children might not fit the
   * arena is expanded in chunks, depth first, so
   * any arena of a few thousand entries completes any query; a larger one
   * only saves rounds. */
  int64_t arena_entries;
} GdConfig;

/* QueryResult (query.py:230-263) + Witness (query.py:136-144). */
typedef struct GdResult {
  double distance;
  double witness_distance;
  double point_a[3];
  double point_b[3];
  int64_t tri_a;             /* -1 when no witness                           */
  int64_t tri_b;
  int64_t expanded_pairs;
  int64_t narrow_pairs;
  int64_t band_pairs;        /* candidates re-evaluated in the exact pass    */
  int64_t overflow_candidates;
  int64_t overflow_front_in;
  int64_t overflow_cap;
  int32_t iterations;
  int32_t status;
  int32_t rounds;            /* traversal rounds (one per leaf chunk)          */
  int32_t pending;           /* nonzero: not final -- the caller runs
                              * gd_query_round(round = rounds) until it is 0
                              * (gd_query / collect do): bit 0 levels remain
                              * (another traversal round), bit 1 the band
                              * overflowed (the rescan pass runs first) */
} GdResult;

/* IterationStat (query.py:147-162). */
typedef struct GdIterStat {
  int64_t front_in;
  int64_t front_out;
  int64_t culled;
  double bound_after;
  int32_t k;
  int32_t _pad;
} GdIterStat;

/* ---- library ---------------------------------------------------------- */
const char* gd_version(void);
const char* gd_last_error(void);
int gd_abi_version(void);
int gd_device_count(int* count);
/* number of hot-path kernels (refit + query) launched by this process */
long long gd_launch_count(void);
/* phase timing of subsequent queries (CUDA events); gd_query_phase_ms
 * returns the count written: [init, expand, narrow, exact pass, final] ms,
 * then (n > 5) the duration of each k_expand launch of the last query */
int gd_set_profiling(int enable);
int gd_query_phase_ms(float* out, int n);

/* ---- f12-BVH build / refit (bvh.py) ----------------------------------- */
/* bvh.py:98-111: L, depth, node count; workspace for gd_bvh_build. */
int gd_bvh_sizes(int64_t m, int64_t nv, GdBvhSizes* out);

/* build_f12 (bvh.py:267-289): Morton codes (bvh.py:69-95) + radix sort on
 * the device, exact greedy power-of-two pairing (bvh.py:98-181) on the host,
 * leaf layout, then a refit.  Writes prim_order (m) and leaf_tris (L, 2)
 * int64 host arrays with the reference's semantics. */
int gd_bvh_build(const GdMesh* mesh, GdBvh* bvh, void* workspace, size_t workspace_bytes,
                 int64_t* prim_order_host, int64_t* leaf_tris_host, void* stream);

/* Leaf records written with ORIGINAL mesh vertex indices (a tree laid out
 * on the host) -> first-use staged numbering: writes vmap, remaps the records
 * in place, stages the vertices.  workspace: GdBvhSizes.build_workspace_bytes.
 * gd_bvh_build does this itself.  Asynchronous. */
int gd_bvh_layout(const GdMesh* mesh, GdBvh* bvh, void* workspace, size_t workspace_bytes, void* stream);
/* How this thread's last gd_bvh_build paired the triangles
 * (_pair_to_power_of_two, bvh.py:98-181): 0 = no merge needed (a power of two),
 * 1 = on the device (the greedy's complete matching by scans + sort; exact
 * because the reference's slack stayed positive, checked), 2 = the exact
 * host restatement (a deferral was possible, or NaN surface areas). */
int gd_build_pairing_mode(void);

/* float32 copy of mesh->vtx (the base vertices, before mesh->rot/trans)
 * into bvh->vtx32 at the slots of bvh->vmap.  Needed once per base vertex
 * buffer. Asynchronous. */
int gd_stage_vertices(const GdMesh* mesh, GdBvh* bvh, void* stream);

/* *out = *a with the rigid transform of A expressed in B's local frame:
 * R = Rb^T Ra, t = Rb^T (ta - tb) (float64, fixed operation order; the
 * transform GdConfig.frame = 1 queries apply to A).  Host only. */
int gd_mesh_relative(const GdMesh* a, const GdMesh* b, GdMesh* out);

/* refit (bvh.py:292-306) with apply_transform (mesh.py:102-105) fused:
 * leaf boxes of the transformed staged vertices, bottom-up unions.
 * Asynchronous. */
int gd_refit(const GdMesh* mesh, GdBvh* bvh, void* stream);

/* Node boxes with the reference's dtype semantics (bvh.py:242-264):
 * precision 64 -> double (n_nodes, 3) min / max, precision 32 -> float.
 * node_min / node_max are device pointers.  Synchronous. */
int gd_export_boxes(const GdMesh* mesh, const GdBvh* bvh, int precision, void* node_min,
                    void* node_max, void* stream);

/* Exact greedy pairing on the host (bvh.py:98-181), exposed for testing:
 * sa = pair surface areas (n - 1), writes is_left (n bytes, 1 where pair
 * (i, i+1) merges).  Needs no GPU. */
int gd_pair_greedy(const double* sa_host, int64_t n, uint8_t* is_left_host);

/* ---- traversal engine (query.py) -------------------------------------- */
int gd_query_workspace_size(const GdBvh* a, const GdBvh* b, const GdConfig* cfg, size_t* bytes);

/* run_min_query / run_max_query (query.py:480-568).  Synchronous: one
 * device->host copy of the result at the end.  stats may be NULL. */
int gd_query(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
             const GdConfig* cfg, void* workspace, size_t workspace_bytes, GdResult* out,
             GdIterStat* stats, int max_stats, void* stream);

/* Asynchronous variant: enqueue only; the result is written by the device
 * into `result_dev` (a device GdResult) -- collect with gd_query_collect. */
int gd_query_async(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                   const GdConfig* cfg, void* workspace, size_t workspace_bytes,
                   GdResult* result_dev, void* stream);
/* Resume a query whose record (gd_query_collect / gd_query_result_async)
 * has `pending` set, with round = the record's `rounds`: if the round's band
 * overflowed (pending bit 1) the rescan pass and the exact pass again, else
 * traversal round `round` with its narrow and exact phases, on the same
 * workspace; the record is rewritten at its end.  Reads two flags of the
 * workspace (a short synchronisation of `stream`).  gd_query loops itself. */
int gd_query_round(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                   const GdConfig* cfg, void* workspace, size_t workspace_bytes, int round, void* stream);
/* gd_query_async that also records `traversal_done` (a cudaEvent_t, may be
 * NULL) on `stream` right after the traversal kernel: the node boxes are
 * read by the traversal only, so a refit of these trees for the next frame
 * may run on another stream once the event fires, overlapping this query's
 * narrow and exact phases (frame pipelining). */
int gd_query_async_ev(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                      const GdConfig* cfg, void* workspace, size_t workspace_bytes, GdResult* result_dev,
                      void* stream, void* traversal_done);
/* Bound-exchange rounds of a split query (the per-round
 * ncclAllReduce of the bound): enqueue ONLY the traversal -- round 0 starts
 * the query, a later round continues it -- limited to `sweep_budget` (>= 1)
 * expansion sweeps per call; a call after the traversal ended is a no-op.
 * Between calls the caller may combine the ranks' bound cells
 * (gd_query_bound_device: uint32 bits of a non-negative float, so an
 * integer MIN / MAX all-reduce is the float one).  gd_query_finish then
 * enqueues the rest of the traversal (no budget) and the narrow / exact
 * phases into `result_dev` (may be NULL); collect as after gd_query_async;
 * a record with `pending` resumes with gd_query_round as usual. */
int gd_query_traverse(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                      const GdConfig* cfg, void* workspace, size_t workspace_bytes, int round,
                      int sweep_budget, void* stream);
int gd_query_finish(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                    const GdConfig* cfg, void* workspace, size_t workspace_bytes, GdResult* result_dev,
                    void* stream);
/* Several queries on the same trees and meshes (config 3: the min and max
 * query of one frame), each on its own workspace: their traversals back to
 * back on `stream` (each needs the whole GPU), then every query's narrow /
 * exact chain on its own stream, forked after the last traversal and joined
 * back into `stream` -- the short, latency-bound chains overlap.  n in
 * [1, 8]; host_dst[i] (pinned, may be NULL) receives query i's result record
 * + max_stats GdIterStat at the end of its chain; traversal_done (a
 * cudaEvent_t or NULL) is recorded after the last traversal (the boxes are
 * free for the next frame's refits). */
int gd_query_group_async(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b, int n,
                         const GdConfig* cfgs, void* const* workspaces, const size_t* workspace_bytes,
                         void* const* host_dst, int max_stats, void* stream, void* traversal_done);
/* Frame graph: refit A and / or B, then n_queries
 * (<= 8) single-GPU queries (cfgs[i] on workspaces[i]; launched as by
 * gd_query_group_async) each followed, when host_dst[i] is not NULL, by the
 * copy of its result record + max_stats GdIterStat into host_dst[i]
 * (pinned) -- captured ONCE as a CUDA graph.
 * gd_frame_graph_launch replays it on `stream` for new rigid transforms of
 * the same meshes (same base vertices; mesh_a / mesh_b carry the frame's
 * rot / trans): one call per frame.  A record with `pending` (a chunked
 * traversal) resumes with gd_query_round as after gd_query_async.  The
 * workspaces and host buffers stay bound to the graph until destroy.
 * wait_before / traversal_done (cudaEvent_t or NULL): external event nodes
 * -- every replay first waits for wait_before's latest record, and records
 * traversal_done once its last traversal has read the trees' boxes.  Two
 * graphs alternating on two streams, each waiting for the other's
 * traversal_done, start frame f + 1's refits while frame f's narrow / exact
 * phases still run. */
int gd_frame_graph_create(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* a, const GdBvh* b,
                          int n_queries, const GdConfig* cfgs, void* const* workspaces,
                          const size_t* workspace_bytes, void* const* host_dst, int max_stats, int refit_a,
                          int refit_b, void* wait_before, void* traversal_done, void** graph_out);
int gd_frame_graph_launch(void* graph, const GdMesh* mesh_a, const GdMesh* mesh_b, void* stream);
int gd_frame_graph_destroy(void* graph);
/* Enqueue the device->host copy of the result record followed by
 * min(max_stats, 64) GdIterStat into host_dst (pinned memory of at least
 * sizeof(GdResult) + max_stats * sizeof(GdIterStat) bytes) on `stream`;
 * the caller synchronises (e.g. an event).  Lets several queries, each with
 * its own workspace, be in flight. */
/* Device address of the result record inside a query workspace (valid
 * after a query on that workspace completes in stream order). */
int gd_query_result_device(const GdConfig* cfg, void* workspace, const void** out);
/* Device address of the bound cell inside a query workspace (the target of
 * the peers' GdConfig.peer_bounds). */
int gd_query_bound_device(const GdConfig* cfg, void* workspace, void** out);
/* CUDA IPC for the bound exchange: the handle (64 bytes) of the allocation
 * holding `ptr` and ptr's offset in it; open maps a peer's handle into this
 * process (peer access enabled lazily) and returns base + offset; close
 * unmaps (pass the base, i.e. the opened pointer minus the offset). */
int gd_ipc_handle(const void* ptr, void* handle_out, uint64_t* offset);
int gd_ipc_open(const void* handle, uint64_t offset, void** ptr_out);
int gd_ipc_close(void* base);
int gd_query_result_async(const GdConfig* cfg, void* workspace, void* host_dst, int max_stats, void* stream);
int gd_query_collect(const GdBvh* a, const GdBvh* b, const GdConfig* cfg, void* workspace,
                     const GdResult* result_dev, GdResult* out, GdIterStat* stats, int max_stats,
                     void* stream);

/* Per-triangle DFS comparator (query.py:622-708 run_dfs_baseline): every
 * triangle of A descends B's tree depth-first, nearer child first, pruning
 * against one shared bound; synchronous.  `b` must be refit to mesh_b in the
 * world frame (cfg->frame = 0); cfg->kind / precision / band_cap apply, the
 * workspace is gd_query_workspace_size(b, b, cfg).  *visited_nodes = node
 * examinations (pops), summed over A's triangles. */
int gd_dfs_query(const GdMesh* mesh_a, const GdMesh* mesh_b, const GdBvh* b, const GdConfig* cfg,
                 void* workspace, size_t workspace_bytes, GdResult* out, int64_t* visited_nodes,
                 void* stream);

/* ---- OBJ ingest (mesh.py:112-163 load_obj), host only ------------------ */
/* Parse a Wavefront OBJ file with the reference's semantics (v / f records,
 * `#` comments, fan triangulation, negative relative indices, every other
 * record ignored).  On success *handle owns the mesh (read it with
 * gd_obj_read into caller buffers of 3 * n_vertices doubles and
 * 3 * n_triangles int64, then gd_obj_close).  On a malformed record returns
 * GD_ERR_INVALID with *err_line = its 1-based line and the reference's
 * message in gd_last_error(); *err_line = 0 means the file could not be
 * opened. */
int gd_obj_open(const char* path, void** handle, int64_t* n_vertices, int64_t* n_triangles, int64_t* err_line);
int gd_obj_read(void* handle, double* vertices, int64_t* triangles);
void gd_obj_close(void* handle);

/* ---- batch math (bounds.py) ------------------------------------------- */
/* batch_tri_tri_min / batch_tri_tri_max (bounds.py:245-330), exact
 * reference arithmetic in `precision` (32 / 64).  t1, t2: device (n, 3, 3);
 * d: (n); p, q: (n, 3); element type double for 64, float for 32. */
int gd_tri_tri_batch(int kind, int precision, const void* t1, const void* t2, int64_t n, void* d,
                     void* p, void* q, void* stream);

/* Fast float32 narrow phase used by the traversal (FMA-contracted): d only.
 * kind 0 = min, 1 = max, 2 = the min distance's conditioning-aware lower
 * bound the exact band windows on.  t1, t2 float
 * (n, 3, 3), d float (n).  For error-bound tests. */
int gd_tri_tri_fast(int kind, const float* t1, const float* t2, int64_t n, float* d, void* stream);

/* batch_min_lower / batch_max_upper / batch_enhanced_min_upper /
 * batch_enhanced_max_lower (bounds.py:47-101): which = 0..3.
 * amin .. bmax: device (n, 3) in `precision`; out (n). */
int gd_box_bounds_batch(int which, int precision, const void* amin, const void* amax,
                        const void* bmin, const void* bmax, int64_t n, void* out, void* stream);

/* brute_force_min / brute_force_max (query.py:571-619) on the device:
 * all pairs, lexicographic tie-break. pts: device (m, 3, 3) in precision. */
int gd_brute_force(int kind, int precision, const void* pts_a, int64_t ma, const void* pts_b,
                   int64_t mb, GdResult* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GDIST_H */
