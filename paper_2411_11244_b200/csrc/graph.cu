// graph.cu -- a whole frame (refit A, refit B, the frame's queries and the
// copies of their result records to pinned host memory) as ONE CUDA graph
// ("CUDA-graph capture of refit + min + max per
// frame").  Captured once through the ordinary launch paths (cooperative
// traversal, programmatic dependent launches, memsets, copies); a replay for
// the next frame's rigid transforms rewrites only the transform arguments of
// the refit and query kernel nodes in the executable graph
// (cudaGraphExecKernelNodeSetParams) and launches it: one host call per
// frame instead of ~12 launches, no launch gaps inside the frame.
#include <vector>

#include "engine.cuh"

namespace gd {

void refit(const GdMesh& m, const GdBvh& T, cudaStream_t s);
bool is_refit_kernel(const void* f);
void query_async(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, const GdConfig& cfg,
                 void* ws, size_t ws_bytes, GdResult* result_dev, cudaStream_t s, cudaEvent_t traversal_done,
                 int round);
void query_result_async(const GdConfig& cfg, void* ws, void* host_dst, int max_stats, cudaStream_t s);
void query_group_prepare();
void query_group_async(const GdMesh& ma, const GdMesh& mb, const GdBvh& a, const GdBvh& b, int n,
                       const GdConfig* cfgs, void* const* wss, const size_t* ws_bytes, void* const* host_dst,
                       int max_stats, cudaStream_t s, cudaEvent_t traversal_done, bool external_record);
bool is_query_kernel(const void* f);
void retransform(QArgs& q, const GdMesh& ma, const GdMesh& mb);

struct FrameGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int dev = -1;
  GdBvh A{}, B{};
  GdMesh ma{}, mb{};
  std::vector<cudaGraphNode_t> refit_nodes, query_nodes;
  std::vector<cudaKernelNodeParams> refit_params, query_params;  // captured launch configurations
  std::vector<GdBvh> refit_trees;
  std::vector<QArgs> query_args;
  long long kernels = 0;
};

// wait_before / traversal_done (cudaEvent_t or null): external event nodes
// at the graph's start / after its last traversal.  Two graphs alternating
// on two streams, each waiting for the other's traversal_done, run frame
// f + 1's refits as soon as frame f's traversals have read the boxes --
// overlapping frame f's narrow / exact chains (run_sequence_minmax).
void* frame_graph_create(const GdMesh& ma, const GdMesh& mb, const GdBvh& A, const GdBvh& B, int n_queries,
                         const GdConfig* cfgs, void* const* wss, const size_t* ws_bytes, void* const* host_dst,
                         int max_stats, int refit_a, int refit_b, cudaEvent_t wait_before,
                         cudaEvent_t traversal_done) {
  GD_CHECK(n_queries >= 0 && n_queries <= 8, GD_ERR_INVALID, "a frame graph holds 0 - 8 queries");
  for (int i = 0; i < n_queries; ++i)
    GD_CHECK(cfgs[i].split_world <= 1 && cfgs[i].n_peers == 0, GD_ERR_CONFIG,
             "frame graphs hold single-GPU queries (no split, no peer bounds)");
  auto* fg = new FrameGraph();
  fg->dev = current_device();
  fg->A = A;
  fg->B = B;
  fg->ma = ma;
  fg->mb = mb;
  cudaStream_t cap = nullptr;
  try {
    query_group_prepare();  // the side streams of the narrow chains exist before the capture
    GD_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    GD_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    if (wait_before) GD_CUDA(cudaStreamWaitEvent(cap, wait_before, cudaEventWaitExternal));
    if (refit_a) refit(ma, A, cap);
    if (refit_b) refit(mb, B, cap);
    // the traversals back to back, then the queries' narrow / exact chains
    // side by side (a fork / join in the graph, query.cu query_group_async)
    if (n_queries > 0)
      query_group_async(ma, mb, A, B, n_queries, cfgs, wss, ws_bytes, host_dst, max_stats, cap, traversal_done,
                        true);
    else if (traversal_done)
      GD_CUDA(cudaEventRecordWithFlags(traversal_done, cap, cudaEventRecordExternal));
    GD_CUDA(cudaStreamEndCapture(cap, &fg->graph));
    GD_CUDA(cudaStreamDestroy(cap));
    cap = nullptr;
    GD_CUDA(cudaGraphInstantiate(&fg->exec, fg->graph, 0));
    size_t n = 0;
    GD_CUDA(cudaGraphGetNodes(fg->graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    GD_CUDA(cudaGraphGetNodes(fg->graph, nodes.data(), &n));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      GD_CUDA(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams p;
      GD_CUDA(cudaGraphKernelNodeGetParams(nd, &p));
      ++fg->kernels;
      if (is_refit_kernel(p.func)) {
        fg->refit_nodes.push_back(nd);
        fg->refit_params.push_back(p);
        fg->refit_trees.push_back(*static_cast<const GdBvh*>(p.kernelParams[0]));
      } else if (is_query_kernel(p.func)) {
        fg->query_nodes.push_back(nd);
        fg->query_params.push_back(p);
        fg->query_args.push_back(*static_cast<const QArgs*>(p.kernelParams[0]));
      }
    }
  } catch (...) {
    if (cap) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(cap, &g);
      if (g) cudaGraphDestroy(g);
      cudaStreamDestroy(cap);
    }
    if (fg->exec) cudaGraphExecDestroy(fg->exec);
    if (fg->graph) cudaGraphDestroy(fg->graph);
    delete fg;
    throw;
  }
  return fg;
}

// one frame: new rigid transforms of the captured meshes, then the graph
void frame_graph_launch(void* h, const GdMesh& ma, const GdMesh& mb, cudaStream_t s) {
  auto* fg = static_cast<FrameGraph*>(h);
  GD_CHECK(fg != nullptr, GD_ERR_INVALID, "null frame graph");
  GD_CHECK(current_device() == fg->dev, GD_ERR_INVALID, "frame graph launched on another device");
  GD_CHECK(ma.vtx == fg->ma.vtx && mb.vtx == fg->mb.vtx && ma.nv == fg->ma.nv && mb.nv == fg->mb.nv,
           GD_ERR_TOPOLOGY, "a frame graph replays the meshes it was captured with (same base vertices), moved");
  GD_CHECK(ma.xf_order == fg->ma.xf_order && mb.xf_order == fg->mb.xf_order, GD_ERR_INVALID,
           "a frame graph's exact pass is instantiated for the captured meshes' transform order (xf_order)");
  const XfF32 xa = xf32_host(ma), xb = xf32_host(mb);
  for (size_t i = 0; i < fg->refit_nodes.size(); ++i) {
    cudaKernelNodeParams p = fg->refit_params[i];
    GdBvh T = fg->refit_trees[i];
    XfF32 x = T.box == fg->A.box ? xa : xb;
    void* args[] = {&T, &x};
    p.kernelParams = args;
    p.extra = nullptr;
    GD_CUDA(cudaGraphExecKernelNodeSetParams(fg->exec, fg->refit_nodes[i], &p));
  }
  for (size_t i = 0; i < fg->query_nodes.size(); ++i) {
    cudaKernelNodeParams p = fg->query_params[i];
    QArgs q = fg->query_args[i];
    retransform(q, ma, mb);
    void* args[] = {&q};
    p.kernelParams = args;
    p.extra = nullptr;
    GD_CUDA(cudaGraphExecKernelNodeSetParams(fg->exec, fg->query_nodes[i], &p));
  }
  GD_CUDA(cudaGraphLaunch(fg->exec, s));
  count_launches(fg->kernels);
}

void frame_graph_destroy(void* h) {
  auto* fg = static_cast<FrameGraph*>(h);
  if (!fg) return;
  if (fg->exec) cudaGraphExecDestroy(fg->exec);
  if (fg->graph) cudaGraphDestroy(fg->graph);
  delete fg;
}

}  // namespace gd
