// Device-resident Krylov loops: a CUDA graph whose single node is a
// conditional WHILE node; its body (captured once from the stream the solver
// launches one iteration on) ends with a one-thread check kernel that decides
// on the device whether the loop continues (cudaGraphSetConditional).  The
// host launches the graph once per solve (plus once per true-residual
// refresh, every 50 iterations, solvers.py:145-150) instead of enqueueing
// ~30 kernels and synchronising on the stopping test every iteration.
//
// PCG check (the reference loop, solvers.py:138-165): with device scalars
// s = [rz, pAp, alpha, rz_new, beta] the kernel reproduces, in order,
//   if pAp <= 0: break
//   relres = sqrt|rz_new| / norm0; history.append(relres)
//   if rel_tol > 0 and relres <= rel_tol: converged
//   if rz_new == 0: converged
//   beta = rz_new / rz; rz = rz_new
// and stops after max_iters, or pauses before an iteration whose index is a
// multiple of 50 (the host runs that true-residual iteration eagerly).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "fb_common.cuh"

namespace fb {

// state: [0] iterations done, [1] stop reason (0 running / paused,
// 1 converged, 2 pAp <= 0, 3 max_iters), [2] max_iters; cfg = [norm0,
// rel_tol]: per-solve values live in device memory, so one captured graph
// serves every solve with the same operator and preconditioner)
__global__ void cg_check_kernel(unsigned long long handle, int in_graph, double* __restrict__ s,
                                int* __restrict__ state, double* __restrict__ hist,
                                const double* __restrict__ cfg, int period) {
  const double norm0 = cfg[0], rel_tol = cfg[1];
  const int max_iters = state[2];
  const int it = state[0] + 1;
  state[0] = it;
  const double pAp = s[1], rz_new = s[3];
  int stop = 0;
  if (pAp <= 0.0) {
    stop = 2;
  } else {
    const double relres = sqrt(fabs(rz_new)) / norm0;
    hist[it] = relres;
    if ((rel_tol > 0.0 && relres <= rel_tol) || rz_new == 0.0) {
      stop = 1;
    } else {
      s[4] = __ddiv_rn(rz_new, s[0]);  // beta
      s[0] = rz_new;
      if (it >= max_iters) stop = 3;
    }
  }
  state[1] = stop;
  if (in_graph) {
    const bool pause = period > 0 && (it + 1) % period == 0;
    cudaGraphSetConditional(cudaGraphConditionalHandle(handle), (stop == 0 && !pause) ? 1u : 0u);
  }
}

// p = z + beta p with beta on the device (s[4]); numpy rounding
__global__ void xpby_dev_kernel(int64_t n, const double* __restrict__ z,
                                const double* __restrict__ beta, double* __restrict__ p) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const double b = beta[0];
  if (i < n) p[i] = __dadd_rn(z[i], __dmul_rn(b, p[i]));
}

}  // namespace fb

using namespace fb;

struct fb_while_graph {
  cudaGraph_t graph = nullptr;
  cudaGraph_t body = nullptr;  // owned by `graph`
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
};

extern "C" {

int fb_while_graph_create(fb_while_graph** out) {
  FB_REQUIRE(out != nullptr, "out is NULL");
  *out = nullptr;
  fb_while_graph* G = new fb_while_graph();
  cudaError_t e = cudaGraphCreate(&G->graph, 0);
  if (e == cudaSuccess)
    e = cudaGraphConditionalHandleCreate(&G->handle, G->graph, 1, cudaGraphCondAssignDefault);
  if (e == cudaSuccess) {
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = G->handle;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    e = cudaGraphAddNode(&node, G->graph, nullptr, 0, &p);
    if (e == cudaSuccess) G->body = p.conditional.phGraph_out[0];
  }
  if (e != cudaSuccess) {
    if (G->graph) cudaGraphDestroy(G->graph);
    delete G;
    set_error(std::string("while graph: ") + cudaGetErrorString(e));
    return FB_ERR_CUDA;
  }
  *out = G;
  return FB_OK;
}

unsigned long long fb_while_graph_handle(const fb_while_graph* G) {
  return G ? (unsigned long long)G->handle : 0ull;
}

int fb_while_graph_begin(fb_while_graph* G, void* stream) {
  FB_REQUIRE(G != nullptr && G->exec == nullptr, "graph missing or already captured");
  FB_TRY_CUDA(cudaStreamBeginCaptureToGraph(as_stream(stream), G->body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal));
  return FB_OK;
}

int fb_while_graph_end(fb_while_graph* G, void* stream) {
  FB_REQUIRE(G != nullptr, "graph is NULL");
  cudaGraph_t g = nullptr;
  FB_TRY_CUDA(cudaStreamEndCapture(as_stream(stream), &g));
  FB_TRY_CUDA(cudaGraphInstantiate(&G->exec, G->graph, 0));
  return FB_OK;
}

int fb_while_graph_launch(const fb_while_graph* G, void* stream) {
  FB_REQUIRE(G != nullptr && G->exec != nullptr, "graph not instantiated");
  FB_TRY_CUDA(cudaGraphLaunch(G->exec, as_stream(stream)));
  count_launch();
  return FB_OK;
}

void fb_while_graph_destroy(fb_while_graph* G) {
  if (!G) return;
  if (G->exec) cudaGraphExecDestroy(G->exec);
  if (G->graph) cudaGraphDestroy(G->graph);
  delete G;
}

int fb_cg_check(unsigned long long handle, int in_graph, double* s, int* state, double* hist,
                const double* cfg, int period, void* stream) {
  cg_check_kernel<<<1, 1, 0, as_stream(stream)>>>(handle, in_graph, s, state, hist, cfg, period);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

int fb_xpby_dev(int64_t n, const double* z, const double* beta, double* p, void* stream) {
  if (n <= 0) return FB_OK;
  xpby_dev_kernel<<<ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, z, beta, p);
  FB_CHECK_LAUNCH();
  return FB_OK;
}

}  // extern "C"
