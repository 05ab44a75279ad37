// Device-resident LM level: the control flow of _solve_level_multi
// (solver.py:505-537, bundle._lm_level) run on the GPU as a CUDA graph with a
// conditional WHILE node.  The loop body is captured once from the caller's
// stream (solve -> pose update -> linearise -> assemble, all through the
// ordinary pba_* calls), followed by
//   lm_decide_kernel  — the accept / reject / lambda / termination logic of
//                       one iteration, one IterationRecord appended to a
//                       device array, and the loop condition set for the
//                       next iteration (cudaGraphSetConditional);
//                       On acceptance the same kernel copies the candidate
//                       buffers (poses, generations, H, b, totals) over the
//                       current ones, so the captured body reads buffer 0.
// One graph launch then runs a whole level with no host round trip per
// iteration; the host reads the records and the final state once.

#include <stdint.h>

#include "pba_common.cuh"

struct pba_lm_loop {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
  cudaStream_t capture = nullptr;
  bool capturing = false;
};

namespace pba {
namespace {

struct CopySegs {
  uint32_t* dst[PBA_LM_MAX_COPY];
  const uint32_t* src[PBA_LM_MAX_COPY];
  int64_t words[PBA_LM_MAX_COPY];
  int n;
};

// One iteration's decision (state layout in include/pba.h PBA_LM_*): the
// accept / reject, lambda, record and stop logic of solver.py:505-537.
// Returns whether the candidate was accepted.
__device__ bool lm_decide(double* __restrict__ s, double* __restrict__ records,
                          const int32_t* __restrict__ status_solve,
                          const int32_t* __restrict__ status_step,
                          const double* __restrict__ new_totals, double* __restrict__ lam_dev,
                          cudaGraphConditionalHandle handle) {
  double cost = s[PBA_LM_COST], count = s[PBA_LM_COUNT], lam = s[PBA_LM_LAMBDA];
  const double factor = s[PBA_LM_FACTOR], rel_tol = s[PBA_LM_REL_TOL];
  const double ceiling = s[PBA_LM_LAMBDA_CEILING], floor_pb = s[PBA_LM_COST_FLOOR];
  const int it = (int)s[PBA_LM_ITERATION], max_it = (int)s[PBA_LM_MAX_ITERATIONS];
  const int n_rec = (int)s[PBA_LM_N_RECORDS];
  bool stop = false, accepted = false, record = true;
  if (*status_solve != 0) {  // LinAlgError from the solve
    if (it == 1) {
      s[PBA_LM_ERROR] = PBA_LM_ERR_UNDERCONSTRAINED;
      stop = true;
      record = false;
    } else {
      lam *= factor;
      stop = lam > ceiling;
    }
  } else if (*status_step != 0) {  // ||dq|| >= 1
    s[PBA_LM_ERROR] = PBA_LM_ERR_PERTURBATION;
    stop = true;
    record = false;
  } else {
    const double new_cost = new_totals[0], new_count = new_totals[1];
    const double rel_change = fabs(cost - new_cost) / fmax(cost, 1e-300);
    if (new_cost < cost && new_count > 0.0) {
      cost = new_cost;
      count = new_count;
      lam = fmax(lam * 0.5, 1e-12);
      accepted = true;
    } else {
      lam *= factor;
    }
    stop = rel_change < rel_tol || lam > ceiling;
  }
  if (record) {
    double* r = records + PBA_LM_RECORD_DOUBLES * n_rec;
    r[0] = lam;
    r[1] = cost;
    r[2] = count;
    r[3] = accepted ? 1.0 : 0.0;
    r[4] = new_totals[0];  // the candidate's cost and count (what this
    r[5] = new_totals[1];  // iteration's linearisation evaluated)
    s[PBA_LM_N_RECORDS] = n_rec + 1;
  }
  // the loop head of the next iteration (solver.py:510-511)
  if (it + 1 > max_it || cost <= floor_pb * fmax(count, 1.0)) stop = true;
  s[PBA_LM_COST] = cost;
  s[PBA_LM_COUNT] = count;
  s[PBA_LM_LAMBDA] = lam;
  s[PBA_LM_ITERATION] = it + 1;
  s[PBA_LM_ACCEPTED] = accepted ? 1.0 : 0.0;
  s[PBA_LM_STOP] = stop ? 1.0 : 0.0;
  *lam_dev = lam;
  cudaGraphSetConditional(handle, stop ? 0u : 1u);
  return accepted;
}

// Thread 0 decides; on acceptance the whole CTA copies the candidate
// buffers over the current ones, so the loop body always reads buffer 0.
__global__ void __launch_bounds__(256) lm_decide_kernel(double* __restrict__ s,
                                                        double* __restrict__ records,
                                                        const int32_t* __restrict__ status_solve,
                                                        const int32_t* __restrict__ status_step,
                                                        const double* __restrict__ new_totals,
                                                        double* __restrict__ lam_dev,
                                                        cudaGraphConditionalHandle handle,
                                                        CopySegs segs) {
  __shared__ int take;
  if (threadIdx.x == 0)
    take = lm_decide(s, records, status_solve, status_step, new_totals, lam_dev, handle) ? 1 : 0;
  __syncthreads();
  if (!take) return;
  for (int k = 0; k < segs.n; ++k)
    for (int64_t i = threadIdx.x; i < segs.words[k]; i += blockDim.x) segs.dst[k][i] = segs.src[k][i];
}

__global__ void stamp_kernel(const double* __restrict__ state, int64_t* __restrict__ out, int slot) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const int it = (int)state[PBA_LM_ITERATION];
  out[8 * it + slot] = (int64_t)t;
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" int pba_diag_lm_stamp(const double* state, int64_t* out, int32_t slot, void* stream) {
  PBA_ARG_CHECK(state && out && slot >= 0 && slot < 8, "bad argument");
  stamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(state, out, slot);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

extern "C" int pba_lm_loop_begin(void* stream, pba_lm_loop** out, uint64_t* handle) {
  PBA_ARG_CHECK(stream && out && handle, "NULL argument (the default stream cannot be captured)");
  pba_lm_loop* L = new pba_lm_loop();
  auto fail = [&](cudaError_t e) {
    cudaGetLastError();  // not sticky: clear it so later launch checks do not report it
    if (L->graph) cudaGraphDestroy(L->graph);
    delete L;
    set_error("CUDA error %s: %s (conditional graph)", cudaGetErrorName(e), cudaGetErrorString(e));
    return PBA_ERR_CUDA;
  };
  cudaError_t e = cudaGraphCreate(&L->graph, 0);
  if (e != cudaSuccess) return fail(e);
  // default 1: the body runs at least once (the host checks the loop head first)
  e = cudaGraphConditionalHandleCreate(&L->handle, L->graph, 1, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) return fail(e);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = L->handle;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, L->graph, nullptr, 0, &p);
  if (e != cudaSuccess) return fail(e);
  L->capture = static_cast<cudaStream_t>(stream);
  e = cudaStreamBeginCaptureToGraph(L->capture, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                    cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) return fail(e);
  L->capturing = true;
  *out = L;
  *handle = (uint64_t)L->handle;
  return PBA_OK;
}

extern "C" int pba_lm_decide(double* state, double* records, const int32_t* status_solve,
                             const int32_t* status_step, const double* new_totals,
                             double* lam_dev, uint64_t handle, void* const* dst,
                             const void* const* src, const int64_t* bytes, int32_t n,
                             void* stream) {
  PBA_ARG_CHECK(state && records && status_solve && status_step && new_totals && lam_dev,
                "NULL buffer");
  PBA_ARG_CHECK(n >= 0 && n <= PBA_LM_MAX_COPY && (n == 0 || (dst && src && bytes)),
                "bad copy segments");
  CopySegs segs{};
  for (int k = 0; k < n; ++k) {
    PBA_ARG_CHECK(bytes[k] >= 0 && bytes[k] % 4 == 0, "copy sizes must be multiples of 4 bytes");
    segs.dst[k] = static_cast<uint32_t*>(dst[k]);
    segs.src[k] = static_cast<const uint32_t*>(src[k]);
    segs.words[k] = bytes[k] / 4;
  }
  segs.n = n;
  lm_decide_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      state, records, status_solve, status_step, new_totals, lam_dev,
      (cudaGraphConditionalHandle)handle, segs);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

extern "C" int pba_lm_loop_end(pba_lm_loop* L) {
  PBA_ARG_CHECK(L && L->capturing, "no loop being captured");
  cudaGraph_t body = nullptr;
  L->capturing = false;
  PBA_CUDA_TRY(cudaStreamEndCapture(L->capture, &body));
  PBA_CUDA_TRY(cudaGraphInstantiate(&L->exec, L->graph, 0));
  return PBA_OK;
}

extern "C" int pba_lm_loop_launch(pba_lm_loop* L, void* stream) {
  PBA_ARG_CHECK(L && L->exec, "loop not instantiated");
  PBA_CUDA_TRY(cudaGraphLaunch(L->exec, static_cast<cudaStream_t>(stream)));
  return PBA_OK;
}

extern "C" void pba_lm_loop_destroy(pba_lm_loop* L) {
  if (!L) return;
  if (L->capturing) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(L->capture, &g);
    cudaGetLastError();
  }
  if (L->exec) cudaGraphExecDestroy(L->exec);
  if (L->graph) cudaGraphDestroy(L->graph);
  delete L;
}
