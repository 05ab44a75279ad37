// Feasibility probe: a CUDA graph with a conditional WHILE node whose body
// (captured from a stream) runs until a device-side decision clears the
// condition — the mechanism a device-resident LM loop would use.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void body_kernel(int* counter, int limit, cudaGraphConditionalHandle h) {
  int c = ++(*counter);
  cudaGraphSetConditional(h, c < limit ? 1 : 0);
}

__global__ void work_kernel(double* x) { x[threadIdx.x] += 1.0; }

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  int* counter;
  double* x;
  cudaMalloc(&counter, sizeof(int));
  cudaMalloc(&x, 256 * sizeof(double));
  cudaMemset(counter, 0, sizeof(int));
  cudaMemset(x, 0, 256 * sizeof(double));
  cudaGraph_t g;
  cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  printf("handle create: %s\n", cudaGetErrorString(e));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  printf("add node: %s\n", cudaGetErrorString(e));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  printf("begin capture: %s\n", cudaGetErrorString(e));
  work_kernel<<<1, 256, 0, s>>>(x);
  cudaMemsetAsync(x + 255, 0, sizeof(double), s);
  body_kernel<<<1, 1, 0, s>>>(counter, 50, h);
  cudaGraph_t captured;
  e = cudaStreamEndCapture(s, &captured);
  printf("end capture: %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ge;
  e = cudaGraphInstantiate(&ge, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  e = cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaStreamSynchronize(s);
  printf("launch: %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  int c = 0;
  double x0 = 0;
  cudaMemcpy(&c, counter, sizeof(int), cudaMemcpyDeviceToHost);
  cudaMemcpy(&x0, x, sizeof(double), cudaMemcpyDeviceToHost);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("iterations %d, x[0] %.0f, %.2f us per iteration\n", c, x0, ms * 1e3 / c);
  return 0;
}
