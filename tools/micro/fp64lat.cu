// Microbenchmark: fp64 dependent-chain latency and throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void indep(double* out, double a, double b, int n, long long* cyc) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void fchain(float* out, float a, float b, int n, long long* cyc) {
  float x = threadIdx.x * 1e-3f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x = fmaf(x, a, b); x = fmaf(x, a, b); x = fmaf(x, a, b); x = fmaf(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void divchain(double* out, double a, int n, long long* cyc) {
  double x = threadIdx.x + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = a / x + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void sqrtchain(double* out, int n, long long* cyc) {
  double x = threadIdx.x + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&f, 1 << 20); cudaMalloc(&c, 8);
  const int n = 4096;
  chain<<<1, 32>>>(d, 1.0000001, 1e-9, n, c); cudaDeviceSynchronize();
  chain<<<1, 32>>>(d, 1.0000001, 1e-9, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  fchain<<<1, 32>>>(f, 1.0000001f, 1e-9f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  for (int w : {1, 2, 4, 8, 16}) {
    indep<<<1, 32 * w>>>(d, 1.0000001, 1e-9, n, c); cudaDeviceSynchronize();
    indep<<<1, 32 * w>>>(d, 1.0000001, 1e-9, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 8 indep chains, %2d warps/SM: %.2f cycles per warp-DFMA per SM (%.1f lanes/clk)\n", w,
           (double)h / (8.0 * n * w), 32.0 * 8.0 * n * w / (double)h);
  }
  divchain<<<1, 32>>>(d, 3.0, n, c); cudaDeviceSynchronize();
  divchain<<<1, 32>>>(d, 3.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp64 divide+add dependent latency: %.1f cycles\n", (double)h / n);
  sqrtchain<<<1, 32>>>(d, n, c); cudaDeviceSynchronize();
  sqrtchain<<<1, 32>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp64 sqrt+add dependent latency: %.1f cycles\n", (double)h / n);
  return 0;
}
