// DMMA (fp64 mma.sync) throughput on B200: m8n8k4 and m16n8k16.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma16816(double* out, int iters) {
  double a[8], b[4];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int k = 0; k < 4; ++k) b[k] = 1.0 + threadIdx.x * 1e-4 + k;
  double c[2][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int k = 0; k < 2; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_peak(double* out, int iters) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  const double m = 1.0000001, ad = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], m, ad);
  }
  double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.0) out[0] = s;
}

// Both streams in the same warps: per iteration NM m8n8k4 DMMAs and NF
// independent DFMAs (NF / 8 rounds over 8 accumulators).  If DMMA and DFMA
// run on separate pipes the time is max(t_mma, t_fma); on one shared pipe it
// is t_mma + t_fma.
template <int NM, int NF>
__global__ void mixed(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  const double m = 1.0000001, ad = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NM; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int r = 0; r < NF / 8; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], m, ad);
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.0) out[0] = s;
}

template <int NM, int NF>
float time_mixed(double* out, int blocks, int threads, int iters, cudaEvent_t e0, cudaEvent_t e1) {
  mixed<NM, NF><<<blocks, threads>>>(out, 16);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  mixed<NM, NF><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  float ms;
  dmma884<<<blocks, threads>>>(out, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); dmma884<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 8 * 8 * 4 * 4.0 * iters * blocks * (threads / 32);
  printf("m8n8k4   : %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  dmma16816<<<blocks, threads>>>(out, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); dmma16816<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 16 * 8 * 16 * 2.0 * iters * blocks * (threads / 32);
  printf("m16n8k16 : %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  dfma_peak<<<blocks, threads>>>(out, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); dfma_peak<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 8.0 * iters * blocks * threads;
  printf("DFMA     : %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  // concurrency: 4 DMMA alone, 32 DFMA alone, both together (per warp-iteration)
  const float tm = time_mixed<4, 0>(out, blocks, threads, iters, e0, e1);
  const float tf = time_mixed<0, 32>(out, blocks, threads, iters, e0, e1);
  const float tb = time_mixed<4, 32>(out, blocks, threads, iters, e0, e1);
  printf("mixed: 4 DMMA %.3f ms, 32 DFMA %.3f ms, both %.3f ms (sum %.3f, max %.3f) -> %s\n",
         tm, tf, tb, tm + tf, tm > tf ? tm : tf,
         tb < 0.75f * (tm + tf) ? "overlap (separate pipes)" : "no overlap (shared pipe)");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
