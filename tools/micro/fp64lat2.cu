#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_nr(double x) {
  double r = (double)__frcp_rn((float)x);
  r = fma(r, fma(-x, r, 1.0), r); r = fma(r, fma(-x, r, 1.0), r); r = fma(r, fma(-x, r, 1.0), r);
  return r;
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y = (double)rsqrtf((float)x);
  double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5); y = y * fma(-h * y, y, 1.5); y = y * fma(-h * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rsqrt_nr2(double x) {  // seed + 2 steps (quartic)
  double y = (double)rsqrtf((float)x);
  double e = fma(-x * y, y, 1.0);           // e = 1 - x y^2
  y = fma(y * e, fma(0.375, e, 0.5), y);    // y (1 + e/2 + 3e^2/8)
  e = fma(-x * y, y, 1.0);
  y = fma(y * e, fma(0.375, e, 0.5), y);
  return y;
}
#define CHAIN(name, expr) \
__global__ void name(double* out, int n, long long* cyc) { \
  double x = threadIdx.x + 1.5; long long t0 = clock64(); \
  for (int i = 0; i < n; ++i) x = (expr) + 1.0; \
  long long t1 = clock64(); out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0; }
CHAIN(k_div, 3.0 / x)
CHAIN(k_rcp_rn, __drcp_rn(x))
CHAIN(k_rcp_nr, rcp_nr(x))
CHAIN(k_sqrt, sqrt(x))
CHAIN(k_rsqrt, rsqrt(x))
CHAIN(k_rsqrt_nr, rsqrt_nr(x))
CHAIN(k_rsqrt_nr2, rsqrt_nr2(x))
CHAIN(k_dsqrt_rn, __dsqrt_rn(x))
typedef void (*K)(double*, int, long long*);
int main() {
  double* d; long long* c; long long h; const int n = 2048;
  cudaMalloc(&d, 1 << 20); cudaMalloc(&c, 8);
  const char* names[] = {"3.0/x", "__drcp_rn", "rcp_nr(3 NR)", "sqrt", "rsqrt", "rsqrt_nr(3 NR)", "rsqrt_nr2(2 quartic)", "__dsqrt_rn"};
  K ks[] = {k_div, k_rcp_rn, k_rcp_nr, k_sqrt, k_rsqrt, k_rsqrt_nr, k_rsqrt_nr2, k_dsqrt_rn};
  for (int i = 0; i < 8; ++i) {
    ks[i]<<<1, 32>>>(d, n, c); cudaDeviceSynchronize();
    ks[i]<<<1, 32>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-22s + add: %.1f cycles\n", names[i], (double)h / n);
  }
  // accuracy of rsqrt variants vs 1/sqrt on host
  return 0;
}
