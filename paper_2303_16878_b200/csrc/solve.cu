// K3: the LM linear solve  (H + lam * diag(H)) delta = -b
// Reference: np.linalg.solve(damped, -b) (LAPACK gesv) at solver.py:510-512.
//
// The damped normal matrix is symmetric positive definite whenever the
// reference's LU succeeds (H is a sum of J^T W J with W > 0 and lam > 0), so
// the device path factors it with a tiled right-looking fp64 Cholesky:
//   per 64-column panel k:  potrf(diagonal tile) -> trsm(panel) -> syrk/gemm(trailing)
// A per-tile non-zero map (filled after damping, updated as fill-in appears)
// lets every kernel skip structurally-zero tiles, so block-banded systems
// (corridor trajectories) cost O(n * band^2) instead of
// O(n^3) while general graphs get the full dense factorisation.  A status
// word reports a non-positive pivot — the reference's LinAlgError path
// (solver.py:513-522).

#include <math.h>

#include "pba_common.cuh"

namespace pba {
namespace {

constexpr int NB = 64;  // tile size

struct SolveWork {
  double* A;      // dim x dim (lower triangle used)
  double* y;      // dim
  int32_t* nz;    // T x T tile non-zero flags
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

SolveWork carve(void* work, int dim) {
  const int T = (dim + NB - 1) / NB;
  char* p = static_cast<char*>(work);
  SolveWork w;
  w.A = reinterpret_cast<double*>(p);
  p += align_up((size_t)dim * dim * sizeof(double), 256);
  w.y = reinterpret_cast<double*>(p);
  p += align_up((size_t)dim * sizeof(double), 256);
  w.nz = reinterpret_cast<int32_t*>(p);
  (void)T;
  return w;
}

__global__ void damp_copy_kernel(const double* __restrict__ H, int dim, double lam,
                                 double* __restrict__ A) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)dim * dim) return;
  const int i = (int)(t / dim), j = (int)(t - (long)i * dim);
  if (j > i) return;
  const double h = H[t];
  A[t] = (i == j) ? h + lam * h : h;  // h + lam * np.diag(np.diag(h))
}

// One CTA per lower tile: flag it if any entry is non-zero.
__global__ void tile_flags_kernel(const double* __restrict__ A, int dim, int T,
                                  int32_t* __restrict__ nz) {
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bj > bi) {
    if (threadIdx.x == 0) nz[bi * T + bj] = 0;
    return;
  }
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  int mine = 0;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = bi * NB + e / NB, c = bj * NB + e % NB;
    if (r < dim && c < dim && c <= r && A[(long)r * dim + c] != 0.0) mine = 1;
  }
  if (mine) any = 1;
  __syncthreads();
  if (threadIdx.x == 0) nz[bi * T + bj] = any || bi == bj;
}

// Unblocked Cholesky of diagonal tile k in shared memory (one CTA).
__global__ void potrf_kernel(double* __restrict__ A, int dim, int k, int32_t* __restrict__ status) {
  __shared__ double a[NB][NB + 1];
  __shared__ int bad;
  if (*status) return;
  const int k0 = k * NB;
  const int n = min(NB, dim - k0);
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    a[r][c] = (r < n && c <= r) ? A[(long)(k0 + r) * dim + k0 + c] : 0.0;
  }
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double d = a[j][j];
      if (!(d > 0.0) || !isfinite(d)) bad = 1;
      a[j][j] = sqrt(d);
    }
    __syncthreads();
    if (bad) break;
    const double piv = a[j][j];
    for (int r = j + 1 + threadIdx.x; r < n; r += blockDim.x) a[r][j] /= piv;
    __syncthreads();
    const int m = n - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int r = j + 1 + e / m, c = j + 1 + e % m;
      if (c <= r) a[r][c] -= a[r][j] * a[c][j];
    }
    __syncthreads();
  }
  if (bad) {
    if (threadIdx.x == 0) *status = 1;
    return;
  }
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    if (r < n && c <= r) A[(long)(k0 + r) * dim + k0 + c] = a[r][c];
  }
}

// L21 = A21 * L11^{-T} for row tiles bi > k with a non-zero (bi, k) tile.
// One CTA per row tile; each thread owns one row and substitutes forward.
__global__ void trsm_kernel(double* __restrict__ A, int dim, int k, int T,
                            const int32_t* __restrict__ nz, const int32_t* __restrict__ status) {
  if (*status) return;
  const int bi = k + 1 + blockIdx.x;
  if (!nz[bi * T + k]) return;
  extern __shared__ double tsm[];
  double(*L)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(tsm);
  double(*X)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(tsm + NB * (NB + 1));
  const int k0 = k * NB, r0 = bi * NB;
  const int nk = min(NB, dim - k0), nr = min(NB, dim - r0);
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    L[r][c] = (r < nk && c <= r) ? A[(long)(k0 + r) * dim + k0 + c] : 0.0;
    X[r][c] = (r < nr && c < nk) ? A[(long)(r0 + r) * dim + k0 + c] : 0.0;
  }
  __syncthreads();
  const int r = threadIdx.x;
  if (r < nr) {
    for (int j = 0; j < nk; ++j) {
      double s = X[r][j];
      for (int m = 0; m < j; ++m) s -= X[r][m] * L[j][m];
      X[r][j] = s / L[j][j];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int rr = e / NB, c = e % NB;
    if (rr < nr && c < nk) A[(long)(r0 + rr) * dim + k0 + c] = X[rr][c];
  }
}

// Trailing update C(bi,bj) -= L(bi,k) L(bj,k)^T for bi >= bj > k.  One CTA
// (256 threads, 4x4 outputs each) per lower tile; skipped when either panel
// tile is zero.  Marks the target tile non-zero (fill-in).
__global__ void __launch_bounds__(256) syrk_kernel(double* __restrict__ A, int dim, int k, int T,
                                                   int32_t* __restrict__ nz,
                                                   const int32_t* __restrict__ status) {
  if (*status) return;
  // blockIdx.x enumerates lower tiles of the trailing (T-k-1)^2 matrix.
  const int m = T - k - 1;
  const int t = blockIdx.x;
  // invert t = bi*(bi+1)/2 + bj with 0 <= bj <= bi < m
  int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  while (bi * (bi + 1) / 2 > t) --bi;
  const int bj = t - bi * (bi + 1) / 2;
  if (bi >= m) return;
  const int ti = k + 1 + bi, tj = k + 1 + bj;
  if (!nz[ti * T + k] || !nz[tj * T + k]) return;
  extern __shared__ double smem[];
  double* Pi = smem;               // NB x (NB+1)
  double* Pj = smem + NB * (NB + 1);
  const int k0 = k * NB, ri = ti * NB, rj = tj * NB;
  const int nk = min(NB, dim - k0);
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    Pi[r * (NB + 1) + c] = (ri + r < dim && c < nk) ? A[(long)(ri + r) * dim + k0 + c] : 0.0;
    Pj[r * (NB + 1) + c] = (rj + r < dim && c < nk) ? A[(long)(rj + r) * dim + k0 + c] : 0.0;
  }
  __syncthreads();
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
  for (int kk = 0; kk < NB; ++kk) {
    double x[4], y[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      x[a] = Pi[(tr + 16 * a) * (NB + 1) + kk];
      y[a] = Pj[(tc + 16 * a) * (NB + 1) + kk];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c] += x[a] * y[c];
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int r = ri + tr + 16 * a, col = rj + tc + 16 * c;
      if (r < dim && col < dim && col <= r) A[(long)r * dim + col] -= acc[a][c];
    }
  if (threadIdx.x == 0) nz[ti * T + tj] = 1;
}

// Forward (L y = -b) and backward (L^T x = y) substitution in one CTA,
// tile by tile, skipping zero tiles.
__global__ void __launch_bounds__(1024) trisolve_kernel(const double* __restrict__ A, int dim, int T,
                                                         const int32_t* __restrict__ nz,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ y,
                                                         double* __restrict__ x,
                                                         const int32_t* __restrict__ status) {
  if (*status) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  for (int i = tid; i < dim; i += blockDim.x) y[i] = -b[i];
  __syncthreads();
  // forward
  for (int k = 0; k < T; ++k) {
    const int k0 = k * NB, nk = min(NB, dim - k0);
    if (warp == 0) {
      for (int j = 0; j < nk; ++j) {
        const double yj = y[k0 + j] / A[(long)(k0 + j) * dim + k0 + j];
        __syncwarp();
        if (lane == 0) y[k0 + j] = yj;
        for (int r = j + 1 + lane; r < nk; r += 32) y[k0 + r] -= A[(long)(k0 + r) * dim + k0 + j] * yj;
        __syncwarp();
      }
    }
    __syncthreads();
    // update rows of non-zero tiles below
    for (int bi = k + 1; bi < T; ++bi) {
      if (!nz[bi * T + k]) continue;
      const int r0 = bi * NB, nr = min(NB, dim - r0);
      for (int r = warp; r < nr; r += nwarp) {
        const double* row = A + (long)(r0 + r) * dim + k0;
        double s = 0.0;
        for (int c = lane; c < nk; c += 32) s += row[c] * y[k0 + c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) y[r0 + r] -= s;
      }
    }
    __syncthreads();
  }
  // backward: x = L^{-T} y
  for (int i = tid; i < dim; i += blockDim.x) x[i] = y[i];
  __syncthreads();
  for (int k = T - 1; k >= 0; --k) {
    const int k0 = k * NB, nk = min(NB, dim - k0);
    // subtract contributions of already-solved tiles below: x_k -= L(bi,k)^T x_bi
    for (int c = tid; c < nk; c += blockDim.x) {
      double s = 0.0;
      for (int bi = k + 1; bi < T; ++bi) {
        if (!nz[bi * T + k]) continue;
        const int r0 = bi * NB, nr = min(NB, dim - r0);
        for (int r = 0; r < nr; ++r) s += A[(long)(r0 + r) * dim + k0 + c] * x[r0 + r];
      }
      x[k0 + c] -= s;
    }
    __syncthreads();
    if (warp == 0) {
      for (int j = nk - 1; j >= 0; --j) {
        const double xj = x[k0 + j] / A[(long)(k0 + j) * dim + k0 + j];
        __syncwarp();
        if (lane == 0) x[k0 + j] = xj;
        for (int r = lane; r < j; r += 32) x[k0 + r] -= A[(long)(k0 + j) * dim + k0 + r] * xj;
        __syncwarp();
      }
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" size_t pba_solve_work_bytes(int32_t dim) {
  if (dim <= 0) return 0;
  const size_t T = (dim + NB - 1) / NB;
  return align_up((size_t)dim * dim * sizeof(double), 256) +
         align_up((size_t)dim * sizeof(double), 256) + align_up(T * T * sizeof(int32_t), 256);
}

extern "C" int pba_solve_dense(const double* H, const double* b, int32_t dim, double lam,
                               void* work, double* delta, int32_t* status, void* stream) {
  PBA_ARG_CHECK(dim > 0, "dim must be positive");
  PBA_ARG_CHECK(H && b && work && delta && status, "NULL buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SolveWork w = carve(work, dim);
  const int T = (dim + NB - 1) / NB;
  PBA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  const long n2 = (long)dim * dim;
  damp_copy_kernel<<<(unsigned)((n2 + 255) / 256), 256, 0, st>>>(H, dim, lam, w.A);
  PBA_LAUNCH_CHECK();
  tile_flags_kernel<<<dim3(T, T), 256, 0, st>>>(w.A, dim, T, w.nz);
  PBA_LAUNCH_CHECK();
  const int syrk_smem = 2 * NB * (NB + 1) * sizeof(double);
  PBA_CUDA_TRY(cudaFuncSetAttribute(syrk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    syrk_smem));
  PBA_CUDA_TRY(cudaFuncSetAttribute(trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    syrk_smem));
  for (int k = 0; k < T; ++k) {
    potrf_kernel<<<1, 256, 0, st>>>(w.A, dim, k, status);
    PBA_LAUNCH_CHECK();
    const int m = T - k - 1;
    if (m > 0) {
      trsm_kernel<<<m, NB, syrk_smem, st>>>(w.A, dim, k, T, w.nz, status);
      PBA_LAUNCH_CHECK();
      syrk_kernel<<<m * (m + 1) / 2, 256, syrk_smem, st>>>(w.A, dim, k, T, w.nz, status);
      PBA_LAUNCH_CHECK();
    }
  }
  trisolve_kernel<<<1, 1024, 0, st>>>(w.A, dim, T, w.nz, b, w.y, delta, status);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
