// K3b: block-Jacobi preconditioned conjugate gradients for the LM system
//   (H + lam * diag(H)) delta = -b
// the iterative alternative of App. C's c3 configuration ("LM with
// block-Jacobi PCG").  The reference solves exactly (np.linalg.solve,
// solver.py:510-512); PCG run to a tight relative residual gives the same
// step to that tolerance, and a looser one gives the inexact-LM step that the
// accept/reject test of solver.py:524-531 then judges.
//
// The whole solve is ONE persistent cooperative kernel: up to one CTA per
// resident slot, each owning a contiguous range of 6x6 block rows, 8 block
// rows per pass (48 scalar rows; in the mat-vec 4 adjacent lanes split each
// row's neighbour blocks, so 192 threads keep 4 L2 loads in flight per row).  H stays where the
// assembly wrote it (dense, row-major) and the mat-vec reads only the
// structurally non-zero blocks (block-row CSR built once per level from the
// pair list: the diagonal block plus one block per neighbouring pose).  Per
// iteration two grid barriers:
//   phase 1: x += a p, r -= a q, z = M^-1 r            -> partial r.r, r.z
//   phase 2: beta, p = z + beta p, q = A z + beta q    -> partial p.q
// (q = A p is carried by linearity, so the mat-vec reads z, which phase 1
// finished everywhere before the barrier).  Dot products are reduced per
// CTA by a fixed tree and across CTAs by every CTA summing the same partials
// in the same order, so the result is deterministic and every CTA takes the
// same convergence decision without a broadcast.

#include <cooperative_groups.h>
#include <math.h>

#include "pba_common.cuh"

namespace cg = cooperative_groups;

namespace pba {
namespace {

constexpr int kPcgRows = 8;   // block rows per CTA pass
constexpr int kSplit = 4;     // lanes per scalar row in the mat-vec (neighbour blocks split)
constexpr int kPcgThreads = 6 * kPcgRows * kSplit;
constexpr int kPcgWarps = kPcgThreads / 32;
constexpr int kMaxPasses = 4;  // block-row passes per CTA (vectors live in registers)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct PcgWork {
  double* minv;      // n_free x 36: inverses of the damped diagonal blocks
  double* x;         // dim
  double* r;         // dim
  double* p;         // dim
  double* q;         // dim
  double* z;         // dim
  double* partials;  // grid x 4
};

PcgWork carve(void* work, int n_free, int grid) {
  const size_t dim = 6 * (size_t)n_free;
  char* c = static_cast<char*>(work);
  PcgWork w;
  w.minv = reinterpret_cast<double*>(c);
  c += align_up(36 * (size_t)n_free * sizeof(double), 256);
  double** vecs[5] = {&w.x, &w.r, &w.p, &w.q, &w.z};
  for (double** v : vecs) {
    *v = reinterpret_cast<double*>(c);
    c += align_up(dim * sizeof(double), 256);
  }
  w.partials = reinterpret_cast<double*>(c);
  return w;
}

// Fixed-order CTA reduction of two values; thread 0 gets the sums.
__device__ void cta_sum2(double& a, double& b, double (*sm)[kPcgWarps]) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) {
    sm[0][warp] = a;
    sm[1][warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0.0;
    b = 0.0;
    for (int k = 0; k < kPcgWarps; ++k) {
      a += sm[0][k];
      b += sm[1][k];
    }
  }
}

// Sum of partials[g * 4 + slot] over all CTAs, in CTA order (warp 0 loads
// with a fixed lane assignment, fixed butterfly); broadcast through smem.
__device__ double grid_sum(const double* partials, int grid, int slot, double* bcast) {
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int g = threadIdx.x; g < grid; g += 32) s += __ldcg(partials + 4 * g + slot);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *bcast = s;
  }
  __syncthreads();
  const double v = *bcast;
  __syncthreads();
  return v;
}

// 6x6 SPD inverse by Cholesky; false when a pivot is not positive.
__device__ bool spd_inverse6(const double* a, double* inv) {
  double L[6][6];
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) L[i][j] = 0.0;
  for (int j = 0; j < 6; ++j) {
    double d = a[6 * j + j];
    for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
    if (!(d > 0.0)) return false;
    L[j][j] = sqrt(d);
    for (int i = j + 1; i < 6; ++i) {
      double s = a[6 * i + j];
      for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
      L[i][j] = s / L[j][j];
    }
  }
  // columns of L^-1, then inv = L^-T L^-1
  double Li[6][6];
  for (int c = 0; c < 6; ++c) {
    for (int i = 0; i < 6; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= L[i][k] * Li[k][c];
      Li[i][c] = (i < c) ? 0.0 : s / L[i][i];
    }
  }
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      double s = 0.0;
      for (int k = (i > j ? i : j); k < 6; ++k) s += Li[k][i] * Li[k][j];
      inv[6 * i + j] = s;
    }
  return true;
}

// Part of (H x)_row over every kSplit-th non-zero block of the row, starting
// at block `sp`; the kSplit lanes of a row are adjacent and are combined by
// a fixed butterfly in matvec_pass.
// H is either the dense matrix (bsr false: row-major dim x dim) or the
// block-sparse one (bsr true: 6x6 blocks in the order of the block-row CSR
// row_ptr / cols, Hb[e * 36 + 6 k + l], pba_assemble_bsr).
__device__ __forceinline__ double row_part(const double* __restrict__ H, long dim, bool bsr,
                                           const int32_t* __restrict__ row_ptr,
                                           const int32_t* __restrict__ cols, int br, int k,
                                           int sp, const double* v) {
  const double* h = H + (6L * br + k) * dim;
  double acc = 0.0;
  const int e1 = row_ptr[br + 1];
#pragma unroll 2
  for (int e = row_ptr[br] + sp; e < e1; e += kSplit) {
    const int c = PBA_DCHECK_INDEX(__ldg(cols + e), dim / 6);
    const double* hb = bsr ? H + 36L * e + 6 * k : h + 6L * c;
    const double* vb = v + 6L * c;
#pragma unroll
    for (int l = 0; l < 6; ++l) acc = fma(__ldg(hb + l), __ldcg(vb + l), acc);
  }
  return acc;
}

// mv[lr * 6 + k] = ((H + lam diag H) v)_row for the pass's block rows; all
// threads call it (the butterfly is warp-wide), a __syncthreads follows.
__device__ __forceinline__ double hdiag(const double* __restrict__ H, long dim,
                                        const int32_t* __restrict__ diag_blk, int br, int i,
                                        int j) {
  return diag_blk ? __ldg(H + 36L * diag_blk[br] + 6 * i + j)
                  : __ldg(H + (6L * br + i) * dim + 6L * br + j);
}

__device__ __forceinline__ void matvec_pass(const double* __restrict__ H, long dim,
                                            const int32_t* __restrict__ diag_blk, double lam,
                                            const int32_t* __restrict__ row_ptr,
                                            const int32_t* __restrict__ cols, int base, int br1,
                                            const double* v, double* mv) {
  const int t = threadIdx.x;
  const int lr = t / (6 * kSplit), k = (t / kSplit) % 6, sp = t % kSplit;
  const int br = base + lr;
  double acc = br < br1 ? row_part(H, dim, diag_blk != nullptr, row_ptr, cols, br, k, sp, v)
                        : 0.0;
#pragma unroll
  for (int o = 1; o < kSplit; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (sp == 0 && br < br1) {
    const long row = 6L * br + k;
    mv[lr * 6 + k] = fma(lam * hdiag(H, dim, diag_blk, br, k, k), __ldcg(v + row), acc);
  }
}

// Sums of two partial slots over all CTAs (see grid_sum), one L2 round trip.
__device__ void grid_sum2(const double* partials, int grid, int s0, int s1, double* bc,
                          double& a, double& b) {
  if (threadIdx.x < 32) {
    double u = 0.0, v = 0.0;
    for (int g = threadIdx.x; g < grid; g += 32) {
      u += __ldcg(partials + 4 * g + s0);
      v += __ldcg(partials + 4 * g + s1);
    }
    for (int o = 16; o > 0; o >>= 1) {
      u += __shfl_xor_sync(0xffffffffu, u, o);
      v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    if (threadIdx.x == 0) {
      bc[0] = u;
      bc[1] = v;
    }
  }
  __syncthreads();
  a = bc[0];
  b = bc[1];
  __syncthreads();
}

__global__ void __launch_bounds__(kPcgThreads)
    pcg_kernel(const double* __restrict__ H, const double* __restrict__ b, int n_free,
               double lam_arg, const double* __restrict__ lam_dev,
               const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols,
               const int32_t* __restrict__ diag_blk,
               int max_iter, double tol, PcgWork w, double* __restrict__ delta,
               int32_t* __restrict__ status, double* __restrict__ info) {
  cg::grid_group grid = cg::this_grid();
  const double lam = lam_dev ? *lam_dev : lam_arg;  // device lambda: graph-replayable step
  __shared__ double red[2][kPcgWarps];
  __shared__ double mv[6 * kPcgRows];  // mat-vec results of the pass
  __shared__ double rb[6 * kPcgRows];  // residual of the pass (block-Jacobi needs whole blocks)
  __shared__ double bc[2];
  __shared__ int bad;
  const int G = gridDim.x;
  const long dim = 6L * n_free;
  const int per = (n_free + G - 1) / G;
  const int br0 = min(n_free, (int)blockIdx.x * per), br1 = min(n_free, br0 + per);
  const int passes = (br1 - br0 + kPcgRows - 1) / kPcgRows;  // <= kMaxPasses (host-checked)
  // vector role: threads [0, 6 kPcgRows) own one scalar row per pass; the
  // CTA's x, r, p, q, z and block-Jacobi rows stay in their registers, only
  // z goes to global memory (the neighbours' mat-vec reads it)
  const bool vec = threadIdx.x < 6 * kPcgRows;
  const int lr = threadIdx.x / 6, k = threadIdx.x - 6 * (threadIdx.x / 6);
  double mi[kMaxPasses][6], xv[kMaxPasses], rv[kMaxPasses], pv[kMaxPasses], qv[kMaxPasses],
      zv[kMaxPasses];

  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
#pragma unroll
  for (int ps = 0; ps < kMaxPasses; ++ps) {
    const int br = br0 + ps * kPcgRows + lr;
    if (ps < passes && vec && k == 0 && br < br1) {
      double a[36];
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
          const double h = hdiag(H, dim, diag_blk, br, i, j);
          a[6 * i + j] = (i == j) ? h + lam * h : h;
        }
      if (!spd_inverse6(a, w.minv + 36L * br)) bad = 1;
    }
  }
  __syncthreads();
  // x = 0, r = -b, z = M^-1 r, p = z
  double bb = 0.0, rz = 0.0;
#pragma unroll
  for (int ps = 0; ps < kMaxPasses; ++ps) {
    xv[ps] = rv[ps] = pv[ps] = qv[ps] = zv[ps] = 0.0;
    if (ps < passes) {
      const int br = br0 + ps * kPcgRows + lr;
      const long row = 6L * br + k;
      const bool own = vec && br < br1;
      if (own) {
#pragma unroll
        for (int l = 0; l < 6; ++l) mi[ps][l] = w.minv[36L * br + 6 * k + l];
        rv[ps] = -b[row];
        bb = fma(rv[ps], rv[ps], bb);
        rb[threadIdx.x] = rv[ps];
      }
      __syncthreads();
      if (own) {
        double z = 0.0;
#pragma unroll
        for (int l = 0; l < 6; ++l) z = fma(mi[ps][l], rb[6 * lr + l], z);
        zv[ps] = pv[ps] = z;
        w.z[row] = z;
        rz = fma(rv[ps], z, rz);
      }
      __syncthreads();
    }
  }
  cta_sum2(bb, rz, red);
  if (threadIdx.x == 0) {
    w.partials[4 * blockIdx.x + 0] = bb;
    w.partials[4 * blockIdx.x + 1] = rz;
    w.partials[4 * blockIdx.x + 3] = bad ? 1.0 : 0.0;
  }
  grid.sync();
  double flag = 0.0;
  grid_sum2(w.partials, G, 3, 0, bc, flag, bb);
  if (flag != 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *status = 1;  // non-SPD diagonal block
    return;
  }
  rz = grid_sum(w.partials, G, 1, bc);
  const double stop = tol * tol * bb;
  // q = A p (p = z, already global)
  double pq = 0.0, dummy = 0.0;
#pragma unroll
  for (int ps = 0; ps < kMaxPasses; ++ps) {
    if (ps < passes) {
      const int base = br0 + ps * kPcgRows;
      matvec_pass(H, dim, diag_blk, lam, row_ptr, cols, base, br1, w.z, mv);
      __syncthreads();
      if (vec && base + lr < br1) {
        qv[ps] = mv[threadIdx.x];
        pq = fma(pv[ps], qv[ps], pq);
      }
      __syncthreads();
    }
  }
  cta_sum2(pq, dummy, red);
  if (threadIdx.x == 0) w.partials[4 * blockIdx.x + 2] = pq;
  grid.sync();

  int it = 0;
  double rr = bb;
  bool converged = bb == 0.0;
  while (!converged && it < max_iter) {
    ++it;
    // phase 1: x, r, z
    pq = grid_sum(w.partials, G, 2, bc);
    if (!(pq > 0.0)) {  // A not positive definite along p
      if (blockIdx.x == 0 && threadIdx.x == 0) *status = 1;
      return;
    }
    const double alpha = rz / pq;
    double rr_p = 0.0, rz_p = 0.0;
#pragma unroll
    for (int ps = 0; ps < kMaxPasses; ++ps) {
      if (ps < passes) {
        const int br = br0 + ps * kPcgRows + lr;
        const bool own = vec && br < br1;
        if (own) {
          xv[ps] = fma(alpha, pv[ps], xv[ps]);
          rv[ps] = fma(-alpha, qv[ps], rv[ps]);
          rr_p = fma(rv[ps], rv[ps], rr_p);
          rb[threadIdx.x] = rv[ps];
        }
        __syncthreads();
        if (own) {
          double z = 0.0;
#pragma unroll
          for (int l = 0; l < 6; ++l) z = fma(mi[ps][l], rb[6 * lr + l], z);
          zv[ps] = z;
          w.z[6L * br + k] = z;
          rz_p = fma(rv[ps], z, rz_p);
        }
        __syncthreads();
      }
    }
    cta_sum2(rr_p, rz_p, red);
    if (threadIdx.x == 0) {
      w.partials[4 * blockIdx.x + 0] = rr_p;
      w.partials[4 * blockIdx.x + 1] = rz_p;
    }
    grid.sync();
    // phase 2: beta, p, q = A z + beta q
    double rz_new;
    grid_sum2(w.partials, G, 0, 1, bc, rr, rz_new);
    if (rr <= stop) {
      converged = true;
      break;
    }
    const double beta = rz_new / rz;
    rz = rz_new;
    double pq_p = 0.0;
#pragma unroll
    for (int ps = 0; ps < kMaxPasses; ++ps) {
      if (ps < passes) {
        const int base = br0 + ps * kPcgRows;
        matvec_pass(H, dim, diag_blk, lam, row_ptr, cols, base, br1, w.z, mv);
        __syncthreads();
        if (vec && base + lr < br1) {
          pv[ps] = fma(beta, pv[ps], zv[ps]);
          qv[ps] = fma(beta, qv[ps], mv[threadIdx.x]);
          pq_p = fma(pv[ps], qv[ps], pq_p);
        }
        __syncthreads();
      }
    }
    cta_sum2(pq_p, dummy, red);
    if (threadIdx.x == 0) w.partials[4 * blockIdx.x + 2] = pq_p;
    grid.sync();
  }
#pragma unroll
  for (int ps = 0; ps < kMaxPasses; ++ps) {
    const int br = br0 + ps * kPcgRows + lr;
    if (ps < passes && vec && br < br1) delta[6L * br + k] = xv[ps];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    info[0] = (double)it;
    info[1] = bb > 0.0 ? sqrt(rr / bb) : 0.0;
    info[2] = converged ? 1.0 : 0.0;
  }
}

int pcg_cap() {
  static int cap = 0;
  if (cap == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_kernel, kPcgThreads, 0) !=
            cudaSuccess)
      return 0;
    cap = sms * (per_sm < 1 ? 1 : per_sm);
  }
  return cap;
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" size_t pba_pcg_work_bytes(int32_t n_free) {
  if (n_free <= 0) return 0;
  const size_t dim = 6 * (size_t)n_free;
  const size_t max_grid = 148 * 16;  // >= any cooperative grid on one B200
  return align_up(36 * (size_t)n_free * sizeof(double), 256) +
         5 * align_up(dim * sizeof(double), 256) + align_up(4 * max_grid * sizeof(double), 256);
}

namespace {
int solve_pcg_impl(const double* H, const double* b, int32_t n_free, double lam,
                   const double* lam_dev, const int32_t* row_ptr, const int32_t* cols,
                   const int32_t* diag_blk, int32_t max_iter, double tol, void* work,
                   double* delta, int32_t* status, double* info, void* stream) {
  PBA_ARG_CHECK(n_free > 0, "n_free must be positive");
  PBA_ARG_CHECK(max_iter >= 1 && tol >= 0.0, "bad iteration limit or tolerance");
  PBA_ARG_CHECK(H && b && row_ptr && cols && work && delta && status && info, "NULL buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cap = pcg_cap();
  if (cap <= 0) {
    set_error("pba_solve_pcg: occupancy query failed");
    return PBA_ERR_CUDA;
  }
  const int want = (n_free + kPcgRows - 1) / kPcgRows;  // one pass per CTA when it fits
  const int grid = want < cap ? want : cap;
  const int per = (n_free + grid - 1) / grid;
  PBA_ARG_CHECK((per + kPcgRows - 1) / kPcgRows <= kMaxPasses,
                "system too large for the register-resident PCG (n_free > 32 x resident CTAs)");
  PBA_ARG_CHECK(grid <= 148 * 16, "cooperative grid larger than the work buffer allows");
  PcgWork w = carve(work, n_free, grid);
  PBA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  void* args[] = {(void*)&H,       (void*)&b,       (void*)&n_free, (void*)&lam,
                  (void*)&lam_dev, (void*)&row_ptr, (void*)&cols,   (void*)&diag_blk,
                  (void*)&max_iter, (void*)&tol,    (void*)&w,      (void*)&delta,
                  (void*)&status,  (void*)&info};
  PBA_CUDA_TRY(cudaLaunchCooperativeKernel((void*)pcg_kernel, dim3(grid), dim3(kPcgThreads), args,
                                           0, st));
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
}  // namespace

extern "C" int pba_solve_pcg_ex(const double* H, const double* b, int32_t n_free, double lam,
                                const double* lam_dev, const int32_t* row_ptr,
                                const int32_t* cols, int32_t max_iter, double tol, void* work,
                                double* delta, int32_t* status, double* info, void* stream) {
  return solve_pcg_impl(H, b, n_free, lam, lam_dev, row_ptr, cols, nullptr, max_iter, tol, work,
                        delta, status, info, stream);
}

extern "C" int pba_solve_pcg_bsr(const double* Hb, const double* b, int32_t n_free, double lam,
                                 const double* lam_dev, const int32_t* row_ptr,
                                 const int32_t* cols, const int32_t* diag_blk, int32_t max_iter,
                                 double tol, void* work, double* delta, int32_t* status,
                                 double* info, void* stream) {
  PBA_ARG_CHECK(diag_blk != nullptr, "NULL diag_blk");
  return solve_pcg_impl(Hb, b, n_free, lam, lam_dev, row_ptr, cols, diag_blk, max_iter, tol,
                        work, delta, status, info, stream);
}

extern "C" int pba_solve_pcg(const double* H, const double* b, int32_t n_free, double lam,
                             const int32_t* row_ptr, const int32_t* cols, int32_t max_iter,
                             double tol, void* work, double* delta, int32_t* status,
                             double* info, void* stream) {
  return pba_solve_pcg_ex(H, b, n_free, lam, nullptr, row_ptr, cols, max_iter, tol, work, delta,
                          status, info, stream);
}
