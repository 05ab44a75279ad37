// K3: the LM linear solve  (H + lam * diag(H)) delta = -b
// Reference: np.linalg.solve(damped, -b) (LAPACK gesv) at solver.py:510-512.
//
// The damped normal matrix is symmetric positive definite whenever the
// reference's LU succeeds (H is a sum of J^T W J with W > 0 and lam > 0), so
// the device path factors it with a tiled right-looking fp64 Cholesky on
// 64x64 tiles.  Per panel k:
//   potrf_inv : factor the diagonal tile in shared memory (8-column warp
//               panels, 16 CTA barriers) and form its explicit inverse
//   panel     : L_ik = A_ik L_kk^-T as a 64x64x64 product with that inverse
//   syrk      : trailing update A_ij -= L_ik L_jk^T
// A per-tile non-zero map (filled after damping, updated on fill-in) lets
// every kernel skip structurally zero tiles, so block-banded systems
// (corridor trajectories: bandwidth ~20 poses) cost O(n * band^2) while
// general graphs get the full factorisation.  The substitutions use the
// tile inverses: one CTA walks the tile rows, each step a short dot-product
// gather over the non-zero tiles plus a 64x64 mat-vec.
// A status word reports a non-positive pivot — the reference's LinAlgError
// path (solver.py:513-522).

#include <math.h>
#include <stdlib.h>

#include <vector>

#include "pba_common.cuh"

namespace pba {
namespace {

constexpr int NB = 64;  // tile size
constexpr int LD = NB + 1;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct SolveWork {
  double* A;     // D x D, D = NB * T (lower triangle used; the dense path uses dim x dim)
  double* Linv;  // T x NB x NB inverses of the diagonal tiles
  double* y;     // D
  double* bp;    // D: permuted right-hand side (dissection path)
  double* xp;    // D: permuted solution (dissection path)
  int32_t* lists;  // schedule of the dissection path (kListInts ints)
  int32_t* nz;   // T x T tile non-zero flags, then env / last (2T)
};

constexpr int kMaxBand = 3;  // dissection: widest tile band handled

// schedule buffer: new->old tile map, structural tiles, tile lists, pairs, triples
size_t list_ints(size_t T) {
  const size_t B = kMaxBand;
  return T * (4 + 2 * (2 * B + 1) + 4 * B + 3 * B * (2 * B + 1));
}

SolveWork carve(void* work, int dim) {
  const size_t T = (dim + NB - 1) / NB, D = T * NB;
  char* p = static_cast<char*>(work);
  SolveWork w;
  w.A = reinterpret_cast<double*>(p);
  p += align_up(D * D * sizeof(double), 256);
  w.Linv = reinterpret_cast<double*>(p);
  p += align_up(T * NB * NB * sizeof(double), 256);
  w.y = reinterpret_cast<double*>(p);
  p += align_up(D * sizeof(double), 256);
  w.bp = reinterpret_cast<double*>(p);
  p += align_up(D * sizeof(double), 256);
  w.xp = reinterpret_cast<double*>(p);
  p += align_up(D * sizeof(double), 256);
  w.lists = reinterpret_cast<int32_t*>(p);
  p += align_up(list_ints(T) * sizeof(int32_t), 256);
  w.nz = reinterpret_cast<int32_t*>(p);
  return w;
}

// H entry (r, c): dense row-major, or from the block-sparse matrix of
// pba_assemble_bsr (6x6 blocks in block-row CSR order; a block absent from
// the row's column list is zero).
struct HSource {
  const double* H;
  const int32_t* row_ptr;  // nullptr: dense
  const int32_t* cols;
  int dim;
  __device__ __forceinline__ double at(int r, int c) const {
    if (!row_ptr) return H[(long)r * dim + c];
    const int br = r / 6, bc = c / 6;
    int lo = row_ptr[br], hi = row_ptr[br + 1] - 1;
    while (lo <= hi) {  // columns ascending per block row
      const int mid = (lo + hi) >> 1;
      const int cm = cols[mid];
      if (cm == bc) return H[36L * mid + 6 * (r - 6 * br) + (c - 6 * bc)];
      if (cm < bc) lo = mid + 1; else hi = mid - 1;
    }
    return 0.0;
  }
};

__global__ void damp_copy_kernel(HSource H, int dim, double lam_arg,
                                 const double* __restrict__ lam_dev,
                                 const int32_t* __restrict__ env, double* __restrict__ A) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)dim * dim) return;
  const double lam = lam_dev ? *lam_dev : lam_arg;  // device lambda: graph-replayable step
  const int i = (int)(t / dim), j = (int)(t - (long)i * dim);
  if (j > i || j / NB < env[i / NB]) return;
  const double h = H.at(i, j);
  A[t] = (i == j) ? h + lam * h : h;  // h + lam * np.diag(np.diag(h))
}

// One CTA per lower tile: flag it if any entry is non-zero.  Tiles left of
// the row's envelope are structurally zero and never touched.
__global__ void tile_flags_kernel(const double* __restrict__ A, int dim, int T,
                                  const int32_t* __restrict__ env, int32_t* __restrict__ nz) {
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bj > bi || bj < env[bi]) {
    if (threadIdx.x == 0) nz[bi * T + bj] = 0;
    return;
  }
  int mine = 0;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = bi * NB + e / NB, c = bj * NB + e % NB;
    if (r < dim && c < dim && c <= r && A[(long)r * dim + c] != 0.0) mine = 1;
  }
  const int any = __syncthreads_or(mine);
  if (threadIdx.x == 0) nz[bi * T + bj] = any || bi == bj;
}

// Factor diagonal tile k in shared memory and store L_kk and L_kk^{-1}.
// 1024 threads.  Columns are processed in panels of 8: 64 threads (one row
// each) factor the panel between named barriers, then all threads apply the
// rank-8 update to the trailing part of the tile.
__global__ void __launch_bounds__(1024) potrf_inv_kernel(double* __restrict__ A, int dim, int k,
                                                        double* __restrict__ Linv,
                                                        int32_t* __restrict__ status) {
  extern __shared__ double psm[];
  double(*a)[LD] = reinterpret_cast<double(*)[LD]>(psm);
  double(*x)[LD] = reinterpret_cast<double(*)[LD]>(psm + NB * LD);
  __shared__ int bad;
  if (*status) return;
  const int tid = threadIdx.x;
  const int k0 = k * NB;
  const int n = min(NB, dim - k0);
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    a[r][c] = (r < n && c <= r) ? A[(long)(k0 + r) * dim + k0 + c] : (r == c ? 1.0 : 0.0);
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  __shared__ double rdiag[NB];
  for (int c0 = 0; c0 < n; c0 += 8) {
    const int c1 = min(c0 + 8, n);
    if (tid < NB) {
      // panel of 8 columns: thread r owns row r; steps are separated by a
      // 64-thread named barrier (warps 0-1 only)
      const int r = tid;
      for (int j = c0; j < c1; ++j) {
        if (r == j) {
          const double d = a[j][j];
          if (!(d > 0.0) || !isfinite(d)) bad = 1;
          const double piv = sqrt(d);
          a[j][j] = piv;
          rdiag[j] = 1.0 / piv;
        }
        asm volatile("bar.sync 1, 64;");
        if (r > j && r < n) {
          const double arj = a[r][j] * rdiag[j];
          a[r][j] = arj;
          const int cmax = min(c1, r + 1);
          for (int c = j + 1; c < cmax; ++c) a[r][c] -= arj * a[c][j];
        }
        asm volatile("bar.sync 1, 64;");
      }
    }
    __syncthreads();
    if (bad) break;
    // rank-(c1-c0) update of the trailing tile: a[r][c] -= sum_j a[r][j] a[c][j], c1 <= c <= r
    const int m = n - c1;
    for (int e = tid; e < m * NB; e += blockDim.x) {
      const int r = c1 + (e >> 6), c = e & (NB - 1);
      if (c >= c1 && c <= r) {
        double s0 = 0.0, s1 = 0.0;
        int j = c0;
        for (; j + 1 < c1; j += 2) {  // two independent chains
          s0 = fma(a[r][j], a[c][j], s0);
          s1 = fma(a[r][j + 1], a[c][j + 1], s1);
        }
        if (j < c1) s0 = fma(a[r][j], a[c][j], s0);
        a[r][c] -= s0 + s1;
      }
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) *status = 1;
    return;
  }
  // x = L^{-1} by a row sweep over 8-row blocks: the 64 column threads solve
  // the 8x8 diagonal block of their column (no barrier), then all threads
  // apply the rank-8 update to the rows below (one barrier per block).
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    x[r][c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += 8) {
    const int c1 = min(c0 + 8, n);
    if (tid < NB) {
      const int col = tid;
      for (int j = c0; j < c1; ++j) {
        const double xj = x[j][col] * rdiag[j];
        x[j][col] = xj;
        for (int i = j + 1; i < c1; ++i) x[i][col] -= a[i][j] * xj;
      }
    }
    __syncthreads();
    const int m = n - c1;
    for (int e = tid; e < m * NB; e += blockDim.x) {
      const int i = c1 + (e >> 6), col = e & (NB - 1);
      if (col <= i) {
        double s0 = 0.0, s1 = 0.0;
        int j = c0;
        for (; j + 1 < c1; j += 2) {
          s0 = fma(a[i][j], x[j][col], s0);
          s1 = fma(a[i][j + 1], x[j + 1][col], s1);
        }
        if (j < c1) s0 = fma(a[i][j], x[j][col], s0);
        x[i][col] -= s0 + s1;
      }
    }
    __syncthreads();
  }
  double* Li = Linv + (long)k * NB * NB;
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    Li[e] = (c <= r) ? x[r][c] : 0.0;
    if (r < n && c <= r) A[(long)(k0 + r) * dim + k0 + c] = a[r][c];
  }
}

// Register-panel variant of potrf_inv (256 threads).  The NB = 64 tile is
// factored in NB / PW = 8 panels of PW = 8 columns; warp 0 factors a panel
// with the panel rows in registers (lane l owns rows l and l + 32, 2 x PW
// doubles), pivots and column entries exchanged by shuffles, so a column
// step is a shuffle, an rsqrt and one FMA wave with no shared-memory round
// trip.  All eight warps then apply the rank-PW trailing update.  The
// inverse is blocked PW x PW: the NB / PW diagonal-block inverses in
// parallel (warp w < NB / PW inverts block w, lanes < PW own its columns),
// then the NB / PW - 1 block rows below with two barriers each.  Rows past
// the matrix end are identity, so every tile runs the same schedule.
constexpr int PW = 8;  // panel width

template <bool kRB>
__global__ void potrf_reg_kernel(double* __restrict__ A, int dim, int k_arg,
                                 const int32_t* __restrict__ klist, double* __restrict__ Linv,
                                 int32_t* __restrict__ status);

// PBA_POTRF_RB=0 selects the shared-memory trailing update (comparison).
bool potrf_rb() {
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("PBA_POTRF_RB");
    v = !(env && env[0] == '0');
  }
  return v == 1;
}

// kRB: the trailing update runs on register-held 4x4 blocks (thread t owns
// rows 4(t/16).., cols 4(t%16)..), reading only the 8 panel columns from
// shared memory; the owners of the next panel's columns publish them to
// shared memory before warp 0 factors it.
template <bool kRB>
__global__ void __launch_bounds__(256) potrf_reg_kernel(double* __restrict__ A, int dim,
                                                        int k_arg,
                                                        const int32_t* __restrict__ klist,
                                                        double* __restrict__ Linv,
                                                        int32_t* __restrict__ status) {
  extern __shared__ double psm[];
  double(*a)[LD] = reinterpret_cast<double(*)[LD]>(psm);
  double(*x)[LD] = reinterpret_cast<double(*)[LD]>(psm + NB * LD);
  double(*tt)[PW + 1] = reinterpret_cast<double(*)[PW + 1]>(psm + 2 * NB * LD);
  __shared__ double rdiag[NB];
  __shared__ int bad;
  if (*status) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = klist ? klist[blockIdx.x] : k_arg;  // dissection path: one tile per CTA
  const int k0 = k * NB;
  const int n = min(NB, dim - k0);
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    a[r][c] = (r < n && c <= r) ? A[(long)(k0 + r) * dim + k0 + c] : (r == c ? 1.0 : 0.0);
    x[r][c] = 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  const int rb = tid >> 4, cb = tid & 15;  // kRB: this thread's 4x4 block
  double blk[4][4];
  if (kRB) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) blk[i][j] = a[4 * rb + i][4 * cb + j];
  }
#pragma unroll 1
  for (int c0 = 0; c0 < NB; c0 += PW) {
    if (kRB && c0 > 0) {  // publish the panel's columns (updated in registers)
      if (4 * cb >= c0 && 4 * cb < c0 + PW && cb <= rb) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) a[4 * rb + i][4 * cb + j] = blk[i][j];
      }
      __syncthreads();
    }
    if (warp == 0) {
      const int hp = c0 >> 5;  // half (row block) the panel's diagonal rows live in
      double v0[PW], v1[PW];
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        v0[c] = a[lane][c0 + c];
        v1[c] = a[lane + 32][c0 + c];
      }
#pragma unroll
      for (int jj = 0; jj < PW; ++jj) {
        const int j = c0 + jj;
        const double dj = __shfl_sync(0xffffffffu, hp ? v1[jj] : v0[jj], j & 31);
        if (lane == 0 && (!(dj > 0.0) || !isfinite(dj))) bad = 1;
        const double inv = rsqrt(dj);
        const double piv = dj * inv;
        if (lane == 0) rdiag[j] = inv;
        if (lane > j) v0[jj] *= inv;
        else if (lane == j) v0[jj] = piv;
        if (lane + 32 > j) v1[jj] *= inv;
        else if (lane + 32 == j) v1[jj] = piv;
#pragma unroll
        for (int cc = jj + 1; cc < PW; ++cc) {
          const int c = c0 + cc;
          const double lcj = __shfl_sync(0xffffffffu, hp ? v1[jj] : v0[jj], c & 31);
          if (lane >= c) v0[cc] = fma(-v0[jj], lcj, v0[cc]);
          if (lane + 32 >= c) v1[cc] = fma(-v1[jj], lcj, v1[cc]);
        }
      }
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        a[lane][c0 + c] = v0[c];
        a[lane + 32][c0 + c] = v1[c];
      }
    }
    __syncthreads();
    if (bad) break;
    // rank-8 trailing update: a[r][c] -= sum_j a[r][j] a[c][j], c1 <= c <= r
    const int c1 = c0 + PW, m = NB - c1;
    if (kRB) {
      if (4 * cb >= c1 && cb <= rb) {
        double pr[4][PW], pc[4][PW];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int q = 0; q < PW; ++q) {
            pr[i][q] = a[4 * rb + i][c0 + q];
            pc[i][q] = a[4 * cb + i][c0 + q];
          }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int q = 0; q < PW; q += 2) {
              s0 = fma(pr[i][q], pc[j][q], s0);
              s1 = fma(pr[i][q + 1], pc[j][q + 1], s1);
            }
            blk[i][j] -= s0 + s1;
          }
      }
    } else {
      for (int e = tid; e < m * m; e += blockDim.x) {
        const int r = c1 + e / m, c = c1 + e % m;
        if (c <= r) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int j = 0; j < PW; j += 4) {
            s0 = fma(a[r][c0 + j], a[c][c0 + j], s0);
            s1 = fma(a[r][c0 + j + 1], a[c][c0 + j + 1], s1);
            s2 = fma(a[r][c0 + j + 2], a[c][c0 + j + 2], s2);
            s3 = fma(a[r][c0 + j + 3], a[c][c0 + j + 3], s3);
          }
          a[r][c] -= (s0 + s1) + (s2 + s3);
        }
      }
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) *status = 1;
    return;
  }
  // inverse, diagonal blocks: warp b < NB / PW inverts L_bb, lane c < PW owns column c
  if (warp < NB / PW && lane < PW) {
    const int o = warp * PW, c = lane;
    for (int i = 0; i < PW; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int j = c; j < i; ++j) s = fma(-a[o + i][o + j], x[o + j][o + c], s);
      x[o + i][o + c] = (i >= c) ? s * rdiag[o + i] : 0.0;
    }
  }
  __syncthreads();
  // block rows i = 1 .. NB/PW - 1: T_ij = sum_{k=j}^{i-1} L_ik X_kj, then X_ij = -X_ii T_ij
  for (int bi = 1; bi < NB / PW; ++bi) {
    const int oi = bi * PW;
    for (int e = tid; e < bi * PW * PW; e += blockDim.x) {
      const int bj = e / (PW * PW), r = (e / PW) % PW, c = e % PW;
      const int oj = bj * PW;
      double s0 = 0.0, s1 = 0.0;
      for (int q = oj; q < oi; q += 2) {
        s0 = fma(a[oi + r][q], x[q][oj + c], s0);
        s1 = fma(a[oi + r][q + 1], x[q + 1][oj + c], s1);
      }
      tt[bj * PW + r][c] = s0 + s1;
    }
    __syncthreads();
    for (int e = tid; e < bi * PW * PW; e += blockDim.x) {
      const int bj = e / (PW * PW), r = (e / PW) % PW, c = e % PW;
      double s = 0.0;
      for (int q = 0; q <= r; ++q) s = fma(x[oi + r][oi + q], tt[bj * PW + q][c], s);
      x[oi + r][bj * PW + c] = -s;
    }
    __syncthreads();
  }
  double* Li = Linv + (long)k * NB * NB;
  for (int e = tid; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    Li[e] = (c <= r) ? x[r][c] : 0.0;
    if (r < n && c <= r) A[(long)(k0 + r) * dim + k0 + c] = a[r][c];
  }
}

// out(64x64) = P(64x64) * Q(64x64)^T with P, Q in shared memory (LD stride);
// each of 256 threads owns a 4x4 block of outputs.
__device__ __forceinline__ void tile_abt(const double* P, const double* Q, double acc[4][4]) {
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
  for (int kk = 0; kk < NB; ++kk) {
    double xv[4], yv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      xv[a] = P[(tr + 16 * a) * LD + kk];
      yv[a] = Q[(tc + 16 * a) * LD + kk];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c] = fma(xv[a], yv[c], acc[a][c]);
  }
}

// L_ik = A_ik L_kk^{-T} for the non-zero tiles below diagonal tile k.
__global__ void __launch_bounds__(256) panel_kernel(double* __restrict__ A, int dim, int k, int T,
                                                    const int32_t* __restrict__ nz,
                                                    const double* __restrict__ Linv,
                                                    const int32_t* __restrict__ status) {
  if (*status) return;
  const int bi = k + 1 + blockIdx.x;
  if (bi >= T || !nz[bi * T + k]) return;
  extern __shared__ double smem[];
  double* P = smem;
  double* Q = smem + NB * LD;
  const int k0 = k * NB, r0 = bi * NB;
  const int nk = min(NB, dim - k0), nr = min(NB, dim - r0);
  const double* Li = Linv + (long)k * NB * NB;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    P[r * LD + c] = (r < nr && c < nk) ? A[(long)(r0 + r) * dim + k0 + c] : 0.0;
    Q[r * LD + c] = Li[e];
  }
  __syncthreads();
  double acc[4][4];
  tile_abt(P, Q, acc);
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int r = tr + 16 * a, col = tc + 16 * c;
      if (r < nr && col < nk) A[(long)(r0 + r) * dim + k0 + col] = acc[a][c];
    }
}

// Trailing update C(bi,bj) -= L(bi,k) L(bj,k)^T for bi >= bj > k, skipping
// tiles whose panel factors are zero; marks fill-in.
__global__ void __launch_bounds__(256) syrk_kernel(double* __restrict__ A, int dim, int k, int T,
                                                   int32_t* __restrict__ nz,
                                                   const int32_t* __restrict__ status) {
  if (*status) return;
  const int m = T - k - 1;
  const int t = blockIdx.x;
  int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
  while (bi * (bi + 1) / 2 > t) --bi;
  const int bj = t - bi * (bi + 1) / 2;
  if (bi >= m) return;
  const int ti = k + 1 + bi, tj = k + 1 + bj;
  if (!nz[ti * T + k] || !nz[tj * T + k]) return;
  extern __shared__ double smem[];
  double* Pi = smem;
  double* Pj = smem + NB * LD;
  const int k0 = k * NB, ri = ti * NB, rj = tj * NB;
  const int nk = min(NB, dim - k0);
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    Pi[r * LD + c] = (ri + r < dim && c < nk) ? A[(long)(ri + r) * dim + k0 + c] : 0.0;
    Pj[r * LD + c] = (rj + r < dim && c < nk) ? A[(long)(rj + r) * dim + k0 + c] : 0.0;
  }
  __syncthreads();
  double acc[4][4];
  tile_abt(Pi, Pj, acc);
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int r = ri + tr + 16 * a, col = rj + tc + 16 * c;
      if (r < dim && col < dim && col <= r) A[(long)r * dim + col] -= acc[a][c];
    }
  if (threadIdx.x == 0) nz[ti * T + tj] = 1;
}

// Forward (L y = -b) and backward (L^T x = y) substitution in one CTA of 1024
// threads with the tile inverses: per tile row a gather over the non-zero
// tiles (16 threads per row, shuffle-reduced), then a 64x64 mat-vec.
// ---- nested-dissection path (long chain-like pose graphs) ---------------
// Tiles are reordered so that P independent chain segments come first and
// the (band-wide) separators between them last; the segments' steps run as
// batched launches (one CTA per segment), then the separators' small Schur
// complement is factored as usual.  See pba_solve_dense.

// Ap (D x D, lower) = P (H + lam diag H) P^T on the structural tiles listed in
// tiles (pairs of new tile indices, row >= col); padding rows are identity.
__global__ void damp_copy_perm_kernel(HSource H, int dim, double lam_arg,
                                      const double* __restrict__ lam_dev, int D,
                                      const int32_t* __restrict__ tiles,
                                      const int32_t* __restrict__ new_to_old,
                                      double* __restrict__ Ap) {
  const double lam = lam_dev ? *lam_dev : lam_arg;
  const int ti = tiles[2 * blockIdx.x], tj = tiles[2 * blockIdx.x + 1];
  const int oi = new_to_old[ti], oj = new_to_old[tj];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    const int gr = oi * NB + r, gc = oj * NB + c;  // original scalar indices
    double v;
    if (gr >= dim || gc >= dim) {
      v = (ti == tj && r == c) ? 1.0 : 0.0;
    } else {
      const int hi = max(gr, gc), lo = min(gr, gc);
      const double h = H.at(hi, lo);
      v = (gr == gc) ? h + lam * h : h;
    }
    Ap[(long)(ti * NB + r) * D + tj * NB + c] = v;
  }
}

__global__ void permute_vec_kernel(const double* __restrict__ src, int dim, int T,
                                   const int32_t* __restrict__ new_to_old,
                                   double* __restrict__ dst, int to_new) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T * NB) return;
  const int g = new_to_old[i / NB] * NB + i % NB;  // original index of new index i
  if (to_new) {
    dst[i] = g < dim ? src[g] : 0.0;
  } else if (g < dim) {
    dst[g] = src[i];
  }
}

// L_ik = A_ik L_kk^{-T} for listed (k, i) pairs
__global__ void __launch_bounds__(256) panel_list_kernel(double* __restrict__ A, int D,
                                                         const int32_t* __restrict__ pairs,
                                                         const double* __restrict__ Linv,
                                                         const int32_t* __restrict__ status) {
  if (*status) return;
  const int k = pairs[2 * blockIdx.x], bi = pairs[2 * blockIdx.x + 1];
  extern __shared__ double smem[];
  double* P = smem;
  double* Q = smem + NB * LD;
  const int k0 = k * NB, r0 = bi * NB;
  const double* Li = Linv + (long)k * NB * NB;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    P[r * LD + c] = A[(long)(r0 + r) * D + k0 + c];
    Q[r * LD + c] = Li[e];
  }
  __syncthreads();
  double acc[4][4];
  tile_abt(P, Q, acc);
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) A[(long)(r0 + tr + 16 * a) * D + k0 + tc + 16 * c] = acc[a][c];
}

// A_ij -= L_ik L_jk^T for listed (k, i, j) triples, i >= j
__global__ void __launch_bounds__(256) syrk_list_kernel(double* __restrict__ A, int D,
                                                        const int32_t* __restrict__ triples,
                                                        const int32_t* __restrict__ status) {
  if (*status) return;
  const int k = triples[3 * blockIdx.x], ti = triples[3 * blockIdx.x + 1],
            tj = triples[3 * blockIdx.x + 2];
  extern __shared__ double smem[];
  double* Pi = smem;
  double* Pj = smem + NB * LD;
  const int k0 = k * NB, ri = ti * NB, rj = tj * NB;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e / NB, c = e % NB;
    Pi[r * LD + c] = A[(long)(ri + r) * D + k0 + c];
    Pj[r * LD + c] = A[(long)(rj + r) * D + k0 + c];
  }
  __syncthreads();
  double acc[4][4];
  tile_abt(Pi, Pj, acc);
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int r = ri + tr + 16 * a, col = rj + tc + 16 * c;
      if (col <= r) A[(long)r * D + col] -= acc[a][c];
    }
}

// One forward step of L y = -b on tile row k: y_k = Linv_kk (-b_k - sum_{j<k} L_kj y_j)
__device__ __forceinline__ void fwd_step(const double* __restrict__ A, int dim, int T, int k,
                                         const int32_t* __restrict__ env,
                                         const int32_t* __restrict__ nz,
                                         const double* __restrict__ Linv,
                                         const double* __restrict__ b, double* __restrict__ y,
                                         double* r) {
  const int tid = threadIdx.x;
  const int row = tid >> 4, sub = tid & 15;  // 64 rows x 16 lanes
  const int k0 = k * NB, nk = min(NB, dim - k0);
  double s = 0.0;
  if (row < nk) {
    for (int j = env[k]; j < k; ++j) {
      if (!nz[k * T + j]) continue;
      const double* Lr = A + (long)(k0 + row) * dim + j * NB;
      const double* yj = y + j * NB;
      for (int c = sub; c < NB; c += 16) s += Lr[c] * yj[c];
    }
  }
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (sub == 0) r[row] = (row < nk) ? -b[k0 + row] - s : 0.0;
  __syncthreads();
  const double* Li = Linv + (long)k * NB * NB;
  double t = 0.0;
  for (int c = sub; c <= row; c += 16) t += Li[row * NB + c] * r[c];
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  if (sub == 0 && row < nk) y[k0 + row] = t;
  __syncthreads();
}

// One backward step of L^T x = y on tile row k: x_k = Linv_kk^T (y_k - sum_{i>k} L_ik^T x_i)
__device__ __forceinline__ void bwd_step(const double* __restrict__ A, int dim, int T, int k,
                                         const int32_t* __restrict__ last,
                                         const int32_t* __restrict__ nz,
                                         const double* __restrict__ Linv,
                                         const double* __restrict__ y, double* __restrict__ x,
                                         double* r) {
  const int tid = threadIdx.x;
  const int row = tid >> 4, sub = tid & 15;
  const int k0 = k * NB, nk = min(NB, dim - k0);
  double s = 0.0;
  if (row < nk) {
    for (int i = k + 1; i <= last[k]; ++i) {
      if (!nz[i * T + k]) continue;
      const int i0 = i * NB, ni = min(NB, dim - i0);
      for (int rr = sub; rr < ni; rr += 16) s += A[(long)(i0 + rr) * dim + k0 + row] * x[i0 + rr];
    }
  }
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (sub == 0) r[row] = (row < nk) ? y[k0 + row] - s : 0.0;
  __syncthreads();
  const double* Li = Linv + (long)k * NB * NB;
  double t = 0.0;
  for (int c = row + sub; c < NB; c += 16) t += Li[c * NB + row] * r[c];
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  if (sub == 0 && row < nk) x[k0 + row] = t;
  __syncthreads();
}

__global__ void __launch_bounds__(1024) trisolve_kernel(const double* __restrict__ A, int dim, int T,
                                                         const int32_t* __restrict__ env,
                                                         const int32_t* __restrict__ last,
                                                         const int32_t* __restrict__ nz,
                                                         const double* __restrict__ Linv,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ y,
                                                         double* __restrict__ x,
                                                         const int32_t* __restrict__ status) {
  if (*status) return;
  __shared__ double r[NB];
  for (int k = 0; k < T; ++k) fwd_step(A, dim, T, k, env, nz, Linv, b, y, r);
  for (int k = T - 1; k >= 0; --k) bwd_step(A, dim, T, k, last, nz, Linv, y, x, r);
}

// Substitution over independent tile ranges (dissection path): CTA c walks
// tiles [ranges[2c], ranges[2c+1]) forwards (forward != 0) or backwards.
__global__ void __launch_bounds__(1024) trisolve_range_kernel(
    const double* __restrict__ A, int dim, int T, const int32_t* __restrict__ env,
    const int32_t* __restrict__ last, const int32_t* __restrict__ nz,
    const double* __restrict__ Linv, const double* __restrict__ b, double* __restrict__ y,
    double* __restrict__ x, const int32_t* __restrict__ ranges, int forward,
    const int32_t* __restrict__ status) {
  if (*status) return;
  __shared__ double r[NB];
  const int lo = ranges[2 * blockIdx.x], hi = ranges[2 * blockIdx.x + 1];
  if (forward) {
    for (int k = lo; k < hi; ++k) fwd_step(A, dim, T, k, env, nz, Linv, b, y, r);
  } else {
    for (int k = hi - 1; k >= lo; --k) bwd_step(A, dim, T, k, last, nz, Linv, y, x, r);
  }
}

}  // namespace
}  // namespace pba

using namespace pba;

// Nested dissection of a chain-like (narrow tile band) system.  Returns
// PBA_OK when solved, 1 when the structure does not qualify (caller falls
// back to the sequential tiled factorisation), or an error code.
//
// The original tile order is cut into P segments separated by w-tile
// separators (w = tile half-bandwidth), so no segment couples to another.
// New order: all segments, then all separators.  The right-looking tiled
// Cholesky of P A P^T then has independent segment steps: step s of every
// segment of one parity runs in one batched launch (segments of equal
// parity share no separator, so their trailing updates touch disjoint
// tiles), after which the separators' Schur complement is factored tile by
// tile.  Sequential steps: 2 * max segment length + (P - 1) * w instead of T.
// Each tile update is the same arithmetic as the sequential path, in the
// order of the new elimination sequence.
// Dynamic shared-memory limits of the tile kernels, set once per device (so
// a captured solve issues no attribute calls).
int set_solver_smem_attributes() {
  static bool done[64] = {false};
  int dev = 0;
  PBA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && done[dev]) return PBA_OK;
  const int tile_smem = 2 * NB * LD * sizeof(double);
  const int reg_smem = tile_smem + (NB / PW - 1) * PW * (PW + 1) * (int)sizeof(double);
  PBA_CUDA_TRY(cudaFuncSetAttribute(syrk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    tile_smem));
  PBA_CUDA_TRY(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    tile_smem));
  PBA_CUDA_TRY(cudaFuncSetAttribute(potrf_inv_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
  PBA_CUDA_TRY(cudaFuncSetAttribute(potrf_reg_kernel<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, reg_smem));
  PBA_CUDA_TRY(cudaFuncSetAttribute(potrf_reg_kernel<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, reg_smem));
  PBA_CUDA_TRY(cudaFuncSetAttribute(panel_list_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
  PBA_CUDA_TRY(cudaFuncSetAttribute(syrk_list_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem));
  if (dev >= 0 && dev < 64) done[dev] = true;
  return PBA_OK;
}

int solve_dissected(HSource H, const double* b, int dim, double lam, const double* lam_dev,
                    bool reuse, const std::vector<int32_t>& env, const std::vector<int32_t>& last,
                    const SolveWork& w, double* delta, int32_t* status, cudaStream_t st) {
  const int T = (int)env.size(), D = T * NB;
  int band = 0;
  for (int k = 0; k < T; ++k) band = max(band, last[k] - k);
  if (band < 1 || band > kMaxBand) return 1;
  const int P = min(8, T / (4 * band));
  if (P < 2) return 1;
  // segments and separators in the original tile order
  const int seg_total = T - (P - 1) * band;
  std::vector<int> seg_start(P), seg_len(P);
  for (int g = 0, pos = 0; g < P; ++g) {
    seg_len[g] = seg_total / P + (g < seg_total % P ? 1 : 0);
    seg_start[g] = pos;
    pos += seg_len[g] + (g < P - 1 ? band : 0);
  }
  std::vector<int32_t> n2o, o2n(T);
  std::vector<int> new_seg(P);
  for (int g = 0; g < P; ++g) {
    new_seg[g] = (int)n2o.size();
    for (int t = 0; t < seg_len[g]; ++t) n2o.push_back(seg_start[g] + t);
  }
  const int sep_base = (int)n2o.size();
  for (int g = 0; g + 1 < P; ++g)
    for (int t = 0; t < band; ++t) n2o.push_back(seg_start[g] + seg_len[g] + t);
  if ((int)n2o.size() != T) return 1;
  for (int i = 0; i < T; ++i) o2n[n2o[i]] = i;
  // symbolic structure of the permuted matrix (lower tiles) and its fill
  std::vector<char> S((size_t)T * T, 0);
  for (int oi = 0; oi < T; ++oi)
    for (int oj = env[oi]; oj <= oi; ++oj) {
      const int a = o2n[oi], c = o2n[oj];
      S[(size_t)max(a, c) * T + min(a, c)] = 1;
    }
  std::vector<std::vector<int>> rows(T);
  for (int k = 0; k < T; ++k) {
    for (int i = k + 1; i < T; ++i)
      if (S[(size_t)i * T + k]) rows[k].push_back(i);
    if ((int)rows[k].size() > 2 * kMaxBand) return 1;
    for (int x : rows[k])
      for (int y : rows[k])
        if (y <= x) S[(size_t)x * T + y] = 1;
  }
  // staging: [n2o | tiles | klist | pairs | triples]
  std::vector<int32_t> tiles, klist, pairs, triples;
  for (int i = 0; i < T; ++i)
    for (int j = 0; j <= i; ++j)
      if (S[(size_t)i * T + j] || i == j) tiles.push_back(i), tiles.push_back(j);
  struct Launch { int k0, nk, p0, np, t0, nt; };
  std::vector<Launch> launches;
  auto add_batch = [&](const std::vector<int>& ks) {
    Launch L{(int)klist.size(), (int)ks.size(), (int)pairs.size() / 2, 0, (int)triples.size() / 3, 0};
    for (int k : ks) {
      klist.push_back(k);
      for (int i : rows[k]) pairs.push_back(k), pairs.push_back(i);
      for (size_t a = 0; a < rows[k].size(); ++a)
        for (size_t c = 0; c <= a; ++c)
          triples.push_back(k), triples.push_back(rows[k][a]), triples.push_back(rows[k][c]);
    }
    L.np = (int)pairs.size() / 2 - L.p0;
    L.nt = (int)triples.size() / 3 - L.t0;
    launches.push_back(L);
  };
  int lmax = 0;
  for (int g = 0; g < P; ++g) lmax = max(lmax, seg_len[g]);
  for (int st_ = 0; st_ < lmax; ++st_)
    for (int parity = 0; parity < 2; ++parity) {
      std::vector<int> ks;
      for (int g = parity; g < P; g += 2)
        if (st_ < seg_len[g]) ks.push_back(new_seg[g] + st_);
      if (!ks.empty()) add_batch(ks);
    }
  for (int k = sep_base; k < T; ++k) add_batch(std::vector<int>{k});
  static thread_local std::vector<int32_t> staging;
  staging.clear();
  staging.insert(staging.end(), n2o.begin(), n2o.end());
  const size_t off_tiles = staging.size();
  staging.insert(staging.end(), tiles.begin(), tiles.end());
  const size_t off_k = staging.size();
  staging.insert(staging.end(), klist.begin(), klist.end());
  const size_t off_p = staging.size();
  staging.insert(staging.end(), pairs.begin(), pairs.end());
  const size_t off_t = staging.size();
  staging.insert(staging.end(), triples.begin(), triples.end());
  const size_t off_ranges = staging.size();  // P segment ranges, then the separator range
  for (int g = 0; g < P; ++g) staging.push_back(new_seg[g]), staging.push_back(new_seg[g] + seg_len[g]);
  staging.push_back(sep_base), staging.push_back(T);
  if (staging.size() > list_ints(T)) return 1;
  const size_t off_nz = staging.size();
  // tile flags (with fill) and envelope of the permuted matrix for trisolve
  std::vector<int32_t> envp(T), lastp(T);
  for (int i = 0; i < T; ++i) {
    int e = i;
    for (int j = 0; j <= i; ++j)
      if (S[(size_t)i * T + j]) { e = j; break; }
    envp[i] = e;
  }
  for (int k = 0; k < T; ++k) {
    int l = k;
    for (int i = k + 1; i < T; ++i)
      if (S[(size_t)i * T + k]) l = i;
    lastp[k] = l;
  }
  for (size_t e = 0; e < (size_t)T * T; ++e) staging.push_back(S[e] ? 1 : 0);
  for (int i = 0; i < T; ++i) staging[off_nz + (size_t)i * T + i] = 1;
  staging.insert(staging.end(), envp.begin(), envp.end());
  staging.insert(staging.end(), lastp.begin(), lastp.end());
  int32_t* d_lists = w.lists;
  int32_t* d_env = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(w.nz) +
                                              align_up((size_t)T * T * sizeof(int32_t), 256));
  if (!reuse) {  // the tables depend only on (dim, tile_env): a reused plan is already there
    PBA_CUDA_TRY(cudaMemcpyAsync(d_lists, staging.data(), off_nz * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, st));
    PBA_CUDA_TRY(cudaMemcpyAsync(w.nz, staging.data() + off_nz, (size_t)T * T * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, st));
    PBA_CUDA_TRY(cudaMemcpyAsync(d_env, staging.data() + off_nz + (size_t)T * T,
                                 2 * T * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  }
  const int32_t* d_n2o = d_lists;
  damp_copy_perm_kernel<<<(unsigned)(tiles.size() / 2), 256, 0, st>>>(H, dim, lam, lam_dev, D,
                                                                    d_lists + off_tiles, d_n2o,
                                                                    w.A);
  PBA_LAUNCH_CHECK();
  permute_vec_kernel<<<(D + 255) / 256, 256, 0, st>>>(b, dim, T, d_n2o, w.bp, 1);
  PBA_LAUNCH_CHECK();
  const int tile_smem = 2 * NB * LD * sizeof(double);
  const int reg_smem = tile_smem + (NB / PW - 1) * PW * (PW + 1) * (int)sizeof(double);
  if (int rc = set_solver_smem_attributes()) return rc;
  for (const Launch& L : launches) {
    if (potrf_rb())
      potrf_reg_kernel<true><<<L.nk, 256, reg_smem, st>>>(w.A, D, 0, d_lists + off_k + L.k0,
                                                          w.Linv, status);
    else
      potrf_reg_kernel<false><<<L.nk, 256, reg_smem, st>>>(w.A, D, 0, d_lists + off_k + L.k0,
                                                           w.Linv, status);
    PBA_LAUNCH_CHECK();
    if (L.np) {
      panel_list_kernel<<<L.np, 256, tile_smem, st>>>(w.A, D, d_lists + off_p + 2 * L.p0,
                                                      w.Linv, status);
      PBA_LAUNCH_CHECK();
    }
    if (L.nt) {
      syrk_list_kernel<<<L.nt, 256, tile_smem, st>>>(w.A, D, d_lists + off_t + 3 * L.t0, status);
      PBA_LAUNCH_CHECK();
    }
  }
  // substitutions: segments in parallel, separators after (forward) / before
  // (backward) them
  const int32_t* d_ranges = d_lists + off_ranges;
  trisolve_range_kernel<<<P, 1024, 0, st>>>(w.A, D, T, d_env, d_env + T, w.nz, w.Linv, w.bp, w.y,
                                            w.xp, d_ranges, 1, status);
  PBA_LAUNCH_CHECK();
  trisolve_range_kernel<<<1, 1024, 0, st>>>(w.A, D, T, d_env, d_env + T, w.nz, w.Linv, w.bp, w.y,
                                            w.xp, d_ranges + 2 * P, 1, status);
  PBA_LAUNCH_CHECK();
  trisolve_range_kernel<<<1, 1024, 0, st>>>(w.A, D, T, d_env, d_env + T, w.nz, w.Linv, w.bp, w.y,
                                            w.xp, d_ranges + 2 * P, 0, status);
  PBA_LAUNCH_CHECK();
  trisolve_range_kernel<<<P, 1024, 0, st>>>(w.A, D, T, d_env, d_env + T, w.nz, w.Linv, w.bp, w.y,
                                            w.xp, d_ranges, 0, status);
  PBA_LAUNCH_CHECK();
  permute_vec_kernel<<<(D + 255) / 256, 256, 0, st>>>(w.xp, dim, T, d_n2o, delta, 0);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

extern "C" size_t pba_solve_work_bytes(int32_t dim) {
  if (dim <= 0) return 0;
  const size_t T = (dim + NB - 1) / NB, D = T * NB;
  return align_up(D * D * sizeof(double), 256) + align_up(T * NB * NB * sizeof(double), 256) +
         3 * align_up(D * sizeof(double), 256) + align_up(list_ints(T) * sizeof(int32_t), 256) +
         align_up(T * T * sizeof(int32_t), 256) + align_up(2 * T * sizeof(int32_t), 256);
}

namespace pba {
namespace {
// dim <= 64 (one tile, e.g. c1's 54): damping, factorisation and both
// substitutions in one CTA — the tiled path's four launches (damp, tile
// flags, diagonal-tile potrf with its inverse, substitution) cost ~48 us
// there, mostly launch and barrier latency of kernels sized for big tiles.
// LDL^T by right-looking elimination on the unscaled columns
// (A_ij -= A_ik A_jk / A_kk for k < j <= i) of the matrix bordered by the
// row -b^T, so the elimination also yields the forward substitution (row
// dim ends as L~^{-1} (-b), L~ the unit lower factor).  Eight threads share
// each row (every eighth column of it), so a step updates only the live
// trailing entries (n^3/6 in all) with one barrier (a column-per-thread split
// reads along diagonals: 4-way bank conflicts, 1.4x slower).  Warp 0 then
// solves L~^T x = D^{-1} y with two rows per lane.
constexpr int kSmallQ = 8;  // threads per row
constexpr int kSmallThreads = ((NB + 1) * kSmallQ + 31) / 32 * 32;  // rows 0..64, 544
__global__ void __launch_bounds__(kSmallThreads)
    small_solve_kernel(HSource H, const double* __restrict__ b, int dim, double lam_arg,
                       const double* __restrict__ lam_dev, double* __restrict__ delta,
                       int32_t* __restrict__ status) {
  // unscaled columns; row dim = L~^{-1} (-b).  Row stride 68 doubles: the
  // four rows of a warp's row writes fall on distinct bank halves.
  constexpr int kLd = 68;
  __shared__ double L[NB + 1][kLd];
  __shared__ int rp[NB / 6 + 2];
  const int tid = threadIdx.x;
  const double lam = lam_dev ? *lam_dev : lam_arg;
  // Stage H's lower triangle and the border row in L.  Every global load of
  // a thread is issued before its first shared store (the compiler cannot
  // prove a generic load does not alias the shared tile, so an interleaved
  // loop would wait out one global round trip per entry).
  for (int e = tid; e < (dim + 1) * kLd; e += kSmallThreads) (&L[0][0])[e] = 0.0;
  if (H.row_ptr)
    for (int t = tid; t <= dim / 6; t += kSmallThreads) rp[t] = H.row_ptr[t];
  __syncthreads();
  {
    constexpr int kMaxPer = (NB * NB + kSmallThreads - 1) / kSmallThreads;  // 16
    double v[kMaxPer];
    int at[kMaxPer];  // i * kLd + j, or -1
    const int n = H.row_ptr ? 36 * rp[dim / 6] : dim * dim;
#pragma unroll
    for (int r = 0; r < kMaxPer; ++r) {
      const int e = tid + r * kSmallThreads;
      at[r] = -1;
      v[r] = 0.0;
      if (e < n) {
        int i, jj;
        if (H.row_ptr) {
          const int blk = e / 36, rc = e - 36 * blk;
          int br = 0;
          while (rp[br + 1] <= blk) ++br;
          i = 6 * br + rc / 6;
          jj = 6 * H.cols[blk] + rc % 6;
        } else {
          i = e / dim;
          jj = e - i * dim;
        }
        if (jj <= i) {
          at[r] = i * kLd + jj;
          v[r] = H.H[e];
        }
      }
    }
    const double bj = tid < dim ? -b[tid] : 0.0;
#pragma unroll
    for (int r = 0; r < kMaxPer; ++r)
      if (at[r] >= 0) (&L[0][0])[at[r]] = v[r];
    if (tid < dim) L[dim][tid] = bj;
  }
  __syncthreads();
  if (tid < dim) L[tid][tid] = L[tid][tid] + lam * L[tid][tid];  // h + lam * np.diag(np.diag(h))
  __syncthreads();
  // thread (i, q) updates row i's entries j = k+1+q, k+1+q+8, ... <= min(i, dim-1)
  const int i = tid / kSmallQ, q = tid - i * kSmallQ;
  bool bad = false;
  for (int k = 0; k < dim; ++k) {
    const double d = L[k][k];  // final since step k - 1 (the same value in every thread)
    if (!(d > 0.0)) {
      bad = true;
      break;
    }
    if (i > k && i <= dim) {
      const double f = L[i][k] * __drcp_rn(d);
      const int jmax = min(i, dim - 1);
      // all loads first (column k is read-only in this step), then the updates
      double lk[NB / kSmallQ], li[NB / kSmallQ];
#pragma unroll
      for (int r = 0; r < NB / kSmallQ; ++r) {
        const int jj = k + 1 + q + kSmallQ * r;
        lk[r] = jj <= jmax ? L[jj][k] : 0.0;
        li[r] = jj <= jmax ? L[i][jj] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < NB / kSmallQ; ++r) {
        const int jj = k + 1 + q + kSmallQ * r;
        if (jj <= jmax) L[i][jj] = fma(-lk[r], f, li[r]);
      }
    }
    __syncthreads();
  }
  if (bad) {  // the reference's LinAlgError
    if (tid == 0) *status = 1;
    return;
  }
  if (tid >= 32) return;
  // L~^T x = z, z_j = y_j / d_j, L~_ij = L_ij / d_j: column sweep from the last row
  const int r0 = tid, r1 = tid + 32;
  const double id0 = r0 < dim ? __drcp_rn(L[r0][r0]) : 0.0;
  const double id1 = r1 < dim ? __drcp_rn(L[r1][r1]) : 0.0;
  double z0 = r0 < dim ? L[dim][r0] * id0 : 0.0, z1 = r1 < dim ? L[dim][r1] * id1 : 0.0;
  for (int k = dim - 1; k > 0; --k) {
    const double xk = __shfl_sync(0xffffffffu, k < 32 ? z0 : z1, k & 31);
    if (r0 < k) z0 = fma(-L[k][r0] * id0, xk, z0);
    if (r1 < k) z1 = fma(-L[k][r1] * id1, xk, z1);
  }
  if (r0 < dim) delta[r0] = z0;
  if (r1 < dim) delta[r1] = z1;
  if (tid == 0) *status = 0;
}

}  // namespace
}  // namespace pba

namespace {
int solve_dense_impl(HSource H, const double* b, int32_t dim, double lam, const double* lam_dev,
                     const int32_t* tile_env, void* work, int32_t flags, double* delta,
                     int32_t* status, void* stream) {
  const bool reuse = (flags & PBA_SOLVE_REUSE_PLAN) != 0;
  PBA_ARG_CHECK(dim > 0, "dim must be positive");
  PBA_ARG_CHECK(H.H && b && work && delta && status, "NULL buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SolveWork w = carve(work, dim);
  const int T = (dim + NB - 1) / NB;
  // envelope: env[i] = first tile column that can be non-zero in tile row i
  // (fill-in never leaves it); last[k] = last tile row whose envelope reaches k
  std::vector<int32_t> env(T), last(T);
  for (int i = 0; i < T; ++i) {
    int e = tile_env ? tile_env[i] : 0;
    PBA_ARG_CHECK(e >= 0 && e <= i, "tile_env[i] must lie in [0, i]");
    env[i] = e;
  }
  for (int k = 0; k < T; ++k) {
    int l = k;
    for (int i = k + 1; i < T; ++i)
      if (env[i] <= k) l = i;
    last[k] = l;
  }
  static int potrf_variant = -1;
  if (potrf_variant < 0) {
    const char* env = getenv("PBA_POTRF_VARIANT");
    potrf_variant = env ? atoi(env) : 1;
  }
  static int dissect = -1;
  if (dissect < 0) {
    const char* env = getenv("PBA_SOLVE_DISSECT");
    dissect = !(env && env[0] == '0');
  }
  if (T == 1 && potrf_variant == 1) {
    small_solve_kernel<<<1, kSmallThreads, 0, st>>>(H, b, dim, lam, lam_dev, delta, status);
    PBA_LAUNCH_CHECK();
    return PBA_OK;
  }
  if (dissect && potrf_variant == 1) {
    PBA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
    const int rc = solve_dissected(H, b, dim, lam, lam_dev, reuse, env, last, w, delta, status, st);
    if (rc != 1) return rc;  // 1: structure not suited, the sequential path follows
  }
  int32_t* d_env = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(w.nz) +
                                              align_up((size_t)T * T * sizeof(int32_t), 256));
  int32_t* d_last = d_env + T;
  // the tables are tiny; copy them with the stream so the call stays asynchronous
  static thread_local std::vector<int32_t> staging;
  if (!reuse) {
    staging.assign(env.begin(), env.end());
    staging.insert(staging.end(), last.begin(), last.end());
    PBA_CUDA_TRY(cudaMemcpyAsync(d_env, staging.data(), 2 * T * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, st));
  }
  PBA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  const long n2 = (long)dim * dim;
  damp_copy_kernel<<<(unsigned)((n2 + 255) / 256), 256, 0, st>>>(H, dim, lam, lam_dev, d_env,
                                                                   w.A);
  PBA_LAUNCH_CHECK();
  tile_flags_kernel<<<dim3(T, T), 256, 0, st>>>(w.A, dim, T, d_env, w.nz);
  PBA_LAUNCH_CHECK();
  const int tile_smem = 2 * NB * LD * sizeof(double);
  const int reg_smem = tile_smem + (NB / PW - 1) * PW * (PW + 1) * (int)sizeof(double);
  if (int rc = set_solver_smem_attributes()) return rc;
  for (int k = 0; k < T; ++k) {
    if (potrf_variant == 1 && potrf_rb())
      potrf_reg_kernel<true><<<1, 256, reg_smem, st>>>(w.A, dim, k, nullptr, w.Linv, status);
    else if (potrf_variant == 1)
      potrf_reg_kernel<false><<<1, 256, reg_smem, st>>>(w.A, dim, k, nullptr, w.Linv, status);
    else
      potrf_inv_kernel<<<1, 1024, tile_smem, st>>>(w.A, dim, k, w.Linv, status);
    PBA_LAUNCH_CHECK();
    const int m = last[k] - k;  // tile rows below k inside the envelope
    if (m > 0) {
      panel_kernel<<<m, 256, tile_smem, st>>>(w.A, dim, k, T, w.nz, w.Linv, status);
      PBA_LAUNCH_CHECK();
      syrk_kernel<<<m * (m + 1) / 2, 256, tile_smem, st>>>(w.A, dim, k, T, w.nz, status);
      PBA_LAUNCH_CHECK();
    }
  }
  trisolve_kernel<<<1, 1024, 0, st>>>(w.A, dim, T, d_env, d_last, w.nz, w.Linv, b, w.y, delta,
                                      status);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

}  // namespace

extern "C" int pba_solve_dense_ex(const double* H, const double* b, int32_t dim, double lam,
                                  const double* lam_dev, const int32_t* tile_env, void* work,
                                  int32_t flags, double* delta, int32_t* status, void* stream) {
  return solve_dense_impl(HSource{H, nullptr, nullptr, dim}, b, dim, lam, lam_dev, tile_env,
                          work, flags, delta, status, stream);
}

extern "C" int pba_solve_dense_bsr(const double* Hb, const int32_t* row_ptr, const int32_t* cols,
                                   const double* b, int32_t dim, double lam,
                                   const double* lam_dev, const int32_t* tile_env, void* work,
                                   int32_t flags, double* delta, int32_t* status, void* stream) {
  PBA_ARG_CHECK(row_ptr && cols && dim % 6 == 0, "block-sparse H needs its CSR and dim = 6 n");
  return solve_dense_impl(HSource{Hb, row_ptr, cols, dim}, b, dim, lam, lam_dev, tile_env, work,
                          flags, delta, status, stream);
}

extern "C" int pba_solve_dense(const double* H, const double* b, int32_t dim, double lam,
                               const int32_t* tile_env, void* work, double* delta,
                               int32_t* status, void* stream) {
  return pba_solve_dense_ex(H, b, dim, lam, nullptr, tile_env, work, 0, delta, status, stream);
}
