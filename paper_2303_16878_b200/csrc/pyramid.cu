// K6: cue-pyramid builder on the device.
// Reference: estimate_normals (cues.py:187-246) and _downscale_cues
// (cues.py:278-326) as composed by build_pyramid (cues.py:342-375).
//
// Normals.  The reference fits a plane to the unprojected points of a
// depth-adaptive Chebyshev window through a summed-area table of the ten
// moments [x y z xx xy xz yy yz zz 1].  The table here is built with the
// same summation chains (column-wise running sums, then row-wise), the
// window sums and the scatter matrix with the same operation order and
// explicit roundings, so everything up to the 3x3 eigenproblem is bit-equal
// to numpy.  The eigenproblem (LAPACK dsyevd behind numpy.linalg.eigh) is
// solved by cyclic Jacobi in fp64 instead: the smallest eigenvector agrees
// to ~eps * ||S|| / gap, and the planarity / grazing / orientation gates
// only differ on knife-edge inputs.  See DESIGN.md (K6) for the bound and
// tests/test_gpu_parity.py for the measured agreement.
//
// Downscale.  One thread per output cell walks its footprint in row-major
// order (the order numpy.bincount accumulates in), so intensity sums, the
// normal means and the renormalisation are bit-equal to the reference; the
// depth lower median is selected by exact rank counting.
//
// Layout: frames are batched, (n, H, W) fp64 planes; normals (n, H, W, 3).
// The moment table is scratch (n, 10, H, W) fp64.

#include <math.h>

#include "pba_common.cuh"

namespace pba {
namespace {

constexpr int kMoments = 10;

__device__ __forceinline__ bool depth_in_range(const pba_camera& cam, double d) {
  return isfinite(d) && d >= cam.depth_min && d <= cam.depth_max;
}

// unproject (sensors.py:133-154) through the host-built ray table
// (camera.ray_table): pinhole (a d, e d, d); spherical ((ce ca) d, (ce sa) d, se d).
__device__ __forceinline__ void unproject_px(const pba_camera& cam, const double* __restrict__ tab,
                                             int r, int c, double d, double& x, double& y,
                                             double& z) {
  const int W = cam.width, H = cam.height;
  if (cam.model == PBA_SPHERICAL) {
    const double ce = tab[2 * W + r], se = tab[2 * W + H + r];
    x = __dmul_rn(__dmul_rn(ce, tab[c]), d);
    y = __dmul_rn(__dmul_rn(ce, tab[W + c]), d);
    z = __dmul_rn(se, d);
  } else {
    x = __dmul_rn(tab[c], d);
    y = __dmul_rn(tab[2 * W + r], d);
    z = d;
  }
}

// Column-wise running sums of the moments (np.cumsum(stats, axis=0)).
__global__ void __launch_bounds__(128, 4) moment_colscan_kernel(pba_camera cam,
                                                             const double* __restrict__ tab,
                                                             const double* __restrict__ depth,
                                                             double* __restrict__ sat) {
  const int W = cam.width, H = cam.height;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (c >= W) return;
  const int64_t plane = (int64_t)H * W;
  const double* dp = depth + f * plane + c;
  double* out = sat + (int64_t)f * kMoments * plane + c;
  double acc[kMoments];
  for (int r = 0; r < H; ++r) {
    const double d = dp[(int64_t)r * W];
    double m[kMoments];
    if (depth_in_range(cam, d)) {
      double x, y, z;
      unproject_px(cam, tab, r, c, d, x, y, z);
      m[0] = x, m[1] = y, m[2] = z;
      m[3] = __dmul_rn(x, x), m[4] = __dmul_rn(x, y), m[5] = __dmul_rn(x, z);
      m[6] = __dmul_rn(y, y), m[7] = __dmul_rn(y, z), m[8] = __dmul_rn(z, z);
      m[9] = 1.0;
    } else {
#pragma unroll
      for (int k = 0; k < kMoments; ++k) m[k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < kMoments; ++k) {
      acc[k] = r == 0 ? m[k] : __dadd_rn(acc[k], m[k]);
      out[k * plane + (int64_t)r * W] = acc[k];
    }
  }
}

// Row-wise running sums in place (np.cumsum(..., axis=1)).  A CTA owns 32
// consecutive rows of the (frame, moment, row) row list and walks them in
// 32-column tiles staged through shared memory: coalesced tile loads and
// stores, and one thread per row carrying the sequential sum across tiles
// (the summation order of cumsum, so results are bit-equal).
__global__ void __launch_bounds__(256) moment_rowscan_kernel(int W, int64_t n_rows,
                                                             double* __restrict__ sat) {
  __shared__ double tile[32][33];
  const int64_t row0 = (int64_t)blockIdx.x * 32;
  const int t = threadIdx.x;
  double acc = 0.0;
  for (int c0 = 0; c0 < W; c0 += 32) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = t + 256 * k, r = e >> 5, c = e & 31;
      if (row0 + r < n_rows && c0 + c < W) tile[r][c] = sat[(row0 + r) * W + c0 + c];
    }
    __syncthreads();
    if (t < 32) {
      const int n = min(32, W - c0);
      for (int c = 0; c < n; ++c) {
        acc = (c0 == 0 && c == 0) ? tile[t][0] : __dadd_rn(acc, tile[t][c]);
        tile[t][c] = acc;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = t + 256 * k, r = e >> 5, c = e & 31;
      if (row0 + r < n_rows && c0 + c < W) sat[(row0 + r) * W + c0 + c] = tile[r][c];
    }
    __syncthreads();
  }
}

// One Jacobi rotation annihilating a[p][q] of the symmetric 3x3 matrix
// (diagonal d[], off-diagonal o01, o02, o12) and accumulating it into V.
__device__ __forceinline__ void jacobi_rotate(double* d, double& apq, double& arp, double& arq,
                                              int p, int q, double V[3][3]) {
  if (apq == 0.0) return;
  const double dp = d[p], dq = d[q];
  if (fabs(apq) <= 1e-18 * (fabs(dp) + fabs(dq))) {
    apq = 0.0;
    return;
  }
  const double theta = (dq - dp) / (2.0 * apq);
  double t;
  if (fabs(theta) > 1e150) {
    t = 0.5 / theta;
  } else {
    t = 1.0 / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
    if (theta < 0.0) t = -t;
  }
  const double c = 1.0 / sqrt(fma(t, t, 1.0));
  const double s = t * c;
  const double tau = s / (1.0 + c);
  d[p] = dp - t * apq;
  d[q] = dq + t * apq;
  apq = 0.0;
  const double rp = arp, rq = arq;
  arp = rp - s * (rq + tau * rp);
  arq = rq + s * (rp - tau * rq);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double vp = V[k][p], vq = V[k][q];
    V[k][p] = vp - s * (vq + tau * vp);
    V[k][q] = vq + s * (vp - tau * vq);
  }
}

__device__ __forceinline__ double sat_at(const double* __restrict__ s, int W, int R, int C) {
  return (R == 0 || C == 0) ? 0.0 : s[(int64_t)(R - 1) * W + (C - 1)];
}

// A pixel whose decision (planarity, grazing, orientation) or normal value
// could come out differently under LAPACK's eigensolver is written as zero
// and listed for the host, which re-decides it with numpy.linalg.eigh on the
// same (bit-equal) scatter matrix: record = [pixel index, S00, S11, S22,
// S10, S20, S21, x, y, z] (the lower triangle eigh reads, and the point).
constexpr int kRecheckDoubles = 10;

__global__ void __launch_bounds__(128, 6) normals_kernel(pba_camera cam,
                                                      const double* __restrict__ tab,
                                                      const double* __restrict__ depth,
                                                      const double* __restrict__ sat,
                                                      pba_normal_config cfg,
                                                      double* __restrict__ normals,
                                                      double* __restrict__ recheck,
                                                      int recheck_cap,
                                                      int* __restrict__ recheck_count) {
  const int W = cam.width, H = cam.height;
  const int64_t plane = (int64_t)H * W;
  const int64_t px = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (px >= plane) return;
  const int r = (int)(px / W), c = (int)(px - (int64_t)r * W);
  double* out = normals + (f * plane + px) * 3;
  out[0] = 0.0, out[1] = 0.0, out[2] = 0.0;
  const double d = depth[f * plane + px];
  if (!depth_in_range(cam, d)) return;
  double x, y, z;
  unproject_px(cam, tab, r, c, d, x, y, z);

  // radius = clip(round(k_tau / depth), radius_min, radius_max).astype(int)
  const double rr = fmin(fmax(rint(__ddiv_rn(cfg.k_tau, d)), cfg.radius_min), cfg.radius_max);
  const int half = (int)rr;
  const int top = min(max(r - half, 0), H), bot = min(max(r + half + 1, 0), H);
  const int lft = min(max(c - half, 0), W), rgt = min(max(c + half + 1, 0), W);
  const double* s = sat + (int64_t)f * kMoments * plane;
  double win[kMoments];
#pragma unroll
  for (int k = 0; k < kMoments; ++k) {
    const double* sk = s + k * plane;
    const double a = sat_at(sk, W, bot, rgt), b = sat_at(sk, W, top, rgt);
    const double e = sat_at(sk, W, bot, lft), g = sat_at(sk, W, top, lft);
    win[k] = __dadd_rn(__dsub_rn(__dsub_rn(a, b), e), g);
  }
  const double cnt = win[9];
  if (!(cnt >= cfg.min_points)) return;
  const double mu0 = __ddiv_rn(win[0], cnt), mu1 = __ddiv_rn(win[1], cnt),
               mu2 = __ddiv_rn(win[2], cnt);
  const double c0 = __dmul_rn(cnt, mu0), c1 = __dmul_rn(cnt, mu1), c2 = __dmul_rn(cnt, mu2);
  // lower triangle of scatter = S - (count * mu_i) * mu_j (what eigh reads)
  double dg[3] = {__dsub_rn(win[3], __dmul_rn(c0, mu0)), __dsub_rn(win[6], __dmul_rn(c1, mu1)),
                  __dsub_rn(win[8], __dmul_rn(c2, mu2))};
  double o01 = __dsub_rn(win[4], __dmul_rn(c1, mu0));
  double o02 = __dsub_rn(win[5], __dmul_rn(c2, mu0));
  double o12 = __dsub_rn(win[7], __dmul_rn(c2, mu1));
  const double s00 = dg[0], s11 = dg[1], s22 = dg[2], s10 = o01, s20 = o02, s21 = o12;
  double V[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
  for (int sweep = 0; sweep < 12; ++sweep) {
    if (o01 == 0.0 && o02 == 0.0 && o12 == 0.0) break;
    jacobi_rotate(dg, o01, o02, o12, 0, 1, V);  // other row 2: (a20, a21)
    jacobi_rotate(dg, o02, o01, o12, 0, 2, V);  // other row 1: (a10, a12)
    jacobi_rotate(dg, o12, o01, o02, 1, 2, V);  // other row 0: (a01, a02)
  }
  // ascending eigenvalues: smallest -> normal, middle/largest -> planarity
  // (selects instead of indexing keep V and dg in registers)
  double la = dg[0], lb = dg[1], lc = dg[2];
  int i0 = 0, i1 = 1, i2 = 2;
  if (la > lb) { const double t = la; la = lb; lb = t; const int u = i0; i0 = i1; i1 = u; }
  if (lb > lc) { const double t = lb; lb = lc; lc = t; const int u = i1; i1 = i2; i2 = u; }
  if (la > lb) { const double t = la; la = lb; lb = t; const int u = i0; i0 = i1; i1 = u; }
  auto pick = [](double a, double b, double c, int i) { return i == 0 ? a : (i == 1 ? b : c); };
  const double thr = fmax(__dmul_rn(cfg.degeneracy_ratio, lc), 0.0);
  double n0 = pick(V[0][0], V[0][1], V[0][2], i0);
  double n1 = pick(V[1][0], V[1][1], V[1][2], i0);
  double n2 = pick(V[2][0], V[2][1], V[2][2], i0);
  const double facing = __dadd_rn(__dadd_rn(__dmul_rn(n0, x), __dmul_rn(n1, y)), __dmul_rn(n2, z));
  if (facing > 0.0) n0 = -n0, n1 = -n1, n2 = -n2;
  // Certainty margins against any backward-stable 3x3 eigensolver (LAPACK
  // dsyevd or this Jacobi; both within ~10 eps ||S|| = 2.2e-15 ||S||):
  // eigenvalues within m_l = 2e-14 ||S||, the eigenvector within
  // err_n = 2e-14 ||S|| / gap (9x those bounds), so facing = n . p within
  // m_f = 4 |p| err_n (+ rounding).  Outside the margins the gates decide
  // identically and the normal agrees to <= 1e-10.
  const double snorm = fmax(fabs(la), fabs(lc));
  const double m_l = 2e-14 * snorm;
  const double gap = lb - la;
  const double err_n = gap > 0.0 ? 2e-14 * snorm / gap + 1e-15 : INFINITY;
  const double pn = sqrt(x * x + y * y + z * z);
  const double m_f = 4.0 * pn * err_n + 1e-15 * pn;
  const double af = fabs(facing);
  const bool finite = isfinite(n0) && isfinite(n1) && isfinite(n2);
  const bool surely_not = lb < thr - m_l || af < 1e-12 - m_f;
  const bool surely = lb > thr + m_l && af > 1e-12 + m_f && err_n <= 1e-10 && finite;
  if (surely_not) return;
  if (surely) {
    out[0] = n0, out[1] = n1, out[2] = n2;
    return;
  }
  const int k = atomicAdd(recheck_count, 1);
  if (k < recheck_cap) {
    double* rec = recheck + (int64_t)k * kRecheckDoubles;
    rec[0] = (double)(f * plane + px);
    rec[1] = s00, rec[2] = s11, rec[3] = s22, rec[4] = s10, rec[5] = s20, rec[6] = s21;
    rec[7] = x, rec[8] = y, rec[9] = z;
  }
}

// smallest source index r in [0, n] with floor(r * s) >= R
__device__ __forceinline__ int first_at_or_after(int R, double s, int n) {
  int r = max(0, (int)floor((double)R / s) - 2);
  while (r < n && floor(__dmul_rn((double)r, s)) < (double)R) ++r;
  return r;
}

__device__ __forceinline__ double norm3(double a, double b, double c) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)));
}

__global__ void __launch_bounds__(128) downscale_kernel(
    pba_camera cam, double s, int out_h, int out_w, const double* __restrict__ inten,
    const double* __restrict__ depth, const double* __restrict__ normals,
    double* __restrict__ o_i, double* __restrict__ o_d, double* __restrict__ o_n) {
  const int W = cam.width, H = cam.height;
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (cell >= (int64_t)out_h * out_w) return;
  const int R = (int)(cell / out_w), C = (int)(cell - (int64_t)R * out_w);
  const int r0 = first_at_or_after(R, s, H), r1 = first_at_or_after(R + 1, s, H);
  const int q0 = first_at_or_after(C, s, W), q1 = first_at_or_after(C + 1, s, W);
  const int64_t plane = (int64_t)H * W;
  const double* I = inten + f * plane;
  const double* D = depth + f * plane;
  const double* N = normals + f * plane * 3;
  double sum_v = 0.0, sum_a = 0.0, sn0 = 0.0, sn1 = 0.0, sn2 = 0.0;
  int cnt_v = 0, cnt_a = 0, cnt_n = 0;
  for (int r = r0; r < r1; ++r) {
    for (int q = q0; q < q1; ++q) {
      const int64_t k = (int64_t)r * W + q;
      const double iv = I[k], dv = D[k];
      sum_a = __dadd_rn(sum_a, iv);
      ++cnt_a;
      if (dv >= cam.depth_min && dv <= cam.depth_max) {
        sum_v = __dadd_rn(sum_v, iv);
        ++cnt_v;
      }
      const double a = N[3 * k], b = N[3 * k + 1], c = N[3 * k + 2];
      if (norm3(a, b, c) > 0.5) {
        sn0 = __dadd_rn(sn0, a), sn1 = __dadd_rn(sn1, b), sn2 = __dadd_rn(sn2, c);
        ++cnt_n;
      }
    }
  }
  const int64_t oc = (int64_t)f * out_h * out_w + cell;
  o_i[oc] = cnt_v > 0 ? __ddiv_rn(sum_v, (double)cnt_v) : __ddiv_rn(sum_a, (double)max(cnt_a, 1));

  // lower median of the valid depths: the member with rank (n - 1) / 2
  double med = 0.0;
  if (cnt_v > 0) {
    const int want = (cnt_v - 1) / 2;
    bool found = false;
    for (int r = r0; r < r1 && !found; ++r) {
      for (int q = q0; q < q1 && !found; ++q) {
        const double v = D[(int64_t)r * W + q];
        if (!(v >= cam.depth_min && v <= cam.depth_max)) continue;
        int lt = 0, le = 0;
        for (int r2 = r0; r2 < r1; ++r2) {
          for (int q2 = q0; q2 < q1; ++q2) {
            const double u = D[(int64_t)r2 * W + q2];
            if (!(u >= cam.depth_min && u <= cam.depth_max)) continue;
            lt += u < v;
            le += u <= v;
          }
        }
        if (lt <= want && want < le) {
          med = v;
          found = true;
        }
      }
    }
  }
  o_d[oc] = med;

  const double den = (double)max(cnt_n, 1);
  const double m0 = __ddiv_rn(sn0, den), m1 = __ddiv_rn(sn1, den), m2 = __ddiv_rn(sn2, den);
  const double nm = norm3(m0, m1, m2);
  double* on = o_n + oc * 3;
  if (cnt_n > 0 && nm >= 0.5) {
    on[0] = __ddiv_rn(m0, nm), on[1] = __ddiv_rn(m1, nm), on[2] = __ddiv_rn(m2, nm);
  } else {
    on[0] = 0.0, on[1] = 0.0, on[2] = 0.0;
  }
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" size_t pba_normals_scratch_bytes(const pba_camera* cam, int32_t n_frames) {
  if (!cam || n_frames <= 0) return 0;
  return (size_t)kMoments * cam->width * cam->height * n_frames * sizeof(double);
}

extern "C" int pba_estimate_normals(const pba_camera* cam, const double* ray_table,
                                    const double* depth, int32_t n_frames,
                                    const pba_normal_config* cfg, double* normals, void* scratch,
                                    double* recheck, int32_t recheck_capacity,
                                    int32_t* recheck_count, void* stream) {
  PBA_ARG_CHECK(cam && cfg, "NULL camera/config");
  PBA_ARG_CHECK(n_frames >= 0, "n_frames < 0");
  PBA_ARG_CHECK(recheck_count && recheck_capacity >= 0 && (recheck || recheck_capacity == 0),
                "bad recheck buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PBA_CUDA_TRY(cudaMemsetAsync(recheck_count, 0, sizeof(int32_t), st));
  if (n_frames == 0 || cam->width == 0 || cam->height == 0) return PBA_OK;
  PBA_ARG_CHECK(n_frames <= 65535, "n_frames > 65535 per call");
  PBA_ARG_CHECK(ray_table && depth && normals && scratch, "NULL buffer");
  double* sat = static_cast<double*>(scratch);
  const int W = cam->width, H = cam->height;
  moment_colscan_kernel<<<dim3((W + 127) / 128, n_frames), 128, 0, st>>>(*cam, ray_table, depth,
                                                                         sat);
  PBA_LAUNCH_CHECK();
  const int64_t rows = (int64_t)n_frames * kMoments * H;
  moment_rowscan_kernel<<<(unsigned)((rows + 31) / 32), 256, 0, st>>>(W, rows, sat);
  PBA_LAUNCH_CHECK();
  const int64_t plane = (int64_t)H * W;
  normals_kernel<<<dim3((unsigned)((plane + 127) / 128), n_frames), 128, 0, st>>>(
      *cam, ray_table, depth, sat, *cfg, normals, recheck, recheck_capacity, recheck_count);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

extern "C" int pba_downscale_cues(const pba_camera* cam, double scale, int32_t n_frames,
                                  const double* intensity, const double* depth,
                                  const double* normals, int32_t out_h, int32_t out_w,
                                  double* out_intensity, double* out_depth, double* out_normals,
                                  void* stream) {
  PBA_ARG_CHECK(cam, "NULL camera");
  PBA_ARG_CHECK(scale > 0.0 && scale <= 1.0, "scale outside (0, 1]");
  PBA_ARG_CHECK(n_frames >= 0 && n_frames <= 65535, "n_frames outside [0, 65535]");
  PBA_ARG_CHECK(out_h == (int)floor(cam->height * scale) && out_w == (int)floor(cam->width * scale),
                "output size is not floor(size * scale)");
  const int64_t cells = (int64_t)out_h * out_w;
  if (n_frames == 0 || cells == 0) return PBA_OK;
  PBA_ARG_CHECK(intensity && depth && normals && out_intensity && out_depth && out_normals,
                "NULL buffer");
  downscale_kernel<<<dim3((unsigned)((cells + 127) / 128), n_frames), 128, 0,
                     static_cast<cudaStream_t>(stream)>>>(*cam, scale, out_h, out_w, intensity,
                                                          depth, normals, out_intensity,
                                                          out_depth, out_normals);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
