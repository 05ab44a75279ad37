// K1: fused warp + residual + Jacobian + Huber + JᵀWJ/JᵀWe accumulation.
//
// Reference chain (all per source pixel of one directed pair i -> j):
//   PairContext.build     solver.py:198-220  (source pixels, p_u)
//   PairContext.evaluate  solver.py:222-303  (warp, sample, residuals, J)
//   sample_cues           cues.py:433-457    (bilinear values + gradients)
//   project / Jacobian    sensors.py:95-130, 157-188
//   robust_cue_weights    solver.py:317-337
//   _edge_term            solver.py:356-390  (block sums)
//
// Work decomposition: one CTA per chunk of `chunk_pixels` consecutive source
// pixels of one pair (row-major over the strided source grid).  A thread
// walks pixels tid, tid+256, ... so a warp reads 32 consecutive source
// texels and samples a compact destination footprint.  Per-thread sums
// live in registers (H in fp32, b/cost in fp64), are reduced by a fixed
// warp-shuffle tree and a fixed cross-warp order into one 92-double partial
// per chunk; a second kernel sums the chunk partials of each pair in chunk
// order.  No atomics: results are bit-identical run to run and independent
// of how pairs are spread over GPUs.
//
// Precision: geometry, cue values, residuals, Huber
// weights, Jacobians, b and cost in fp64; only the H outer products are
// accumulated in fp32 per thread (<= chunk_pixels/256 terms) before being
// promoted to fp64 in the reductions.

#include <math.h>

#include "pba_common.cuh"

namespace pba {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kH = 78;  // 21 + 21 + 36 fp32 accumulators

struct PairSetup {
  double Ri[9], Rj[9], Ro[9];
  double Mi[9];    // R_o^T R_j^T R_i                       (solver.py:265)
  double rotn[9];  // R_o^T R_j^T R_i R_o                   (solver.py:241)
  double dt[3];    // t_i - t_j                             (solver.py:235)
  double to[3];
  double occ_tol;
  const Texel* src_tex;
  const uint8_t* src_mask;
  const double* src_ray;
  const Texel* dst_tex;
  const uint8_t* dst_mask;
  pba_camera src_cam, dst_cam;
  int grid_w, n_px, stride;
};

__device__ __forceinline__ void matmul3(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C[3 * r + c] = A[3 * r + 0] * B[0 + c] + A[3 * r + 1] * B[3 + c] + A[3 * r + 2] * B[6 + c];
}
__device__ __forceinline__ void transpose3(const double* A, double* T) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) T[3 * c + r] = A[3 * r + c];
}

__device__ void build_setup(PairSetup& S, const pba_frame* frames, const pba_pair& P,
                            const double* poses, const double* exts, int stride) {
  const double* xi = poses + 12 * P.pose_i;
  const double* xj = poses + 12 * P.pose_j;
  const double* xo = exts + 12 * P.ext;
  for (int k = 0; k < 9; ++k) {
    S.Ri[k] = xi[k];
    S.Rj[k] = xj[k];
    S.Ro[k] = xo[k];
  }
  for (int k = 0; k < 3; ++k) {
    S.dt[k] = xi[9 + k] - xj[9 + k];
    S.to[k] = xo[9 + k];
  }
  double RoT[9], RjT[9], tmp[9];
  transpose3(S.Ro, RoT);
  transpose3(S.Rj, RjT);
  matmul3(RoT, RjT, tmp);
  matmul3(tmp, S.Ri, S.Mi);
  matmul3(S.Mi, S.Ro, S.rotn);
  S.occ_tol = P.occ_tol;
  const pba_frame& fs = frames[P.src];
  const pba_frame& fd = frames[P.dst];
  S.src_tex = static_cast<const Texel*>(fs.texels);
  S.src_mask = fs.mask;
  S.src_ray = fs.ray_table;
  S.dst_tex = static_cast<const Texel*>(fd.texels);
  S.dst_mask = fd.mask;
  S.src_cam = fs.cam;
  S.dst_cam = fd.cam;
  S.stride = stride;
  const int gw = (fs.cam.width + stride - 1) / stride;
  const int gh = (fs.cam.height + stride - 1) / stride;
  S.grid_w = gw;
  S.n_px = gw * gh;
}

// numpy float modulus for a positive divisor (np.mod, sensors.py:122).
__device__ __forceinline__ double py_mod(double a, double w) {
  double m = fmod(a, w);
  if (m != 0.0) {
    if (m < 0.0) m += w;
  } else {
    m = 0.0;  // copysign(0, w) with w > 0
  }
  return m;
}

__device__ __forceinline__ double bil(double v00, double v01, double v10, double v11, double wx,
                                      double wy) {
  // cues.py:394, same association.
  return (1.0 - wy) * ((1.0 - wx) * v00 + wx * v01) + wy * ((1.0 - wx) * v10 + wx * v11);
}

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

template <int K, int L>
struct Upper {
  static constexpr int idx = K * 6 - (K * (K - 1)) / 2 + (L - K);
};

__device__ __forceinline__ int upper_idx(int k, int l) { return k * 6 - (k * (k - 1)) / 2 + (l - k); }

// Rank-1 updates of the three blocks with one channel's Jacobian rows.
__device__ __forceinline__ void accumulate_h(float* h, const double* Ji, const double* Jj,
                                             double ww) {
  float fi[6], fj[6], ai[6], aj[6];
  const float wf = (float)ww;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    fi[k] = (float)Ji[k];
    fj[k] = (float)Jj[k];
    ai[k] = wf * fi[k];
    aj[k] = wf * fj[k];
  }
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int l = k; l < 6; ++l) {
      h[upper_idx(k, l)] = fmaf(ai[k], fi[l], h[upper_idx(k, l)]);
      h[21 + upper_idx(k, l)] = fmaf(aj[k], fj[l], h[21 + upper_idx(k, l)]);
    }
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int l = 0; l < 6; ++l) h[42 + 6 * k + l] = fmaf(ai[k], fj[l], h[42 + 6 * k + l]);
}

template <bool kJac>
__global__ void __launch_bounds__(kThreads, 1)
    linearize_kernel(const pba_frame* __restrict__ frames, const pba_pair* __restrict__ pairs,
                     const int32_t* __restrict__ chunk_table, int chunk_pixels,
                     const double* __restrict__ poses, const double* __restrict__ exts,
                     pba_config cfg, double* __restrict__ partials) {
  __shared__ PairSetup S;
  __shared__ double red[kWarps][kRec];

  const long chunk = blockIdx.x;
  const int pair = chunk_table[2 * chunk];
  const int first = chunk_table[2 * chunk + 1];
  if (threadIdx.x == 0) build_setup(S, frames, pairs[pair], poses, exts, cfg.pixel_stride);
  __syncthreads();

  float h[kH];
#pragma unroll
  for (int k = 0; k < kH; ++k) h[k] = 0.f;
  double bi[6], bj[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) bi[k] = bj[k] = 0.0;
  double cost = 0.0;
  int count = 0;

  const int last = min(first + chunk_pixels, S.n_px);
  const int sW = S.src_cam.width, sH = S.src_cam.height;
  const int dW = S.dst_cam.width, dH = S.dst_cam.height;
  const bool src_sph = S.src_cam.model == PBA_SPHERICAL;
  const bool dst_sph = S.dst_cam.model == PBA_SPHERICAL;
  const double dWd = (double)dW, dHd = (double)dH;

  for (int idx = first + (int)threadIdx.x; idx < last; idx += kThreads) {
    const int gr = idx / S.grid_w;
    const int row = gr * S.stride;
    const int col = (idx - gr * S.grid_w) * S.stride;
    const int sp = row * sW + col;
    const uint32_t sm = __ldg(S.src_mask + sp);
    if (!(sm & PBA_MASK_DEPTH_VALID)) continue;  // PairContext.build: usable = depth_valid

    // ---- source cue values and unprojection (sensors.py:133-154) ----
    const double2* st = reinterpret_cast<const double2*>(S.src_tex + sp);
    const double2 s_id = __ldg(st + 0);   // I, D
    const double2 s_n01 = __ldg(st + 1);  // nx, ny
    const double s_n2 = __ldg(&S.src_tex[sp].v[4]);
    const double d = s_id.y;
    double ps[3];
    if (src_sph) {
      const double ca = __ldg(S.src_ray + col), sa = __ldg(S.src_ray + sW + col);
      const double ce = __ldg(S.src_ray + 2 * sW + row), se = __ldg(S.src_ray + 2 * sW + sH + row);
      ps[0] = (ce * ca) * d;
      ps[1] = (ce * sa) * d;
      ps[2] = se * d;
    } else {
      ps[0] = __ldg(S.src_ray + col) * d;
      ps[1] = __ldg(S.src_ray + 2 * sW + row) * d;
      ps[2] = d;
    }
    // p_u = R_o p + t_o (solver.py:215)
    double pu[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      pu[k] = S.Ro[3 * k + 0] * ps[0] + S.Ro[3 * k + 1] * ps[1] + S.Ro[3 * k + 2] * ps[2] + S.to[k];
    // g = R_j^T (R_i p_u + t_i - t_j);  p_bar = R_o^T (g - t_o)   (solver.py:235-236)
    double q[3], g[3], pb[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      q[k] = S.Ri[3 * k + 0] * pu[0] + S.Ri[3 * k + 1] * pu[1] + S.Ri[3 * k + 2] * pu[2] + S.dt[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) g[k] = q[0] * S.Rj[k] + q[1] * S.Rj[3 + k] + q[2] * S.Rj[6 + k];
    {
      const double a0 = g[0] - S.to[0], a1 = g[1] - S.to[1], a2 = g[2] - S.to[2];
#pragma unroll
      for (int k = 0; k < 3; ++k) pb[k] = a0 * S.Ro[k] + a1 * S.Ro[3 + k] + a2 * S.Ro[6 + k];
    }

    // ---- project into the destination (sensors.py:95-130) ----
    double u, v, dist;
    if (dst_sph) {
      const double az = atan2(pb[1], pb[0]);
      const double el = atan2(pb[2], hypot(pb[0], pb[1]));
      u = py_mod(S.dst_cam.fx * az + S.dst_cam.cx, dWd);
      v = S.dst_cam.fy * el + S.dst_cam.cy;
      dist = sqrt((pb[0] * pb[0] + pb[1] * pb[1]) + pb[2] * pb[2]);
    } else {
      if (!(pb[2] > 0.0)) continue;
      u = S.dst_cam.fx * pb[0] / pb[2] + S.dst_cam.cx;
      v = S.dst_cam.fy * pb[1] / pb[2] + S.dst_cam.cy;
      dist = pb[2];
    }
    if (!(dist >= S.dst_cam.depth_min && dist <= S.dst_cam.depth_max)) continue;
    if (!(u >= 0.0 && u < dWd && v >= 0.0 && v < dHd)) continue;

    // ---- bilinear footprint and validity (cues.py:397-409, 451-456) ----
    if (!(u <= dWd - 1.0 && v <= dHd - 1.0)) continue;  // inside (u, v >= 0 already)
    int x0 = (int)floor(u), y0 = (int)floor(v);
    x0 = min(max(x0, 0), dW - 2);
    y0 = min(max(y0, 0), dH - 2);
    const double wx = u - x0, wy = v - y0;
    const int dp = y0 * dW + x0;
    const uint32_t mk = __ldg(S.dst_mask + dp) & __ldg(S.dst_mask + dp + 1) &
                        __ldg(S.dst_mask + dp + dW) & __ldg(S.dst_mask + dp + dW + 1);
    if (!(mk & PBA_MASK_SAMP_CORE)) continue;  // core_ok
    const Texel* t00 = S.dst_tex + dp;
    const Texel* t01 = t00 + 1;
    const Texel* t10 = t00 + dW;
    const Texel* t11 = t10 + 1;

    const double2 a00 = __ldg(reinterpret_cast<const double2*>(t00));
    const double2 a01 = __ldg(reinterpret_cast<const double2*>(t01));
    const double2 a10 = __ldg(reinterpret_cast<const double2*>(t10));
    const double2 a11 = __ldg(reinterpret_cast<const double2*>(t11));
    const double Dd = bil(a00.y, a01.y, a10.y, a11.y, wx, wy);
    // zeta_d: range for spherical, z for pinhole (solver.py:240)
    const double zeta = dst_sph ? dist : pb[2];
    const double e1 = zeta - Dd;
    if (e1 > S.occ_tol) continue;  // occluded (solver.py:254-258)
    double rho2 = 0.0;
    if (kJac && dst_sph) {
      rho2 = pb[0] * pb[0] + pb[1] * pb[1];
      if (!(rho2 > 0.0)) continue;  // ok_jac (sensors.py:173-175; solver.py:262-263)
    }
    const double Id = bil(a00.x, a01.x, a10.x, a11.x, wx, wy);
    const double e0 = s_id.x - Id;

    const bool normal_on = (mk & PBA_MASK_SAMP_NORMAL) && (sm & PBA_MASK_NORMAL_VALID);
    double e2 = 0.0, e3 = 0.0, e4 = 0.0;
    const double ns[3] = {s_n01.x, s_n01.y, s_n2};
    if (normal_on) {
      const double2 b00 = __ldg(reinterpret_cast<const double2*>(t00) + 1);
      const double2 b01 = __ldg(reinterpret_cast<const double2*>(t01) + 1);
      const double2 b10 = __ldg(reinterpret_cast<const double2*>(t10) + 1);
      const double2 b11 = __ldg(reinterpret_cast<const double2*>(t11) + 1);
      const double c00 = __ldg(&t00->v[4]), c01 = __ldg(&t01->v[4]);
      const double c10 = __ldg(&t10->v[4]), c11 = __ldg(&t11->v[4]);
      double mn[3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        mn[k] = ns[0] * S.rotn[3 * k + 0] + ns[1] * S.rotn[3 * k + 1] + ns[2] * S.rotn[3 * k + 2];
      e2 = mn[0] - bil(b00.x, b01.x, b10.x, b11.x, wx, wy);
      e3 = mn[1] - bil(b00.y, b01.y, b10.y, b11.y, wx, wy);
      e4 = mn[2] - bil(c00, c01, c10, c11, wx, wy);
    }

    // ---- per-cue Huber (solver.py:317-337) ----
    const double sI = sqrt(e0 * e0 * cfg.omega[0]);
    const double sD = sqrt(e1 * e1 * cfg.omega[1]);
    const double sN = sqrt((e2 * e2 * cfg.omega[2] + e3 * e3 * cfg.omega[3]) + e4 * e4 * cfg.omega[4]);
    const double dI = cfg.huber_delta[0], dD = cfg.huber_delta[1], dN = cfg.huber_delta[2];
    const bool smI = sI <= dI, smD = sD <= dD, smN = sN <= dN;
    const double wI = smI ? 1.0 : dI / sI;
    const double wD = smD ? 1.0 : dD / sD;
    const double wN = smN ? 1.0 : dN / sN;
    cost += (smI ? sI * sI : dI * (2.0 * sI - dI)) + (smD ? sD * sD : dD * (2.0 * sD - dD)) +
            (smN ? sN * sN : dN * (2.0 * sN - dN));
    ++count;
    if (!kJac) continue;

    // ---- projective Jacobian (sensors.py:157-188) ----
    double P0[3], P1[3];
    if (dst_sph) {
      const double rho = sqrt(rho2);
      const double r2 = rho2 + pb[2] * pb[2];
      P0[0] = S.dst_cam.fx * (-pb[1] / rho2);
      P0[1] = S.dst_cam.fx * (pb[0] / rho2);
      P0[2] = 0.0;
      P1[0] = S.dst_cam.fy * (-pb[0] * pb[2] / (rho * r2));
      P1[1] = S.dst_cam.fy * (-pb[1] * pb[2] / (rho * r2));
      P1[2] = S.dst_cam.fy * (rho / r2);
    } else {
      const double iz = 1.0 / pb[2];
      P0[0] = S.dst_cam.fx * iz;
      P0[1] = 0.0;
      P0[2] = -S.dst_cam.fx * pb[0] * iz * iz;
      P1[0] = 0.0;
      P1[1] = S.dst_cam.fy * iz;
      P1[2] = -S.dst_cam.fy * pb[1] * iz * iz;
    }
    // depth cue direction: unit p_bar (spherical) or e_z (pinhole)  (solver.py:279-286)
    double ud[3];
    if (dst_sph) {
      ud[0] = pb[0] / zeta;
      ud[1] = pb[1] / zeta;
      ud[2] = pb[2] / zeta;
    } else {
      ud[0] = 0.0;
      ud[1] = 0.0;
      ud[2] = 1.0;
    }
    const double es[5] = {e0, e1, e2, e3, e4};
    const double wwc[5] = {wI * cfg.omega[0], wD * cfg.omega[1], wN * cfg.omega[2],
                           wN * cfg.omega[3], wN * cfg.omega[4]};
    // normal-cue rotation blocks need R_o n and R_j^T R_i R_o n (solver.py:287-291)
    double no[3] = {0.0, 0.0, 0.0}, np_[3] = {0.0, 0.0, 0.0};
    if (normal_on) {
#pragma unroll
      for (int k = 0; k < 3; ++k)
        no[k] = S.Ro[3 * k + 0] * ns[0] + S.Ro[3 * k + 1] * ns[1] + S.Ro[3 * k + 2] * ns[2];
      double ri[3];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        ri[k] = S.Ri[3 * k + 0] * no[0] + S.Ri[3 * k + 1] * no[1] + S.Ri[3 * k + 2] * no[2];
#pragma unroll
      for (int k = 0; k < 3; ++k) np_[k] = ri[0] * S.Rj[k] + ri[1] * S.Rj[3 + k] + ri[2] * S.Rj[6 + k];
    }
    const int n_ch = normal_on ? 5 : 2;
    for (int c = 0; c < n_ch; ++c) {
      // bilinear gradient of channel c (gradients interpolate the
      // central-difference images, cues.py:448-450)
      const double2 g00 = __ldg(reinterpret_cast<const double2*>(&t00->g[2 * c]));
      const double2 g01 = __ldg(reinterpret_cast<const double2*>(&t01->g[2 * c]));
      const double2 g10 = __ldg(reinterpret_cast<const double2*>(&t10->g[2 * c]));
      const double2 g11 = __ldg(reinterpret_cast<const double2*>(&t11->g[2 * c]));
      const double gc = bil(g00.x, g01.x, g10.x, g11.x, wx, wy);
      const double gr_ = bil(g00.y, g01.y, g10.y, g11.y, wx, wy);
      double vv[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) vv[k] = -(gc * P0[k] + gr_ * P1[k]);
      if (c == 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) vv[k] += ud[k];
      }
      double Ji[6], Jj[6], w[3], wp[3], t[3];
      // v^T a_i = [M_i^T v, -2 (M_i^T v) x p_u]
#pragma unroll
      for (int k = 0; k < 3; ++k) w[k] = vv[0] * S.Mi[k] + vv[1] * S.Mi[3 + k] + vv[2] * S.Mi[6 + k];
      cross3(w, pu, t);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        Ji[k] = w[k];
        Ji[3 + k] = -2.0 * t[k];
      }
      // v^T a_j = [-R_o v, 2 (R_o v) x g]
#pragma unroll
      for (int k = 0; k < 3; ++k)
        wp[k] = S.Ro[3 * k + 0] * vv[0] + S.Ro[3 * k + 1] * vv[1] + S.Ro[3 * k + 2] * vv[2];
      cross3(wp, g, t);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        Jj[k] = -wp[k];
        Jj[3 + k] = 2.0 * t[k];
      }
      if (c >= 2) {
        const int r = c - 2;
        const double mrow[3] = {S.Mi[3 * r + 0], S.Mi[3 * r + 1], S.Mi[3 * r + 2]};
        const double rcol[3] = {S.Ro[r], S.Ro[3 + r], S.Ro[6 + r]};
        double x1[3], x2[3];
        cross3(mrow, no, x1);
        cross3(rcol, np_, x2);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          Ji[3 + k] -= 2.0 * x1[k];
          Jj[3 + k] += 2.0 * x2[k];
        }
      }
      const double ww = wwc[c];
      const double we = ww * es[c];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        bi[k] += Ji[k] * we;
        bj[k] += Jj[k] * we;
      }
      accumulate_h(h, Ji, Jj, ww);
    }
  }

  // ---- fixed-order reduction: warp butterfly, then warps in order ----
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double cnt = (double)count;
  if (kJac) {
#pragma unroll
    for (int k = 0; k < kH; ++k) {
      float x = h[k];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
      h[k] = x;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      double x = bi[k], y = bj[k];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        x += __shfl_xor_sync(0xffffffffu, x, off);
        y += __shfl_xor_sync(0xffffffffu, y, off);
      }
      bi[k] = x;
      bj[k] = y;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    cost += __shfl_xor_sync(0xffffffffu, cost, off);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  if (lane == 0) {
    double* r = red[warp];
    if (kJac) {
#pragma unroll
      for (int k = 0; k < kH; ++k) r[k] = (double)h[k];
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        r[PBA_REC_BI + k] = bi[k];
        r[PBA_REC_BJ + k] = bj[k];
      }
    } else {
      for (int k = 0; k < PBA_REC_COST; ++k) r[k] = 0.0;
    }
    r[PBA_REC_COST] = cost;
    r[PBA_REC_COUNT] = cnt;
  }
  __syncthreads();
  if (threadIdx.x < kRec) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[w][threadIdx.x];
    partials[chunk * kRec + threadIdx.x] = s;
  }
}

// Sum chunk partials of each pair in chunk order (fixed) -> per-pair record.
__global__ void reduce_chunks_kernel(const double* __restrict__ partials,
                                     const int32_t* __restrict__ offsets, int n_pairs,
                                     double* __restrict__ records) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)n_pairs * kRec) return;
  const int p = (int)(t / kRec), e = (int)(t - (long)p * kRec);
  const int c0 = offsets[p], c1 = offsets[p + 1];
  double s = 0.0;
  for (int c = c0; c < c1; ++c) s += partials[(long)c * kRec + e];
  records[t] = s;
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" int pba_plan_chunks(pba_pair* pairs, int32_t n_pairs, const pba_camera* src_cams,
                               int32_t pixel_stride, int32_t chunk_pixels, int32_t* chunk_table,
                               int32_t* pair_chunk_offsets, int64_t* n_chunks_out) {
  PBA_ARG_CHECK(n_pairs >= 0, "n_pairs < 0");
  PBA_ARG_CHECK(pixel_stride >= 1, "pixel_stride must be >= 1");
  PBA_ARG_CHECK(chunk_pixels >= 1, "chunk_pixels must be >= 1");
  PBA_ARG_CHECK(n_pairs == 0 || (pairs && src_cams), "NULL pairs/cameras");
  int64_t total = 0;
  for (int p = 0; p < n_pairs; ++p) {
    const pba_camera& c = src_cams[p];
    const int64_t gw = (c.width + pixel_stride - 1) / pixel_stride;
    const int64_t gh = (c.height + pixel_stride - 1) / pixel_stride;
    const int64_t npx = gw * gh;
    PBA_ARG_CHECK(npx < (int64_t)1 << 31, "source image too large");
    const int64_t nc = npx == 0 ? 0 : (npx + chunk_pixels - 1) / chunk_pixels;
    pairs[p].n_chunks = (int32_t)nc;
    if (pair_chunk_offsets) pair_chunk_offsets[p] = (int32_t)total;
    if (chunk_table) {
      for (int64_t k = 0; k < nc; ++k) {
        chunk_table[2 * (total + k)] = p;
        chunk_table[2 * (total + k) + 1] = (int32_t)(k * chunk_pixels);
      }
    }
    total += nc;
  }
  PBA_ARG_CHECK(total < (int64_t)1 << 31, "too many chunks");
  if (pair_chunk_offsets) pair_chunk_offsets[n_pairs] = (int32_t)total;
  if (n_chunks_out) *n_chunks_out = total;
  return PBA_OK;
}

extern "C" int pba_linearize(const pba_frame* frames, const pba_pair* pairs, int32_t n_pairs,
                             const int32_t* chunk_table, int64_t n_chunks,
                             const int32_t* pair_chunk_offsets, int32_t chunk_pixels,
                             const double* poses, const double* extrinsics,
                             const pba_config* cfg, int32_t want_jacobians, double* partials,
                             double* records, void* stream) {
  PBA_ARG_CHECK(cfg != nullptr, "cfg is NULL");
  PBA_ARG_CHECK(cfg->pixel_stride >= 1, "pixel_stride must be >= 1");
  PBA_ARG_CHECK(chunk_pixels >= 1, "chunk_pixels must be >= 1");
  PBA_ARG_CHECK(n_chunks >= 0 && n_chunks < ((int64_t)1 << 31), "bad n_chunks");
  if (n_pairs == 0) return PBA_OK;
  PBA_ARG_CHECK(frames && pairs && chunk_table && pair_chunk_offsets && poses && extrinsics &&
                    partials && records,
                "NULL buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_chunks > 0) {
    if (want_jacobians)
      linearize_kernel<true><<<(unsigned)n_chunks, kThreads, 0, st>>>(
          frames, pairs, chunk_table, chunk_pixels, poses, extrinsics, *cfg, partials);
    else
      linearize_kernel<false><<<(unsigned)n_chunks, kThreads, 0, st>>>(
          frames, pairs, chunk_table, chunk_pixels, poses, extrinsics, *cfg, partials);
    PBA_LAUNCH_CHECK();
  }
  const long total = (long)n_pairs * kRec;
  reduce_chunks_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      partials, pair_chunk_offsets, n_pairs, records);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
