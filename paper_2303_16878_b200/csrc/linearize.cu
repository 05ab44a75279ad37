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
// Structure exploited.  The reference builds, per pixel and cue channel c,
// J_i = v_c^T a_i (+ normal-cue rotation terms) and J_j = v_c^T a_j (+ ...),
// with a_i = M_i [I | -2[p_u]x], a_j = [-R_o^T | 2 R_o^T [g]x]
// (solver.py:265-293).  Because M_i = R_o^T R_j^T R_i and A = R_j^T R_i are
// rotations and g = A p_u + t_g (t_g = R_j^T (t_i - t_j)), both rows are
// fixed linear maps of ONE 6-vector per channel,
//     q_c = [u; r],  u = M_i^T v_c,  r = u x p_u (+ m_k x R_o n for normal k),
//     J_i = D q_c,   J_j = L q_c,   D = diag(1,1,1,-2,-2,-2),
//     L = [[-A, 0], [-2 [t_g]x A, 2A]],
// (the normal-cue terms fold in because A (m_k x n) = (R_o e_k) x (A n)).
// So a pixel only adds ww q q^T (21 numbers) and q ww e (6) to per-thread
// sums, and the per-pair finalisation forms H_ii = D Q D, H_jj = L Q L^T,
// H_ij = D Q L^T, b_i = D beta, b_j = L beta once.  That cuts the per-pixel
// accumulation from 78+12 to 21+6 fp64 FMAs per channel-row and the live
// accumulators from 92 to 29, which lets everything — geometry, cue values,
// residuals, Huber weights, Jacobians and the sums — stay in fp64 (SURVEY.md
// App. B; fp32 H partials measurably broke the 1e-6 LM-cost parity).
//
// Work decomposition: one CTA per chunk of consecutive source pixels of one
// pair (row-major over the strided source grid; whole 8-row bands where the
// grid allows, pair_chunk_pixels).  128-thread CTAs, 3 per SM at 168
// registers.  A band is walked in 16 x 8 tiles (a warp: 16 columns x 2 rows),
// so the CTA's warps read 16-pixel source row segments and sample one
// compact, shared destination footprint; other chunks are walked row-major
// (thread tid takes pixels tid, tid + 128, ...).  Texels are the plane layout of
// pba_common.cuh (16-byte pairs, plane-major).  Per-thread sums are
// reduced by a fixed warp-shuffle tree and a fixed cross-warp order into one
// 32-double partial per chunk; a finalisation kernel sums the chunk partials
// of each pair in chunk order and expands them into the 92-double record.
// No atomics: results are bit-identical run to run and independent of how
// pairs are spread over GPUs.

#include <math.h>
#include <stdlib.h>

#include <cmath>

#include "fastmath.cuh"
#include "pba_common.cuh"

namespace pba {

// The table is built on the host in double-double arithmetic: for each
// theta_k = k pi / 256, (c, s) = cos/sin rounded to double, and the exact
// angle of the rounded pair (theta_k + asin(s cos - c sin) with the
// cross-difference taken in double-double) is stored as hi + lo.
namespace {
struct DD {
  double hi, lo;
};
DD two_prod(double a, double b) {
  const double p = a * b;
  return {p, std::fma(a, b, -p)};
}
DD two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  s.lo += a.lo + b.lo;
  return two_sum(s.hi, s.lo);
}
DD dd_mul(DD a, DD b) {
  DD p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return two_sum(p.hi, p.lo);
}
DD dd_neg(DD a) { return {-a.hi, -a.lo}; }
// cos/sin of a double-double angle by Taylor series (|x| <= pi)
void dd_sincos(DD x, DD& c, DD& s) {
  // reduce by halving: compute for x / 2^8, then double the angle 8 times
  DD y = {std::ldexp(x.hi, -8), std::ldexp(x.lo, -8)};
  DD y2 = dd_mul(y, y);
  DD sn = y, cn = {1.0, 0.0}, term = y;
  for (int n = 1; n < 12; ++n) {  // sin series
    term = dd_mul(term, y2);
    const double f = 1.0 / ((2.0 * n) * (2.0 * n + 1.0));
    term = dd_mul(term, DD{-f, 0.0});
    sn = dd_add(sn, term);
  }
  term = {1.0, 0.0};
  for (int n = 1; n < 12; ++n) {  // cos series
    term = dd_mul(term, y2);
    const double f = 1.0 / ((2.0 * n - 1.0) * (2.0 * n));
    term = dd_mul(term, DD{-f, 0.0});
    cn = dd_add(cn, term);
  }
  for (int i = 0; i < 8; ++i) {  // double-angle formulas
    DD s2 = dd_mul(DD{2.0, 0.0}, dd_mul(sn, cn));
    DD c2 = dd_add(dd_mul(cn, cn), dd_neg(dd_mul(sn, sn)));
    sn = s2;
    cn = c2;
  }
  c = cn;
  s = sn;
}
}  // namespace

int ensure_atan_table() {
  static bool done[64] = {false};
  int dev = 0;
  PBA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && done[dev]) return PBA_OK;
  static AtanEntry host[2 * kAtanHalf + 1];
  const DD pi = {3.141592653589793116, 1.2246467991473532e-16};
  for (int k = -kAtanHalf; k <= kAtanHalf; ++k) {
    const DD th = dd_mul(pi, DD{(double)k / kAtanHalf, 0.0});  // k/256 is exact
    DD cd, sd;
    dd_sincos(th, cd, sd);
    const double c = cd.hi + cd.lo, s = sd.hi + sd.lo;  // rounded cos/sin
    // exact angle of (c, s): th + asin((s cos th - c sin th) / |(c, s)|)
    const DD cross = dd_add(dd_mul(DD{s, 0.0}, cd), dd_neg(dd_mul(DD{c, 0.0}, sd)));
    const double r = std::sqrt(c * c + s * s);
    const double u = (cross.hi + cross.lo) / r;
    const double du = u + u * u * u / 6.0;  // |u| < 1e-16: asin(u) = u to double precision
    const DD ang = dd_add(th, DD{du, 0.0});
    host[k + kAtanHalf] = AtanEntry{c, s, ang.hi, ang.lo};
  }
  PBA_CUDA_TRY(cudaMemcpyToSymbol(g_atan_table, host, sizeof(host)));
  if (dev >= 0 && dev < 64) done[dev] = true;
  return PBA_OK;
}

namespace {

__global__ void atan2_batch_kernel(const double* y, const double* x, int64_t n, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = atan2_tab(y[i], x[i]);
}

constexpr int kThreads = 256;  // default CTA size
constexpr int kQ = 21;    // upper triangle of Q (6x6)
constexpr int kPart = 32; // chunk partial: Q[21], beta[6], cost, count, pad
constexpr int kTileCols = 16, kTileRows = 8;  // K1's tiled walk (128 threads)

// Source pixels per chunk of a pair whose strided grid is gw wide.  Grids
// at least 8 rows of which fit in the launch's chunk_pixels, with a width
// that is a multiple of 16, get chunks of whole 8-row bands (the multiple of
// 8 rows nearest chunk_pixels), which K1 walks in 16 x 8 tiles; others use
// chunk_pixels.  Host (pba_plan_chunks) and device use the same rule.
__host__ __device__ inline int pair_chunk_pixels(int gw, int chunk_pixels) {
  if (gw <= 0 || gw % kTileCols != 0 || kTileRows * gw > chunk_pixels) return chunk_pixels;
  const int bands = (chunk_pixels + kTileRows * gw / 2) / (kTileRows * gw);
  return bands * kTileRows * gw;
}

struct PairSetup {
  double Ri[9], Rj[9], Ro[9];
  double Mi[9];    // R_o^T R_j^T R_i                       (solver.py:265)
  double rotn[9];  // R_o^T R_j^T R_i R_o                   (solver.py:241)
  double dt[3];    // t_i - t_j                             (solver.py:235)
  double to[3];
  double cpb[3];   // R_o^T (R_j^T (t_i - t_j) - t_o): p_bar = M_i p_u + cpb
  double occ_tol;
  const double2* src_tex;  // texel planes (pba_common.cuh): pair k of pixel p at [k * src_np + p]
  const uint8_t* src_mask;
  const double* src_ray;
  const double2* dst_tex;
  const uint8_t* dst_mask;
  pba_camera src_cam, dst_cam;
  int grid_w, n_px, stride;
  int src_np, dst_np;  // pixels per texel plane
  pba_config cfg;      // the launch's config (read through SV in the loop)
  double sqw0, sqw1;   // sqrt(omega_I), sqrt(omega_D)
  // kLean: the three 3x3 maps as 16-byte-aligned rows of four, read as two
  // 16-byte shared loads per row: [R_o | t_o], [M_i | cpb], [rot_n | 0]
  alignas(16) double RoT[12];
  alignas(16) double MiC[12];
  alignas(16) double Rn[12];
  // kLean: scalars the pixel loop reads together, paired for 16-byte loads
  alignas(16) double fx_cx[2], fy_cy[2], fx_fy[2], range[2], wh[2];
  alignas(16) double sqw0_dI[2], sqw1_dD[2], om01[2], om23[2], om4_dN[2];
  alignas(8) int dwh[2], np_sd[2];
  alignas(16) int src_geo[4];      // stride, source width, source plane size, grid width
  alignas(8) int src_mh[2];        // source model, source height
  alignas(16) const void* src_ptrs[2];  // source texels, source ray table
};

// Loop reads of the CTA's pair setup.  kLean: every use is a volatile
// shared-memory load, so the compiler cannot keep the ~30 loop-invariant
// setup values (cameras, config, pointers) in registers across the pixel
// loop; the LDS latency is short and the registers go to occupancy.
template <bool kLean>
struct SetupRead {
  template <typename T>
  __device__ __forceinline__ static T get(const T& x) { return x; }
};
template <>
struct SetupRead<true> {
  __device__ __forceinline__ static double get(const double& x) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(&x)));
    return v;
  }
  __device__ __forceinline__ static int get(const int& x) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(&x)));
    return v;
  }
  template <typename T>
  __device__ __forceinline__ static T* get(T* const& x) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"((unsigned)__cvta_generic_to_shared(&x)));
    return reinterpret_cast<T*>(v);
  }
};
#define SV(x) (SetupRead<kLean>::get(x))

// A 16-byte-aligned double pair / 8-byte-aligned int pair of the setup as one
// volatile shared load (kLean).
__device__ __forceinline__ double2 setup_pair(const double* p) {
  double2 v;
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
template <bool kLean>
__device__ __forceinline__ double2 pair_rd(const double* p) {
  if constexpr (kLean) return setup_pair(p);
  return make_double2(p[0], p[1]);
}
__device__ __forceinline__ int2 setup_pair(const int* p);
template <bool kLean>
__device__ __forceinline__ int2 pair_rd(const int* p) {
  if constexpr (kLean) return setup_pair(p);
  return make_int2(p[0], p[1]);
}
#define SP(f) (pair_rd<kLean>(S.f))
__device__ __forceinline__ int4 setup_quad(const int* p) {
  int4 v;
  asm volatile("ld.volatile.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ void setup_ptrs(const void* const* p, const double2*& a, const double*& b) {
  unsigned long long x, y;
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];"
               : "=l"(x), "=l"(y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  a = reinterpret_cast<const double2*>(x);
  b = reinterpret_cast<const double*>(y);
}
__device__ __forceinline__ int2 setup_pair(const int* p) {
  int2 v;
  asm volatile("ld.volatile.shared.v2.s32 {%0, %1}, [%2];"
               : "=r"(v.x), "=r"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

struct Row4 {
  double2 a, b;  // (r0, r1), (r2, extra)
};
// One 4-double row of the setup (16-byte aligned) as two volatile 16-byte
// shared loads.
__device__ __forceinline__ Row4 setup_row(const double* p) {
  Row4 r;
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.a.x), "=d"(r.a.y) : "r"(a));
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.b.x), "=d"(r.b.y) : "r"(a + 16));
  return r;
}

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
  for (int k = 0; k < 3; ++k) {
    double gt = 0.0;  // (R_j^T dt)_k - t_o,k
    for (int m = 0; m < 3; ++m) gt += S.Rj[3 * m + k] * S.dt[m];
    tmp[k] = gt - S.to[k];
  }
  for (int k = 0; k < 3; ++k)
    S.cpb[k] = S.Ro[k] * tmp[0] + S.Ro[3 + k] * tmp[1] + S.Ro[6 + k] * tmp[2];
  for (int k = 0; k < 3; ++k) {
    for (int c = 0; c < 3; ++c) {
      S.RoT[4 * k + c] = S.Ro[3 * k + c];
      S.MiC[4 * k + c] = S.Mi[3 * k + c];
      S.Rn[4 * k + c] = S.rotn[3 * k + c];
    }
    S.RoT[4 * k + 3] = S.to[k];
    S.MiC[4 * k + 3] = S.cpb[k];
    S.Rn[4 * k + 3] = 0.0;
  }
  S.occ_tol = P.occ_tol;
  const pba_frame& fs = frames[P.src];
  const pba_frame& fd = frames[P.dst];
  S.src_tex = static_cast<const double2*>(fs.texels);
  S.src_np = fs.cam.width * fs.cam.height;
  S.dst_np = fd.cam.width * fd.cam.height;
  S.src_mask = fs.mask;
  S.src_ray = fs.ray_table;
  S.dst_tex = static_cast<const double2*>(fd.texels);
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
  // |a| < 2w (always, for an azimuth in [-pi, pi] with the usual cx, fx):
  // fmod is exact there, so this equals the general path bit for bit.
  if (a >= 0.0 && a < w) return a;
  if (a >= w && a < 2.0 * w) return a - w;
  if (a < 0.0 && a > -w) return a + w;
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

// Move a (row, col) position of the strided source grid forward by `step`
// pixels in row-major order (replaces a per-pixel integer division).
__device__ __forceinline__ void advance_pixel(int& row, int& col, int width, int step) {
  col += step;
  while (col >= width) {
    col -= width;
    ++row;
  }
}

__device__ __forceinline__ uint32_t mask_word(const double2& v) {
  return (uint32_t)(__double_as_longlong(v.y) & 0xffffffffu);
}

__device__ __forceinline__ int upper_idx(int k, int l) { return k * 6 - (k * (k - 1)) / 2 + (l - k); }

// A 16-byte read-only load kept in program order with the other volatile
// asm (kLean's channel-by-channel gradient gathers).
__device__ __forceinline__ double2 ldg2_ordered(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Bilinear interpolation of a (d/dcol, d/drow) gradient pair with corner weights.
__device__ __forceinline__ double2 bil4(double2 g00, double2 g01, double2 g10, double2 g11,
                                        double w00, double w01, double w10, double w11) {
  double2 r;
  r.x = fma(w11, g11.x, fma(w10, g10.x, fma(w01, g01.x, w00 * g00.x)));
  r.y = fma(w11, g11.y, fma(w10, g10.y, fma(w01, g01.y, w00 * g00.y)));
  return r;
}

// One cue channel's contribution in the q-basis (see the file header):
//   q = [u; u x p_u (+ xn)],  u = -(g . P) M_i (+ extra_u),
//   Q += ww q q^T,  beta += q ww e.
__device__ __forceinline__ void accumulate_channel(double* Q, double* beta, double2 g,
                                                   const double* MP0, const double* MP1,
                                                   const double* extra_u, const double* pu,
                                                   const double* xn, double ww, double ec) {
  double q[6];
#pragma unroll
  for (int k = 0; k < 3; ++k) q[k] = -(g.x * MP0[k] + g.y * MP1[k]);
  if (extra_u) {
#pragma unroll
    for (int k = 0; k < 3; ++k) q[k] += extra_u[k];
  }
  cross3(q, pu, &q[3]);
  if (xn) {
    q[3] += xn[0];
    q[4] += xn[1];
    q[5] += xn[2];
  }
  const double we = ww * ec;
  double a[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    a[k] = ww * q[k];
    beta[k] = fma(q[k], we, beta[k]);
  }
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int l = k; l < 6; ++l) Q[upper_idx(k, l)] = fma(a[k], q[l], Q[upper_idx(k, l)]);
}

// ablation (diagnostics only): fold the channel into 7 sums instead of 27
__device__ __forceinline__ void accumulate_cheap(double* Q, double* beta, double2 g,
                                                 const double* MP0, const double* MP1,
                                                 double ww, double ec) {
#pragma unroll
  for (int k = 0; k < 3; ++k) Q[k] = fma(ww, g.x * MP0[k] + g.y * MP1[k], Q[k]);
  beta[0] = fma(ww, ec, beta[0]);
}

// The chunk's per-thread sums -> one 32-double partial, in a fixed order.
template <int kWarps, bool kJac>
__device__ __forceinline__ void store_chunk_partial(const double* Q, const double* beta,
                                                    double cost, int count,
                                                    double (*red)[kPart], int pair, int first,
                                                    int chunk_px,
                                                    const int32_t* __restrict__ pair_chunk_offsets,
                                                    double* __restrict__ partials) {
  // ---- fixed-order reduction: warp reduce-scatter, then warps in order ----
  // The 32 partial values (Q 21, beta 6, cost, count, 3 zero pads) are
  // halved over lanes five times: at offset o a lane keeps the half of its
  // values selected by its lane bit o and adds the partner's copy of that
  // half, so after 16+8+4+2+1 = 31 shuffles lane L holds the warp sum of
  // value L (a butterfly per value would take 29 x 5 = 145).
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v[kPart];
#pragma unroll
  for (int k = 0; k < kQ; ++k) v[k] = kJac ? Q[k] : 0.0;
#pragma unroll
  for (int k = 0; k < 6; ++k) v[kQ + k] = kJac ? beta[k] : 0.0;
  v[27] = cost;
  v[28] = (double)count;
  v[29] = v[30] = v[31] = 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < o; ++k) {
      const double send = upper ? v[k] : v[k + o];
      const double keep = upper ? v[k + o] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  red[warp][lane] = v[0];
  __syncthreads();
  if (threadIdx.x < kPart) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += red[w][threadIdx.x];
    // slot of this chunk in its pair's range (the launch order of the chunk
    // table is free; the per-pair sums always run in chunk order)
    const long slot = PBA_DCHECK_INDEX(pair_chunk_offsets[pair] + first / chunk_px,
                                       pair_chunk_offsets[pair + 1]);
    partials[slot * kPart + threadIdx.x] = s;
  }
}

// Everything a CTA of pair P needs that does not depend on the pixel: the
// pair's geometry (build_setup) plus the paired / grouped copies the lean
// loop reads with 16-byte shared loads.
__device__ void fill_setup(PairSetup& S, const pba_frame* frames, const pba_pair& P,
                           const double* poses, const double* exts, const pba_config& cfg) {
  build_setup(S, frames, P, poses, exts, cfg.pixel_stride);
  S.cfg = cfg;
  S.sqw0 = sqrt(cfg.omega[0]);
  S.sqw1 = sqrt(cfg.omega[1]);
  const pba_camera& dc = S.dst_cam;
  S.fx_cx[0] = dc.fx, S.fx_cx[1] = dc.cx, S.fy_cy[0] = dc.fy, S.fy_cy[1] = dc.cy;
  S.fx_fy[0] = dc.fx, S.fx_fy[1] = dc.fy;
  S.range[0] = dc.depth_min, S.range[1] = dc.depth_max;
  S.wh[0] = (double)dc.width, S.wh[1] = (double)dc.height;
  S.sqw0_dI[0] = S.sqw0, S.sqw0_dI[1] = cfg.huber_delta[0];
  S.sqw1_dD[0] = S.sqw1, S.sqw1_dD[1] = cfg.huber_delta[1];
  S.om01[0] = cfg.omega[0], S.om01[1] = cfg.omega[1];
  S.om23[0] = cfg.omega[2], S.om23[1] = cfg.omega[3];
  S.om4_dN[0] = cfg.omega[4], S.om4_dN[1] = cfg.huber_delta[2];
  S.dwh[0] = dc.width, S.dwh[1] = dc.height;
  S.np_sd[0] = S.src_np, S.np_sd[1] = S.dst_np;
  S.src_geo[0] = S.stride, S.src_geo[1] = S.src_cam.width, S.src_geo[2] = S.src_np;
  S.src_geo[3] = S.grid_w;
  S.src_mh[0] = S.src_cam.model, S.src_mh[1] = S.src_cam.height;
  S.src_ptrs[0] = S.src_tex, S.src_ptrs[1] = S.src_ray;
}

// One thread per pair: the setup every CTA of the pair copies (so no CTA
// spends its start on one thread's serial matrix products).
__global__ void pair_setup_kernel(const pba_frame* __restrict__ frames,
                                  const pba_pair* __restrict__ pairs, int n_pairs,
                                  const double* __restrict__ poses,
                                  const double* __restrict__ exts, pba_config cfg,
                                  PairSetup* __restrict__ setups) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n_pairs) fill_setup(setups[p], frames, pairs[p], poses, exts, cfg);
}

// kProbe 13 (diagnostics only): per-thread clock64 section timing, summed
// into g_sect_cycles / g_sect_count (read by pba_diag_section_cycles).
__device__ unsigned long long g_sect_cycles[8];
__device__ unsigned long long g_sect_count[8];

// kProbe (diagnostics only, K1 ablations): 0 normal; 1 every
// sample reads one fixed destination texel; 10 no gradient gathers; 11 a
// 7-sum stand-in for the 27-sum accumulation.
template <bool kJac, int kT, int kMinBlocks, int kProbe = 0, bool kLean = false,
          bool kTile = kLean, int kPf = 0>
__global__ void __launch_bounds__(kT, kMinBlocks)
    linearize_kernel(const PairSetup* __restrict__ setups, const int32_t* __restrict__ chunk_table,
                     const int32_t* __restrict__ pair_chunk_offsets, int chunk_pixels,
                     double* __restrict__ partials) {
  __shared__ PairSetup S;
  constexpr int kWarps = kT / 32;
  __shared__ double red[kWarps][kPart];

  const long chunk = blockIdx.x;
  const int pair = chunk_table[2 * chunk];
  const int first = chunk_table[2 * chunk + 1];
  {  // the pair's setup, formed once per pair by pair_setup_kernel: a coalesced copy
    static_assert(sizeof(PairSetup) % 16 == 0, "PairSetup is copied in 16-byte words");
    const int4* src = reinterpret_cast<const int4*>(setups + pair);
    int4* dst = reinterpret_cast<int4*>(&S);
    for (int i = threadIdx.x; i < (int)(sizeof(PairSetup) / 16); i += kT) dst[i] = __ldg(src + i);
  }
  __syncthreads();

  double Q[kQ];
#pragma unroll
  for (int k = 0; k < kQ; ++k) Q[k] = 0.0;
  double beta[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) beta[k] = 0.0;
  double cost = 0.0;
  int count = 0;

  const int chunk_px = pair_chunk_pixels(S.grid_w, chunk_pixels);
  const int last = min(first + chunk_px, S.n_px);
  const int sW = S.src_cam.width;

  const int gw = S.grid_w;
  const int stride = S.stride;
  int gr = (first + (int)threadIdx.x) / gw;       // strided-grid row / column of
  int gcol = first + (int)threadIdx.x - gr * gw;  // this thread's current pixel
  // kTile: a chunk of whole 8-row bands (pair_chunk_pixels) is walked in
  // 16-column x 8-row tiles — warp w covers rows 2w, 2w + 1 of the band —
  // so the CTA's four warps sample overlapping destination rows at the same
  // time and each destination row is fetched from L2 about once per band
  // instead of twice (row-major walk: once as the lower corner row of source
  // row r, again as the upper one of row r + 1, a full row later).  Other
  // chunks keep the row-major walk.  Same pixel set, same partial slot.
  __shared__ int walk[2];  // column step, rows per wrap
  if constexpr (kTile) {
    static_assert(kT == kTileCols * kTileRows, "the tiled walk assumes 128-thread CTAs");
    const int n = last - first;
    const bool tiled = first % gw == 0 && n % gw == 0 && (n / gw) % kTileRows == 0 &&
                       gw % kTileCols == 0;
    if (tiled) {
      gr = first / gw + (int)threadIdx.x / kTileCols;
      gcol = (int)threadIdx.x % kTileCols;
    }
    if (threadIdx.x == 0) {
      walk[0] = tiled ? kTileCols : kT;
      walk[1] = tiled ? kTileRows : 1;
    }
    __syncthreads();
  }
  // The source texel of the next pixel is always in flight one iteration
  // ahead: its (I, D) and (nz, mask) pairs, 2 x 16 B.  Masks come from the
  // texel planes themselves (not the separate mask plane), so a pixel costs
  // two dependent round trips (source texel, destination texels), not four.
  double2 nx0 = make_double2(0.0, 0.0), nx2 = make_double2(0.0, 0.0);
  if (first + (int)threadIdx.x < last) {
    const double2* t = S.src_tex + PBA_DCHECK_INDEX(gr * stride * sW + gcol * stride, S.src_np);
    nx0 = __ldg(t);
    nx2 = __ldg(t + kPairNzM * S.src_np);
  }
  int ngr = gr, ngcol = gcol;
  constexpr bool kTime = kProbe == 13;
  long long sect[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int sect_n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t_prev = kTime ? clock64() : 0;
#define PBA_SECT(k)                          \
  if (kTime) {                               \
    const long long t_now = clock64();       \
    sect[k] += t_now - t_prev;               \
    ++sect_n[k];                             \
    t_prev = t_now;                          \
  }
  for (int idx = first + (int)threadIdx.x; idx < last; idx += kT, gr = ngr, gcol = ngcol) {
    PBA_SECT(7)  // tail of the previous iteration (rejected pixels: their last section)
    // source geometry: stride, width, plane size, grid width (kLean: one 16-byte load)
    const int4 sg = kLean ? setup_quad(S.src_geo)
                          : make_int4(S.stride, S.src_cam.width, S.src_np, S.grid_w);
    const int row = gr * sg.x;
    const int col = gcol * sg.x;
    const int sp = row * sg.y + col;
    const double2* s_tex;
    const double* s_ray;
    if constexpr (kLean) {
      setup_ptrs(S.src_ptrs, s_tex, s_ray);
    } else {
      s_tex = S.src_tex;
      s_ray = S.src_ray;
    }
    // kLean: the source texel is loaded when its pixel starts (no prefetch:
    // the registers go to forming the projective Jacobian while the first
    // destination gather is in flight, kEarlyMP)
    constexpr bool kNoPrefetch = kLean;
    constexpr bool kEarlyMP = kLean;
    if constexpr (kNoPrefetch) {
      const double2* t = s_tex + PBA_DCHECK_INDEX(sp, sg.z);
      nx0 = __ldg(t);
      nx2 = __ldg(t + kPairNzM * sg.z);
    }
    const double2 s_id = nx0;  // I, D
    const uint32_t sm = mask_word(nx2);
    const double mask_src_nz = nx2.x;

    ngr = gr;
    ngcol = gcol;
    if constexpr (kTile) {
      const int2 wk = setup_pair(walk);
      ngcol += wk.x;
      while (ngcol >= sg.w) {
        ngcol -= sg.w;
        ngr += wk.y;
      }
    } else {
      advance_pixel(ngr, ngcol, sg.w, kT);
    }
    if (!kNoPrefetch && idx + kT < last) {
      const double2* t = s_tex + PBA_DCHECK_INDEX(ngr * sg.x * sg.y + ngcol * sg.x, sg.z);
      nx0 = __ldg(t);
      nx2 = __ldg(t + kPairNzM * sg.z);
    }
    if (!(sm & PBA_MASK_DEPTH_VALID)) continue;  // PairContext.build: usable = depth_valid
    PBA_SECT(0)  // source texel + next-texel prefetch

    // ---- source cue values and unprojection (sensors.py:133-154) ----
    const double d = s_id.y;
    double ps[3];
    const int2 smh = kLean ? setup_pair(S.src_mh) : make_int2(S.src_cam.model, S.src_cam.height);
#ifdef PBA_CHECKED
    PBA_DCHECK_INDEX(col, sg.y);
    PBA_DCHECK_INDEX(row, smh.y);
#endif
    if (smh.x == PBA_SPHERICAL) {
      const double ca = __ldg(s_ray + col), sa = __ldg(s_ray + sg.y + col);
      const double ce = __ldg(s_ray + 2 * sg.y + row), se = __ldg(s_ray + 2 * sg.y + smh.y + row);
      ps[0] = (ce * ca) * d;
      ps[1] = (ce * sa) * d;
      ps[2] = se * d;
    } else {
      ps[0] = __ldg(s_ray + col) * d;
      ps[1] = __ldg(s_ray + 2 * sg.y + row) * d;
      ps[2] = d;
    }
    // p_u = R_o p + t_o (solver.py:215)
    double pu[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if constexpr (kLean) {
        const Row4 r = setup_row(&S.RoT[4 * k]);
        pu[k] = r.a.x * ps[0] + r.a.y * ps[1] + r.b.x * ps[2] + r.b.y;
      } else {
        pu[k] = S.Ro[3 * k + 0] * ps[0] + S.Ro[3 * k + 1] * ps[1] + S.Ro[3 * k + 2] * ps[2] + S.to[k];
      }
    // p_bar = R_o^T (R_j^T (R_i p_u + t_i - t_j) - t_o) = M_i p_u + cpb  (solver.py:235-236)
    double pb[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if constexpr (kLean) {
        const Row4 r = setup_row(&S.MiC[4 * k]);
        pb[k] = r.a.x * pu[0] + r.a.y * pu[1] + r.b.x * pu[2] + r.b.y;
      } else {
        pb[k] = S.Mi[3 * k + 0] * pu[0] + S.Mi[3 * k + 1] * pu[1] + S.Mi[3 * k + 2] * pu[2] + S.cpb[k];
      }

    // ---- project into the destination (sensors.py:95-130) ----
    // Two independent rsqrt give rho = hypot(x, y), the range and every
    // reciprocal needed below (inv = 1/rho, 1/range; pinhole: 1/z).
    double u, v, dist, rho = 0.0, inv_rho = 0.0, inv_dist;
    const bool dsph = SV(S.dst_cam.model) == PBA_SPHERICAL;
    if (dsph) {
      // The reference's roundings are reproduced where they decide validity:
      // range = sqrt((x^2 + y^2) + z^2) with separately rounded terms
      // (np.linalg.norm), hypot(x, y) correctly rounded (np.hypot), and
      // u = fx * az + cx as a multiply then an add (no FMA contraction).
      // Integer-pixel self-projections make floor(u) sensitive to the last bit.
      const double xx = __dmul_rn(pb[0], pb[0]), yy = __dmul_rn(pb[1], pb[1]);
      const double rr = __dadd_rn(xx, yy);
      const double r2 = __dadd_rn(rr, __dmul_rn(pb[2], pb[2]));
      dist = __dsqrt_rn(r2);
      {
        const double2 rg = SP(range);
        if (!(dist >= rg.x && dist <= rg.y)) continue;
      }
      inv_dist = rsqrt(r2);
      double az;
      if (rr > 1e-60) {
        inv_rho = rsqrt(rr);
        // hypot: sqrt of the exact x^2 + y^2 (double-double) with one Newton
        // correction from the rsqrt estimate -> correctly rounded (almost always)
        const double bb = rr - xx;
        const double sum_err = (xx - (rr - bb)) + (yy - bb);  // two_sum(xx, yy) error
        const double tail = fma(pb[0], pb[0], -xx) + fma(pb[1], pb[1], -yy) + sum_err;
        const double r0 = rr * inv_rho;
        rho = fma(fma(-r0, r0, rr) + tail, 0.5 * inv_rho, r0);
        az = atan2_tab_r(pb[1], pb[0], inv_rho);
      } else {  // (practically) on the polar axis: library path, atan2's zero semantics
        rho = hypot(pb[0], pb[1]);
        inv_rho = rr > 0.0 ? 1.0 / rho : 0.0;
        az = atan2(pb[1], pb[0]);
      }
      const double el = atan2_tab_r(pb[2], rho, inv_dist);
      const double2 fc = SP(fx_cx), fyc = SP(fy_cy);
      u = py_mod(__dadd_rn(__dmul_rn(fc.x, az), fc.y), SP(wh).x);
      v = __dadd_rn(__dmul_rn(fyc.x, el), fyc.y);
    } else {
      {  // z > 0 and the depth range (sensors.py:112-113, 125) before the divisions
        const double2 rg = SP(range);
        if (!(pb[2] > 0.0 && pb[2] >= rg.x && pb[2] <= rg.y)) continue;
      }
      // u, v with true IEEE division and separate roundings, exactly as the
      // reference (sensors.py:114-115): self-projections land on integer
      // pixels where a last-bit difference would move floor() and flip validity.
      const double2 fc = SP(fx_cx), fyc = SP(fy_cy);
      u = __dadd_rn(__ddiv_rn(__dmul_rn(fc.x, pb[0]), pb[2]), fc.y);
      v = __dadd_rn(__ddiv_rn(__dmul_rn(fyc.x, pb[1]), pb[2]), fyc.y);
      inv_dist = __drcp_rn(pb[2]);  // Jacobian only
      dist = pb[2];
    }
    // (the depth range was checked in each model's branch)
    // project's bounds 0 <= u < W, 0 <= v < H (sensors.py:126-127) and
    // sample's inside test u <= W - 1, v <= H - 1 (cues.py:400) in one test:
    // u <= W - 1 implies u < W
    const double2 whd = SP(wh);
    if (!(u >= 0.0 && v >= 0.0 && u <= whd.x - 1.0 && v <= whd.y - 1.0)) continue;

    PBA_SECT(1)  // unprojection + warp + projection
    // ---- bilinear footprint (cues.py:397-409, 451-456) ----
    const int2 dwh = SP(dwh);
    int x0 = (int)floor(u), y0 = (int)floor(v);
    x0 = min(max(x0, 0), dwh.x - 2);
    y0 = min(max(y0, 0), dwh.y - 2);
    const double wx = u - x0, wy = v - y0;
    // kProbe 1 (diagnostics only): every sample reads the same texel block
    const int dnp = SV(S.dst_np);
    // the four corners dp, dp + 1, dp + W, dp + W + 1 lie in the plane
    const int dp = PBA_DCHECK_INDEX(kProbe == 1 ? (dwh.y / 2) * dwh.x + dwh.x / 2 : y0 * dwh.x + x0,
                                    dnp - dwh.x - 1);
    const double2* t00 = SV(S.dst_tex) + dp;  // pair k of corner (r, c): t00[k * dnp + r * W + c]
    const double2* t10 = t00 + dwh.x;
    // (I, D) and (nz, mask) of the four corners in one round trip
    const double2 a00 = __ldg(t00), a01 = __ldg(t00 + 1), a10 = __ldg(t10), a11 = __ldg(t10 + 1);
    const double2 m00 = __ldg(t00 + kPairNzM * dnp), m01 = __ldg(t00 + kPairNzM * dnp + 1);
    const double2 m10 = __ldg(t10 + kPairNzM * dnp), m11 = __ldg(t10 + kPairNzM * dnp + 1);
    if constexpr (kPf > 0) {
      // Pinhole destinations (PBA_CFG_PINHOLE_DST launches): L1 prefetch of
      // the footprint this thread's next pixel (one tile, 16 source columns,
      // to the right) most likely samples, all eight texel planes.  c3/100:
      // 15.84 -> 15.44 ms; on the spherical scans the same prefetch was
      // slower (27.40 -> 28.35 ms c4/200), so it is skipped for them, and
      // launches without pinhole destinations use the kPf = 0 kernel (the
      // prefetch costs registers).
      if (x0 + kTileCols + 1 < dwh.x && !dsph) {
        constexpr int order[8] = {0, kPairNzM, kPairGI, kPairGI + 1, kPairNxy, 5, 6, 7};
#pragma unroll
        for (int k = 0; k < kPf; ++k) {
          const double2* p = t00 + kTileCols + order[k] * dnp;
          asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(p + dwh.x));
        }
      }
    }
    double MP0[3], MP1[3], ud[3];
    double rho2 = 0.0;
    if constexpr (kEarlyMP && kJac) {
      if (dsph) rho2 = pb[0] * pb[0] + pb[1] * pb[1];
      // ---- projective Jacobian folded with M_i (sensors.py:157-188) ----
      // (kEarlyMP: formed while the corner loads are in flight)
      // MP0 = M_i^T P[0,:], MP1 = M_i^T P[1,:], ud = M_i^T (depth-cue direction)
      const Row4 q0 = setup_row(&S.MiC[0]), q1 = setup_row(&S.MiC[4]), q2 = setup_row(&S.MiC[8]);
      const double Mr[9] = {q0.a.x, q0.a.y, q0.b.x, q1.a.x, q1.a.y, q1.b.x, q2.a.x, q2.a.y, q2.b.x};
      const double2 ff = SP(fx_fy);
      if (dsph) {
        const double iz = inv_dist;  // 1/|p_bar| = 1/zeta
        const double f0 = ff.x * (inv_rho * inv_rho);         // fx / rho^2
        const double f1 = ff.y * (inv_rho * (iz * iz));       // fy / (rho r^2)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double m0 = Mr[k], m1 = Mr[3 + k], m2 = Mr[6 + k];
          MP0[k] = f0 * (pb[0] * m1 - pb[1] * m0);
          MP1[k] = f1 * (rho2 * m2 - pb[2] * (pb[0] * m0 + pb[1] * m1));
          ud[k] = iz * (pb[0] * m0 + pb[1] * m1 + pb[2] * m2);
        }
      } else {
        const double iz = inv_dist;  // 1/z
        const double f0 = ff.x * iz, f1 = ff.y * iz;
        const double xz = pb[0] * iz, yz = pb[1] * iz;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double m2 = Mr[6 + k];
          MP0[k] = f0 * (Mr[k] - xz * m2);
          MP1[k] = f1 * (Mr[3 + k] - yz * m2);
          ud[k] = m2;
        }
      }
    }
    const uint32_t mk = mask_word(m00) & mask_word(m01) & mask_word(m10) & mask_word(m11);
    if (!(mk & PBA_MASK_SAMP_CORE)) continue;  // core_ok
    const double Dd = bil(a00.y, a01.y, a10.y, a11.y, wx, wy);
    // zeta_d: range for spherical, z for pinhole (solver.py:240)
    const double zeta = dsph ? dist : pb[2];
    const double e1 = zeta - Dd;
    if constexpr (!kEarlyMP) {
      if (kJac && dsph) rho2 = pb[0] * pb[0] + pb[1] * pb[1];
    }
    // occluded (solver.py:254-258), or no Jacobian (ok_jac, sensors.py:173-175,
    // solver.py:262-263; the Jacobian path only)
    if (e1 > SV(S.occ_tol) || (kJac && dsph && !(rho2 > 0.0))) continue;
    const double e0 = s_id.x - bil(a00.x, a01.x, a10.x, a11.x, wx, wy);

    PBA_SECT(2)  // footprint, first destination gather, masks, occlusion
    const bool normal_on = (mk & PBA_MASK_SAMP_NORMAL) && (sm & PBA_MASK_NORMAL_VALID);
    double e2 = 0.0, e3 = 0.0, e4 = 0.0;
    double no[3] = {0.0, 0.0, 0.0};  // R_o n_src
    if (normal_on) {
      const double2 s_n01 = __ldg(s_tex + kPairNxy * sg.z + sp);  // source nx, ny
      const double ns2 = mask_src_nz;
      const double2 b00 = __ldg(t00 + kPairNxy * dnp), b01 = __ldg(t00 + kPairNxy * dnp + 1);
      const double2 b10 = __ldg(t10 + kPairNxy * dnp), b11 = __ldg(t10 + kPairNxy * dnp + 1);
      // rot_n n_src (solver.py:241-248)
      double m0, m1, m2;
      if constexpr (kLean) {
        const Row4 r0 = setup_row(&S.Rn[0]), r1 = setup_row(&S.Rn[4]), r2 = setup_row(&S.Rn[8]);
        m0 = s_n01.x * r0.a.x + s_n01.y * r0.a.y + ns2 * r0.b.x;
        m1 = s_n01.x * r1.a.x + s_n01.y * r1.a.y + ns2 * r1.b.x;
        m2 = s_n01.x * r2.a.x + s_n01.y * r2.a.y + ns2 * r2.b.x;
      } else {
        m0 = s_n01.x * S.rotn[0] + s_n01.y * S.rotn[1] + ns2 * S.rotn[2];
        m1 = s_n01.x * S.rotn[3] + s_n01.y * S.rotn[4] + ns2 * S.rotn[5];
        m2 = s_n01.x * S.rotn[6] + s_n01.y * S.rotn[7] + ns2 * S.rotn[8];
      }
      e2 = m0 - bil(b00.x, b01.x, b10.x, b11.x, wx, wy);
      e3 = m1 - bil(b00.y, b01.y, b10.y, b11.y, wx, wy);
      e4 = m2 - bil(m00.x, m01.x, m10.x, m11.x, wx, wy);
      if (kJac) {
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if constexpr (kLean) {
            const Row4 r = setup_row(&S.RoT[4 * k]);
            no[k] = r.a.x * s_n01.x + r.a.y * s_n01.y + r.b.x * ns2;
          } else {
            no[k] = S.Ro[3 * k + 0] * s_n01.x + S.Ro[3 * k + 1] * s_n01.y + S.Ro[3 * k + 2] * ns2;
          }
      }
    }

    // ---- per-cue Huber (solver.py:317-337) ----
    // Fast norms (|e| sqrt(w); t * rsqrt(t)) are within a few ulp of the
    // reference's sqrt((e*e)*w) / sqrt(((e2 + e3) + e4)); the "small"
    // decision s <= delta is re-taken with the reference's exact roundings
    // whenever a fast norm lies within 1e-14 relative of its threshold.
    const double2 hI = SP(sqw0_dI), hD = SP(sqw1_dD), o23 = SP(om23), o4 = SP(om4_dN);
    double sI = fabs(e0) * hI.x;
    double sD = fabs(e1) * hD.x;
    const double tN = (e2 * e2 * o23.x + e3 * e3 * o23.y) + e4 * e4 * o4.x;
    const double inv_sN = tN > 1e-300 ? rsqrt(tN) : 0.0;
    double sN = tN > 1e-300 ? tN * inv_sN : sqrt(tN);
    const double dI = hI.y, dD = hD.y, dN = o4.y;
    const bool nearI = fabs(sI - dI) <= 1e-14 * dI, nearD = fabs(sD - dD) <= 1e-14 * dD;
    const bool nearN = fabs(sN - dN) <= 1e-14 * dN;
    if (nearI || nearD || nearN) {  // rare: one branch for the three exact re-takes
      const double2 o01x = SP(om01);
      if (nearI) sI = __dsqrt_rn(__dmul_rn(__dmul_rn(e0, e0), o01x.x));
      if (nearD) sD = __dsqrt_rn(__dmul_rn(__dmul_rn(e1, e1), o01x.y));
      if (nearN)
        sN = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(e2, e2), o23.x),
                                            __dmul_rn(__dmul_rn(e3, e3), o23.y)),
                                  __dmul_rn(__dmul_rn(e4, e4), o4.x)));
    }
    const bool smI = sI <= dI, smD = sD <= dD, smN = sN <= dN;
    cost += (smI ? sI * sI : dI * (2.0 * sI - dI)) + (smD ? sD * sD : dD * (2.0 * sD - dD)) +
            (smN ? sN * sN : dN * (2.0 * sN - dN));
    ++count;
    PBA_SECT(3)  // normal gather, residuals, Huber, cost
    if (!kJac) continue;

    // ---- projective Jacobian folded with M_i (sensors.py:157-188) ----
    // MP0 = M_i^T P[0,:], MP1 = M_i^T P[1,:], ud = M_i^T (depth-cue direction)
    if constexpr (!kEarlyMP) {
    if (dsph) {
      const double iz = inv_dist;  // 1/|p_bar| = 1/zeta
      const double f0 = SV(S.dst_cam.fx) * (inv_rho * inv_rho);         // fx / rho^2
      const double f1 = SV(S.dst_cam.fy) * (inv_rho * (iz * iz));       // fy / (rho r^2)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double m0 = SV(S.Mi[k]), m1 = SV(S.Mi[3 + k]), m2 = SV(S.Mi[6 + k]);
        MP0[k] = f0 * (pb[0] * m1 - pb[1] * m0);
        MP1[k] = f1 * (rho2 * m2 - pb[2] * (pb[0] * m0 + pb[1] * m1));
        ud[k] = iz * (pb[0] * m0 + pb[1] * m1 + pb[2] * m2);
      }
    } else {
      const double iz = inv_dist;  // 1/z
      const double f0 = SV(S.dst_cam.fx) * iz, f1 = SV(S.dst_cam.fy) * iz;
      const double xz = pb[0] * iz, yz = pb[1] * iz;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double m2 = SV(S.Mi[6 + k]);
        MP0[k] = f0 * (SV(S.Mi[k]) - xz * m2);
        MP1[k] = f1 * (SV(S.Mi[3 + k]) - yz * m2);
        ud[k] = m2;
      }
    }
    }
    const double2 o01 = SP(om01);
    const double wI = smI ? o01.x : o01.x * (dI * __drcp_rn(sI));
    const double wD = smD ? o01.y : o01.y * (dD * __drcp_rn(sD));
    const double wN = smN ? 1.0 : dN * inv_sN;
    // Gradients of the four corners, fetched in two batches (the lines are in
    // L1 after the value loads) and interpolated with the corner weights;
    // the gradient images are interpolated, not differentiated (cues.py:448-450).
    const double w00 = (1.0 - wx) * (1.0 - wy), w01 = wx * (1.0 - wy);
    const double w10 = (1.0 - wx) * wy, w11 = wx * wy;
    const double2* g00p = t00 + kPairGI * dnp;  // gradient pair k at g..p + k * dnp
    const double2* g01p = g00p + 1;
    const double2* g10p = g00p + dwh.x;
    const double2* g11p = g10p + 1;
    if constexpr (kLean) {
      // Channel by channel: the four corner loads of one gradient plane are
      // issued (volatile, so not hoisted together) only when that channel is
      // accumulated — fewer load destinations live at once, traded for
      // latency that the extra resident warps cover.
      // One plane of look-ahead: the next channel's four corners are in
      // flight while the current channel accumulates.
      struct Corners {
        double2 c00, c01, c10, c11;
      };
      auto load_plane = [&](int plane) {
        const double2* p0 = g00p + plane * dnp;
        const double2* p1 = g10p + plane * dnp;
        return Corners{ldg2_ordered(p0), ldg2_ordered(p0 + 1), ldg2_ordered(p1),
                       ldg2_ordered(p1 + 1)};
      };
      auto interp = [&](const Corners& c) { return bil4(c.c00, c.c01, c.c10, c.c11, w00, w01, w10, w11); };
      Corners cur = load_plane(0);
      Corners nxt = load_plane(1);
      accumulate_channel(Q, beta, interp(cur), MP0, MP1, nullptr, pu, nullptr, wI, e0);
      cur = nxt;
      if (normal_on) nxt = load_plane(2);
      accumulate_channel(Q, beta, interp(cur), MP0, MP1, ud, pu, nullptr, wD, e1);
      if (normal_on) {
        double xn[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          cur = nxt;
          if (k < 2) nxt = load_plane(3 + k);
          const Row4 r = setup_row(&S.MiC[4 * k]);
          const double mr[3] = {r.a.x, r.a.y, r.b.x};
          cross3(mr, no, xn);
          accumulate_channel(Q, beta, interp(cur), MP0, MP1, nullptr, pu, xn,
                             wN * (k == 0 ? o23.x : (k == 1 ? o23.y : o4.x)),
                             k == 0 ? e2 : (k == 1 ? e3 : e4));
        }
      }
    } else {
      double2 gI, gD;
      if (kProbe == 10) {  // ablation (diagnostics only): no gradient loads
        gI = make_double2(a00.x * w00, a01.x * w01);
        gD = make_double2(a10.y * w10, a11.y * w11);
      } else {
        const double2 i00 = __ldg(g00p), i01 = __ldg(g01p), i10 = __ldg(g10p), i11 = __ldg(g11p);
        const double2 d00 = __ldg(g00p + dnp), d01 = __ldg(g01p + dnp), d10 = __ldg(g10p + dnp),
                      d11 = __ldg(g11p + dnp);
        gI = bil4(i00, i01, i10, i11, w00, w01, w10, w11);
        gD = bil4(d00, d01, d10, d11, w00, w01, w10, w11);
      }
      PBA_SECT(4)  // projective Jacobian, weights, I/D gradient gathers
      double* QA = Q;
      double* bA = beta;
      if (kProbe == 11) {
        accumulate_cheap(QA, bA, gI, MP0, MP1, wI, e0);
        accumulate_cheap(QA, bA, gD, MP0, MP1, wD, e1);
        if (normal_on) {
          accumulate_cheap(QA, bA, make_double2(no[0], no[1]), MP0, MP1, wN, e2 + e3 + e4);
        }
        continue;
      }
      accumulate_channel(QA, bA, gI, MP0, MP1, nullptr, pu, nullptr, wI, e0);
      accumulate_channel(QA, bA, gD, MP0, MP1, ud, pu, nullptr, wD, e1);
      if (normal_on) {
        double2 gN[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
          gN[k] = kProbe == 10 ? make_double2(gI.x * (k + 1), gD.y * k)
                               : bil4(__ldg(g00p + (2 + k) * dnp), __ldg(g01p + (2 + k) * dnp),
                                      __ldg(g10p + (2 + k) * dnp), __ldg(g11p + (2 + k) * dnp), w00,
                                      w01, w10, w11);
        double xn[3];
        {
          const double mr[3] = {SV(S.Mi[0]), SV(S.Mi[1]), SV(S.Mi[2])};
          cross3(mr, no, xn);
        }
        accumulate_channel(QA, bA, gN[0], MP0, MP1, nullptr, pu, xn, wN * SV(S.cfg.omega[2]), e2);
        {
          const double mr[3] = {SV(S.Mi[3]), SV(S.Mi[4]), SV(S.Mi[5])};
          cross3(mr, no, xn);
        }
        accumulate_channel(QA, bA, gN[1], MP0, MP1, nullptr, pu, xn, wN * SV(S.cfg.omega[3]), e3);
        {
          const double mr[3] = {SV(S.Mi[6]), SV(S.Mi[7]), SV(S.Mi[8])};
          cross3(mr, no, xn);
        }
        accumulate_channel(QA, bA, gN[2], MP0, MP1, nullptr, pu, xn, wN * SV(S.cfg.omega[4]), e4);
      }
    }
    PBA_SECT(5)  // q rows + accumulation (incl. normal-gradient gathers)
  }
  PBA_SECT(7)
#undef PBA_SECT
  if (kTime) {
    for (int k = 0; k < 8; ++k) {
      atomicAdd(&g_sect_cycles[k], (unsigned long long)sect[k]);
      atomicAdd(&g_sect_count[k], (unsigned long long)sect_n[k]);
    }
  }

  // (the chunk size re-derived from a fresh shared read: nothing stays live
  // across the pixel loop for it)
  store_chunk_partial<kWarps, kJac>(Q, beta, cost, count, red, pair, first,
                                    pair_chunk_pixels(SetupRead<true>::get(S.grid_w), chunk_pixels),
                                    pair_chunk_offsets, partials);
}

// One warp per pair: sum the pair's chunk partials in chunk order, then
// expand (Q, beta) into the reference _EdgeTerm blocks:
//   H_ii = D Q D, H_jj = L Q L^T, H_ij = D Q L^T, b_i = D beta, b_j = L beta.
__global__ void finalize_pairs_kernel(const double* __restrict__ partials,
                                      const int32_t* __restrict__ offsets,
                                      const pba_pair* __restrict__ pairs,
                                      const double* __restrict__ poses, int n_pairs,
                                      double* __restrict__ records) {
  __shared__ double sQ[4][kPart];
  __shared__ double sL[4][36];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * 4 + w;
  if (p >= n_pairs) return;
  const int c0 = offsets[p], c1 = offsets[p + 1];
  // chunk order, eight loads in flight at a time (same sums, same order)
  double s = 0.0;
  int c = c0;
  for (; c + 8 <= c1; c += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = partials[(long)(c + u) * kPart + lane];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; c < c1; ++c) s += partials[(long)c * kPart + lane];
  sQ[w][lane] = s;
  if (lane == 0) {
    const pba_pair P = pairs[p];
    const double* xi = poses + 12 * P.pose_i;
    const double* xj = poses + 12 * P.pose_j;
    double A[9], tg[3], dt[3];
    for (int k = 0; k < 3; ++k) dt[k] = xi[9 + k] - xj[9 + k];
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c)  // A = R_j^T R_i
        A[3 * r + c] = xj[r] * xi[c] + xj[3 + r] * xi[3 + c] + xj[6 + r] * xi[6 + c];
      tg[r] = xj[r] * dt[0] + xj[3 + r] * dt[1] + xj[6 + r] * dt[2];  // R_j^T (t_i - t_j)
    }
    double* L = sL[w];
    for (int k = 0; k < 36; ++k) L[k] = 0.0;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        L[6 * r + c] = -A[3 * r + c];
        L[6 * (3 + r) + 3 + c] = 2.0 * A[3 * r + c];
        // -2 [t_g]x A
        const double sk0 = (r == 0) ? 0.0 : (r == 1 ? tg[2] : -tg[1]);
        const double sk1 = (r == 0) ? -tg[2] : (r == 1 ? 0.0 : tg[0]);
        const double sk2 = (r == 0) ? tg[1] : (r == 1 ? -tg[0] : 0.0);
        L[6 * (3 + r) + c] = -2.0 * (sk0 * A[c] + sk1 * A[3 + c] + sk2 * A[6 + c]);
      }
  }
  __syncwarp();
  const double* q = sQ[w];
  const double* L = sL[w];
  auto Qf = [&](int a, int b) { return a <= b ? q[upper_idx(a, b)] : q[upper_idx(b, a)]; };
  const double dg[6] = {1.0, 1.0, 1.0, -2.0, -2.0, -2.0};
  double* rec = records + (long)p * kRec;
  const bool any = q[28] > 0.0;
  for (int e = lane; e < kRec; e += 32) {
    double val = 0.0;
    if (!any) {
      val = 0.0;
    } else if (e < PBA_REC_HJJ) {  // H_ii upper
      int k = 0, t = e;
      while (t >= 6 - k) { t -= 6 - k; ++k; }
      const int l = k + t;
      val = dg[k] * dg[l] * Qf(k, l);
    } else if (e < PBA_REC_HIJ) {  // H_jj upper
      int k = 0, t = e - PBA_REC_HJJ;
      while (t >= 6 - k) { t -= 6 - k; ++k; }
      const int l = k + t;
      for (int a = 0; a < 6; ++a) {
        if (L[6 * k + a] == 0.0) continue;
        double inner = 0.0;
        for (int b = 0; b < 6; ++b) inner += Qf(a, b) * L[6 * l + b];
        val += L[6 * k + a] * inner;
      }
    } else if (e < PBA_REC_BI) {  // H_ij full
      const int k = (e - PBA_REC_HIJ) / 6, l = (e - PBA_REC_HIJ) % 6;
      for (int b = 0; b < 6; ++b) val += Qf(k, b) * L[6 * l + b];
      val *= dg[k];
    } else if (e < PBA_REC_BJ) {
      const int k = e - PBA_REC_BI;
      val = dg[k] * q[kQ + k];
    } else if (e < PBA_REC_COST) {
      const int k = e - PBA_REC_BJ;
      for (int b = 0; b < 6; ++b) val += L[6 * k + b] * q[kQ + b];
    } else if (e == PBA_REC_COST) {
      val = q[27];
    } else {
      val = q[28];
    }
    rec[e] = val;
  }
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
    const int64_t cp = pair_chunk_pixels((int)gw, chunk_pixels);
    const int64_t nc = npx == 0 ? 0 : (npx + cp - 1) / cp;
    pairs[p].n_chunks = (int32_t)nc;
    if (pair_chunk_offsets) pair_chunk_offsets[p] = (int32_t)total;
    if (chunk_table) {
      for (int64_t k = 0; k < nc; ++k) {
        chunk_table[2 * (total + k)] = p;
        chunk_table[2 * (total + k) + 1] = (int32_t)(k * cp);
      }
    }
    total += nc;
  }
  PBA_ARG_CHECK(total < (int64_t)1 << 31, "too many chunks");
  if (pair_chunk_offsets) pair_chunk_offsets[n_pairs] = (int32_t)total;
  if (n_chunks_out) *n_chunks_out = total;
  return PBA_OK;
}

namespace {
size_t partials_bytes(int64_t n_chunks) {
  return ((size_t)n_chunks * kPart * sizeof(double) + 255) / 256 * 256;
}
}  // namespace

extern "C" size_t pba_linearize_scratch_bytes(int32_t n_pairs, int64_t n_chunks) {
  if (n_pairs < 0 || n_chunks < 0) return 0;
  return partials_bytes(n_chunks) + (size_t)n_pairs * sizeof(PairSetup);
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
  if (int rc = ensure_atan_table()) return rc;
  // scratch = [chunk partials | per-pair setups] (pba_linearize_scratch_bytes)
  PairSetup* setups = reinterpret_cast<PairSetup*>(reinterpret_cast<char*>(partials) +
                                                   partials_bytes(n_chunks));
  pair_setup_kernel<<<(unsigned)((n_pairs + 127) / 128), 128, 0, st>>>(frames, pairs, n_pairs,
                                                                      poses, extrinsics, *cfg,
                                                                      setups);
  PBA_LAUNCH_CHECK();
  if (n_chunks > 0) {
    // CTA-size / occupancy variant (PBA_LIN_VARIANT overrides):
    //   6 (default): lean, tiled walk, 128 thr, 168 regs (12 warps/SM)
    //   7: lean, row-major walk
    //   1: 256 thr, <=255 regs (8 warps/SM)    2: 256 thr, 128 regs (16 warps/SM)
    //   3: 128 thr, 128 regs (16 warps/SM)     4: round-1 kernel, 128 thr, 168 regs
    //   5: 512 thr, 128 regs (16 warps/SM)
    //   9 / 20 / 21: diagnostics (fixed destination texel / no gradient
    //   gathers / reduced accumulation), see kProbe
    static int variant = -1;
    if (variant < 0) {
      const char* env = getenv("PBA_LIN_VARIANT");
      variant = env ? atoi(env) : 6;
      if (variant < 1 || variant > 24) variant = 6;
    }
    const unsigned grid = (unsigned)n_chunks;
#define PBA_LAUNCH_LIN(J, T, M) \
  linearize_kernel<J, T, M><<<grid, T, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials)
#define PBA_LAUNCH_COST(M) \
  linearize_kernel<false, 128, M, 0, false, true><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials)
    if (want_jacobians) {
      switch (variant) {
        case 1: PBA_LAUNCH_LIN(true, 256, 1); break;
        case 3: PBA_LAUNCH_LIN(true, 128, 4); break;
        case 5: PBA_LAUNCH_LIN(true, 512, 1); break;
        case 2: PBA_LAUNCH_LIN(true, 256, 2); break;
        case 20:
          linearize_kernel<true, 128, 3, 10><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials);
          break;
        case 21:
          linearize_kernel<true, 128, 3, 11><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials);
          break;
        case 24:
          linearize_kernel<true, 128, 3, 13><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials);
          break;
        case 9:  // diagnostics: destination gather replaced by a fixed texel
          linearize_kernel<true, 128, 3, 1><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials);
          break;
        case 4: PBA_LAUNCH_LIN(true, 128, 3); break;  // round-1 kernel (comparison)
        case 7:  // lean, row-major walk (comparison)
          linearize_kernel<true, 128, 3, 0, true, false><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials);
          break;
        default:  // 6: lean, tiled walk (DESIGN.md §3 K1)
          if (cfg->flags & PBA_CFG_PINHOLE_DST)
            linearize_kernel<true, 128, 3, 0, true, true, 8><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials);
          else
            linearize_kernel<true, 128, 3, 0, true, true><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials);
          break;
      }
    } else {
      // Cost-only (total_error) path: no accumulators, so it fits 96
      // registers without spills and runs 20 warps/SM — 1.45x faster than at
      // 12 warps (16.1 -> 11.1 ms on c4/200, the path is latency-bound).
      // PBA_COST_VARIANT 3 / 4 / 6 select 12 / 16 / 24 warps per SM.
      static int cvariant = -1;
      if (cvariant < 0) {
        const char* env = getenv("PBA_COST_VARIANT");
        cvariant = env ? atoi(env) : 5;
      }
      switch (cvariant) {
        case 3: PBA_LAUNCH_COST(3); break;
        case 4: PBA_LAUNCH_COST(4); break;
        case 6: PBA_LAUNCH_COST(6); break;
        case 7:  // row-major walk (comparison)
          linearize_kernel<false, 128, 5><<<grid, 128, 0, st>>>(setups, chunk_table, pair_chunk_offsets, chunk_pixels, partials);
          break;
        default: PBA_LAUNCH_COST(5); break;
      }
    }
#undef PBA_LAUNCH_LIN
#undef PBA_LAUNCH_COST
    PBA_LAUNCH_CHECK();
  }
  finalize_pairs_kernel<<<(unsigned)((n_pairs + 3) / 4), 128, 0, st>>>(
      partials, pair_chunk_offsets, pairs, poses, n_pairs, records);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

extern "C" int pba_diag_section_cycles(uint64_t* cycles, uint64_t* counts, int32_t reset) {
  PBA_ARG_CHECK(cycles && counts, "NULL buffer");
  PBA_CUDA_TRY(cudaMemcpyFromSymbol(cycles, g_sect_cycles, sizeof(g_sect_cycles)));
  PBA_CUDA_TRY(cudaMemcpyFromSymbol(counts, g_sect_count, sizeof(g_sect_count)));
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    PBA_CUDA_TRY(cudaMemcpyToSymbol(g_sect_cycles, z, sizeof(z)));
    PBA_CUDA_TRY(cudaMemcpyToSymbol(g_sect_count, z, sizeof(z)));
  }
  return PBA_OK;
}

extern "C" int pba_atan2_batch(const double* y, const double* x, int64_t n, double* out,
                               void* stream) {
  PBA_ARG_CHECK(n >= 0 && (n == 0 || (y && x && out)), "bad arguments");
  if (int rc = ensure_atan_table()) return rc;
  if (n == 0) return PBA_OK;
  atan2_batch_kernel<<<(unsigned)((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      y, x, n, out);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
