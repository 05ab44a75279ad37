// fp64 atan2 at a third of the cost of the CUDA library routine.
//
// atan2(y, x) = theta_k + atan(d),  d = (y c_k - x s_k) / (x c_k + y s_k)
// for any table angle theta_k with c_k = cos theta_k, s_k = sin theta_k
// (rotate (x, y) by -theta_k).  theta_k is picked from a 513-entry table
// over [-pi, pi] by an fp32 atan2f guess, so |theta - theta_k| <= pi/512 + 1e-6
// and |d| < 0.0062: the odd series d - d^3/3 + ... + d^9/9 is exact to
// d^11/11 < 1e-25 relative, leaving only the rounding of one division and
// the final add (<= 1 ulp, vs ~2 ulp for the library atan2).  Used for the
// spherical projection (sensors.py:120-121), where the two library atan2
// calls were 25% of the linearisation kernel's instructions.
#pragma once

#include <cuda_runtime.h>
#include <math.h>

namespace pba {

constexpr int kAtanHalf = 256;  // table covers k = -256 .. 256
struct __align__(16) AtanEntry {
  double c, s, theta, pad;
};

// Defined here (header-only; include from exactly one translation unit).
__device__ AtanEntry g_atan_table[2 * kAtanHalf + 1];

// Host: fill the table for the current device (idempotent per device).
int ensure_atan_table();

// fp64 reciprocal: fp32 seed + 3 Newton steps (relative error < 1e-17 before
// the final rounding), ~8 instructions instead of the IEEE division sequence.
__device__ __forceinline__ double rcp_nr(double x) {
  const double ax = fabs(x);
  if (!(ax > 1e-30 && ax < 1e30)) return 1.0 / x;  // outside the fp32 seed's range
  double r = (double)__frcp_rn((float)x);
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

// Cheap fp32 atan2 (max error ~1e-5 rad): only has to pick the table slot.
// The sign comes from the fp64 y (signbit) so that y = -0 or a negative y
// that underflows in fp32 still selects the -pi side of the branch cut.
__device__ __forceinline__ float atan2_guess(float y, float x, bool y_negative) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = mn * __frcp_rn(mx);
  const float s = a * a;
  float r = fmaf(fmaf(fmaf(-0.0464964749f, s, 0.15931422f), s, -0.327622764f), s * a, a);
  if (ay > ax) r = 1.57079637f - r;
  if (x < 0.0f) r = 3.14159274f - r;
  return y_negative ? -r : r;
}

__device__ __forceinline__ double atan2_tab(double y, double x) {
  if (x == 0.0 && y == 0.0) return atan2(y, x);  // signed-zero semantics
  const float tf = atan2_guess((float)y, (float)x, signbit(y));
  int k = __float2int_rn(tf * (float)(kAtanHalf / 3.14159265358979323846));
  k = min(max(k, -kAtanHalf), kAtanHalf);
  const AtanEntry* e = &g_atan_table[k + kAtanHalf];
  const double2 cs = __ldg(reinterpret_cast<const double2*>(e));
  const double th = __ldg(&e->theta);
  const double num = y * cs.x - x * cs.y;
  const double den = x * cs.x + y * cs.y;
  const double d = num * rcp_nr(den);  // den ~ |(x, y)| > 0
  const double d2 = d * d;
  double p = fma(d2, 1.0 / 9.0, -1.0 / 7.0);
  p = fma(p, d2, 1.0 / 5.0);
  p = fma(p, d2, -1.0 / 3.0);
  return th + fma(d * d2, p, d);
}

}  // namespace pba
