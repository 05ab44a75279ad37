// Division-free fp64 atan2 for the spherical projection (sensors.py:120-121).
//
// For any table angle theta_k (c_k = cos, s_k = sin), rotating (x, y) by
// -theta_k gives sin(theta - theta_k) = (y c_k - x s_k) / r.  theta_k is
// picked from a 513-entry table over [-pi, pi] by a cheap fp32 guess, so
// |theta - theta_k| <= pi/512 + 1e-5 and asin of that sine is an odd series
// exact to ~1e-25; the result is within ~1 ulp of pi absolute (tested against
// numpy.arctan2).  The library atan2 calls were 25% of the linearisation
// kernel's instructions and long dependent chains.
#pragma once

#include <cuda_runtime.h>
#include <math.h>

namespace pba {

constexpr int kAtanHalf = 256;  // table covers k = -256 .. 256
struct __align__(16) AtanEntry {
  double c, s;          // cos/sin of the table angle, rounded to double
  double theta, theta_lo;  // exact angle of (c, s) as a double-double
};

// Defined here (header-only; include from exactly one translation unit).
__device__ AtanEntry g_atan_table[2 * kAtanHalf + 1];

// Host: fill the table for the current device (idempotent per device).
int ensure_atan_table();

// Cheap fp32 atan2 (max error ~1e-5 rad): only has to pick the table slot.
// The sign comes from the fp64 y (signbit) so that y = -0 or a negative y
// that underflows in fp32 still selects the -pi side of the branch cut.
__device__ __forceinline__ float atan2_guess(float y, float x, bool y_negative) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  // approximate quotient (MUFU.RCP + FMUL, ~2 ulp): the guess only has to
  // land within the series' reach of a table angle (3e-3 rad of margin)
  const float a = __fdividef(mn, mx);
  const float s = a * a;
  float r = fmaf(fmaf(fmaf(-0.0464964749f, s, 0.15931422f), s, -0.327622764f), s * a, a);
  if (ay > ax) r = 1.57079637f - r;
  if (x < 0.0f) r = 3.14159274f - r;
  return y_negative ? -r : r;
}

// atan2(y, x) given inv_r = 1 / |(x, y)| (computed once by the caller with
// rsqrt, which also yields the range and the Jacobian reciprocals):
//   Delta = theta - theta_k,  sin Delta = (y c_k - x s_k) * inv_r,
//   atan2 = theta_k + asin(sin Delta)  (|sin Delta| < 0.0063, odd series to s^9).
// No division; measured on B200: fp64 divide ~130 cycles, sqrt ~100,
// rsqrt ~75 of dependent latency vs 8 for a DFMA.
__device__ __forceinline__ double atan2_tab_r(double y, double x, double inv_r) {
  const float tf = atan2_guess((float)y, (float)x, signbit(y));
  int k = __float2int_rn(tf * (float)(kAtanHalf / 3.14159265358979323846));
  k = min(max(k, -kAtanHalf), kAtanHalf);
  const AtanEntry* e = &g_atan_table[k + kAtanHalf];
  const double2 cs = __ldg(reinterpret_cast<const double2*>(e));
  const double2 th = __ldg(reinterpret_cast<const double2*>(e) + 1);  // (hi, lo)
  // y c - x s with the product error of x s recovered by an FMA: the small
  // difference keeps full relative accuracy, so the only significant rounding
  // is the final add and the result is (almost always) correctly rounded.
  const double w = x * cs.y;
  const double werr = fma(x, cs.y, -w);
  const double num = fma(y, cs.x, -w) - werr;
  const double sd = num * inv_r;
  const double s2 = sd * sd;
  double p = fma(s2, 35.0 / 1152.0, 5.0 / 112.0);
  p = fma(p, s2, 3.0 / 40.0);
  p = fma(p, s2, 1.0 / 6.0);
  return th.x + (th.y + fma(sd * s2, p, sd));
}

// Stand-alone atan2 (diagnostics / rare paths): same method, inv_r via rsqrt.
__device__ __forceinline__ double atan2_tab(double y, double x) {
  if (x == 0.0 && y == 0.0) return atan2(y, x);  // signed-zero semantics
  const double rr = x * x + y * y;
  if (!(rr > 1e-300 && rr < 1e300)) return atan2(y, x);
  return atan2_tab_r(y, x, rsqrt(rr));
}

}  // namespace pba
