// K4: pose update  X_k <- X_k * exp([dt, dq])  for every non-gauge pose.
// Reference: _LevelProblem.apply_step (solver.py:451-460) -> boxplus / exp /
// quat_to_rotation / Pose.compose (geometry.py:30-45, 137-143, 202-219).

#include <math.h>

#include "pba_common.cuh"

namespace pba {
namespace {

// Polar factor of a near-rotation (the SVD u @ vt of geometry.py:91-98):
// Newton iteration X <- (X + X^{-T}) / 2, which converges quadratically to
// the same orthonormal factor.
__device__ void orthonormalize(double* R) {
  for (int it = 0; it < 8; ++it) {
    const double a = R[0], b = R[1], c = R[2], d = R[3], e = R[4], f = R[5], g = R[6], h = R[7],
                 i = R[8];
    const double C0 = e * i - f * h, C1 = -(d * i - f * g), C2 = d * h - e * g;
    const double C3 = -(b * i - c * h), C4 = a * i - c * g, C5 = -(a * h - b * g);
    const double C6 = b * f - c * e, C7 = -(a * f - c * d), C8 = a * e - b * d;
    const double det = a * C0 + b * C1 + c * C2;
    // X^{-T} = cofactor / det
    const double id = 1.0 / det;
    double delta = 0.0;
    const double Cm[9] = {C0, C1, C2, C3, C4, C5, C6, C7, C8};
    for (int k = 0; k < 9; ++k) {
      const double nv = 0.5 * (R[k] + Cm[k] * id);
      delta = fmax(delta, fabs(nv - R[k]));
      R[k] = nv;
    }
    if (delta < 1e-16) break;
  }
}

__global__ void apply_step_kernel(const double* __restrict__ in, const int32_t* __restrict__ gen_in,
                                  const double* __restrict__ delta, int n, int gauge,
                                  double* __restrict__ out, int32_t* __restrict__ gen_out,
                                  int32_t* __restrict__ status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double* X = in + 12 * k;
  double* Y = out + 12 * k;
  if (k == gauge) {
    for (int e = 0; e < 12; ++e) Y[e] = X[e];
    gen_out[k] = gen_in[k];
    return;
  }
  const int s = k < gauge ? k : k - 1;  // slot order skips the gauge (solver.py:433, 453-459)
  const double* v = delta + 6 * s;
  const double qx = v[3], qy = v[4], qz = v[5];
  const double nq2 = qx * qx + qy * qy + qz * qz;
  if (nq2 >= 1.0) {  // InvalidPerturbationError (geometry.py:208-212)
    *status = 1;
    for (int e = 0; e < 12; ++e) Y[e] = X[e];
    gen_out[k] = gen_in[k];
    return;
  }
  const double qw = sqrt(1.0 - nq2);
  // quat_to_rotation (geometry.py:30-45)
  const double nrm = qw * qw + qx * qx + qy * qy + qz * qz;
  const double sc = 2.0 / nrm;
  const double wx = sc * qw * qx, wy = sc * qw * qy, wz = sc * qw * qz;
  const double xx = sc * qx * qx, xy = sc * qx * qy, xz = sc * qx * qz;
  const double yy = sc * qy * qy, yz = sc * qy * qz, zz = sc * qz * qz;
  const double D[9] = {1.0 - (yy + zz), xy - wz,         xz + wy,
                       xy + wz,         1.0 - (xx + zz), yz - wx,
                       xz - wy,         yz + wx,         1.0 - (xx + yy)};
  // compose: R = R_k D, t = R_k dt + t_k (geometry.py:137-143)
  double R[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      R[3 * r + c] = X[3 * r + 0] * D[c] + X[3 * r + 1] * D[3 + c] + X[3 * r + 2] * D[6 + c];
  for (int r = 0; r < 3; ++r)
    Y[9 + r] = X[3 * r + 0] * v[0] + X[3 * r + 1] * v[1] + X[3 * r + 2] * v[2] + X[9 + r];
  int g = gen_in[k] + 1;
  if (g >= 1000) {  // REORTHO_INTERVAL (geometry.py:17, 140-142)
    orthonormalize(R);
    g = 0;
  }
  for (int e = 0; e < 9; ++e) Y[e] = R[e];
  gen_out[k] = g;
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" int pba_apply_step(const double* poses_in, const int32_t* gen_in, const double* delta,
                              int32_t n_poses, int32_t gauge, double* poses_out, int32_t* gen_out,
                              int32_t* status, void* stream) {
  PBA_ARG_CHECK(n_poses >= 1 && gauge >= 0 && gauge < n_poses, "bad pose count / gauge");
  PBA_ARG_CHECK(poses_in && gen_in && delta && poses_out && gen_out && status, "NULL buffer");
  PBA_ARG_CHECK(poses_in != poses_out, "apply_step is out of place");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PBA_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  apply_step_kernel<<<(n_poses + 127) / 128, 128, 0, st>>>(poses_in, gen_in, delta, n_poses, gauge,
                                                           poses_out, gen_out, status);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
