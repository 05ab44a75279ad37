// K5: covisibility overlap counts for match-graph construction.
// Reference: overlap_ratio (graph.py:70-101) inside build_graph
// (graph.py:123-176): the fraction of frame i's valid pixels (at the graph
// level, stride 2) that project validly into frame j, with bound_slack 1e-6.
//
// One CTA per directed candidate pair.  The sensor-frame points of every
// frame are computed on the host with the reference's own numpy expressions
// and uploaded once; the kernel applies the pair's composed transform
// (sensor_j^-1 * sensor_i, also composed on the host exactly as the
// reference) and the projection, and counts valid points with a fixed-order
// block reduction.  The host (pairgraph.build_graph) re-decides any pair
// whose ratio lies within a few points of the threshold with the exact numpy
// path, so the edge list is identical to the reference's.

#include <math.h>

#include "pba_common.cuh"

namespace pba {
namespace {

__device__ __forceinline__ bool project_ok(const pba_camera& cam, double x, double y, double z,
                                           double slack) {
  double u, v, d;
  if (cam.model == PBA_SPHERICAL) {
    const double xx = __dmul_rn(x, x), yy = __dmul_rn(y, y);
    const double rr = __dadd_rn(xx, yy);
    const double r2 = __dadd_rn(rr, __dmul_rn(z, z));
    d = __dsqrt_rn(r2);
    const double az = atan2(y, x);
    const double el = atan2(z, hypot(x, y));
    double m = __dadd_rn(__dmul_rn(cam.fx, az), cam.cx);
    const double w = (double)cam.width;
    m = fmod(m, w);
    if (m != 0.0 && m < 0.0) m += w;
    u = m;
    v = __dadd_rn(__dmul_rn(cam.fy, el), cam.cy);
  } else {
    if (!(z > 0.0)) return false;
    u = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fx, x), z), cam.cx);
    v = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fy, y), z), cam.cy);
    d = z;
  }
  return (d >= cam.depth_min) && (d <= cam.depth_max) && (u >= -slack) &&
         (u < cam.width + slack) && (v >= -slack) && (v < cam.height + slack);
}

__global__ void __launch_bounds__(256) overlap_kernel(const double* __restrict__ points,
                                                      const int64_t* __restrict__ point_offsets,
                                                      const int32_t* __restrict__ pair_src,
                                                      const double* __restrict__ transforms,
                                                      const pba_camera* __restrict__ dst_cams,
                                                      double slack, int64_t* __restrict__ counts) {
  const int p = blockIdx.x;
  const int f = pair_src[p];
  const int64_t b = point_offsets[f], e = point_offsets[f + 1];
  const double* T = transforms + 12 * (int64_t)p;
  const double R0 = T[0], R1 = T[1], R2 = T[2], R3 = T[3], R4 = T[4], R5 = T[5], R6 = T[6],
               R7 = T[7], R8 = T[8], t0 = T[9], t1 = T[10], t2 = T[11];
  const pba_camera cam = dst_cams[p];
  int64_t n = 0;
  for (int64_t k = b + threadIdx.x; k < e; k += blockDim.x) {
    const double x = points[3 * k], y = points[3 * k + 1], z = points[3 * k + 2];
    // p @ R.T + t (Pose.transform, geometry.py:149-152)
    const double X = R0 * x + R1 * y + R2 * z + t0;
    const double Y = R3 * x + R4 * y + R5 * z + t1;
    const double Z = R6 * x + R7 * y + R8 * z + t2;
    n += project_ok(cam, X, Y, Z, slack) ? 1 : 0;
  }
  __shared__ int64_t red[256];
  red[threadIdx.x] = n;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[p] = red[0];
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" int pba_overlap_counts(const double* points, const int64_t* point_offsets,
                                  const int32_t* pair_src, const double* transforms,
                                  const pba_camera* dst_cams, int32_t n_pairs, double bound_slack,
                                  int64_t* counts, void* stream) {
  PBA_ARG_CHECK(n_pairs >= 0, "n_pairs < 0");
  if (n_pairs == 0) return PBA_OK;
  PBA_ARG_CHECK(points && point_offsets && pair_src && transforms && dst_cams && counts,
                "NULL buffer");
  overlap_kernel<<<n_pairs, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      points, point_offsets, pair_src, transforms, dst_cams, bound_slack, counts);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
