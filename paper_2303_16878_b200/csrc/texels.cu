// Device-side CueImage derivation: CueImage.__post_init__ (cues.py:106-147)
// producing the 128-byte texel image and the per-pixel mask plane that the
// linearisation kernel samples.
//
// Three passes over the H x W image (one thread per pixel, coalesced):
//   1. depth clamp (cues.py:113-117), normal validity and zeroing (:118-122)
//   2. 4-neighbour normal coherence (cues.py:47-60, :130)
//   3. central-difference gradients + gradient validity (cues.py:63-81),
//      which are also the sampleable masks (:125-134), written as texels.
// Arithmetic uses explicitly rounded intrinsics where the reference's
// numpy evaluation order matters for bit-exact masks and gradients.

#include <math.h>
#include <stdarg.h>
#include <stdio.h>

#include "pba_common.cuh"

namespace pba {

namespace {

constexpr uint8_t kDV = PBA_MASK_DEPTH_VALID;
constexpr uint8_t kNV = PBA_MASK_NORMAL_VALID;
constexpr uint8_t kCoherent = 0x80;  // scratch bit: normal_valid & neighbour-coherent

// Frame f = blockIdx.y of a batch: inputs at f * H * W (normals f * 3 H W),
// scratch at f * scratch_stride bytes, texels at f * kTexelBytes * H * W.
struct FrameScratch {
  double* d;
  double* n;
  uint8_t* flags;
};
__device__ __forceinline__ FrameScratch frame_scratch(char* scratch, size_t stride, size_t px) {
  char* s = scratch + blockIdx.y * stride;
  FrameScratch f;
  f.d = reinterpret_cast<double*>(s);
  f.n = reinterpret_cast<double*>(s + ((px * sizeof(double) + 255) / 256) * 256);
  f.flags = reinterpret_cast<uint8_t*>(s + ((px * sizeof(double) + 255) / 256) * 256 +
                                       ((px * 3 * sizeof(double) + 255) / 256) * 256);
  return f;
}

__global__ void clean_pass(int H, int W, double dmin, double dmax, const double* __restrict__ depth,
                           const double* __restrict__ normals, char* __restrict__ scratch,
                           size_t scratch_stride) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= H * W) return;
  const size_t px = (size_t)H * W;
  const FrameScratch fs = frame_scratch(scratch, scratch_stride, px);
  double* __restrict__ d_out = fs.d;
  double* __restrict__ n_out = fs.n;
  uint8_t* __restrict__ flags = fs.flags;
  depth += blockIdx.y * px;
  normals += blockIdx.y * 3 * px;
  double d = depth[p];
  // cues.py:114-115: non-finite or out-of-range depth becomes 0 (invalid).
  if (!isfinite(d) || d < dmin || d > dmax) d = 0.0;
  const bool dv = d > 0.0;
  const double nx = normals[3 * p + 0], ny = normals[3 * p + 1], nz = normals[3 * p + 2];
  // np.linalg.norm over the last axis of a 3-vector: sqrt((x*x + y*y) + z*z).
  const double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(nx, nx), __dmul_rn(ny, ny)),
                                         __dmul_rn(nz, nz)));
  const bool nv = (nn > 0.5) && dv;
  d_out[p] = d;
  n_out[3 * p + 0] = nv ? nx : 0.0;
  n_out[3 * p + 1] = nv ? ny : 0.0;
  n_out[3 * p + 2] = nv ? nz : 0.0;
  flags[p] = (dv ? kDV : 0) | (nv ? kNV : 0);
}

__device__ __forceinline__ double dot3_rn(const double* a, const double* b) {
  // einsum("rck,rck->rc") over k = 0..2, summed left to right.
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

__global__ void coherence_pass(int H, int W, char* __restrict__ scratch, size_t scratch_stride) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= H * W) return;
  const FrameScratch fs = frame_scratch(scratch, scratch_stride, (size_t)H * W);
  const double* __restrict__ n = fs.n;
  uint8_t* __restrict__ flags = fs.flags;
  const int r = p / W, c = p - r * W;
  uint8_t f = flags[p];
  bool coherent = false;
  if ((f & kNV) && r > 0 && r < H - 1 && c > 0 && c < W - 1) {
    const double* ctr = n + 3 * p;
    // cues.py:52-58: right, left, down, up neighbours, each dot >= 0.9.
    coherent = dot3_rn(ctr, n + 3 * (p + 1)) >= 0.9 && dot3_rn(ctr, n + 3 * (p - 1)) >= 0.9 &&
               dot3_rn(ctr, n + 3 * (p + W)) >= 0.9 && dot3_rn(ctr, n + 3 * (p - W)) >= 0.9;
  }
  flags[p] = coherent ? (f | kCoherent) : f;
}

__global__ void gradient_pass(int H, int W, const double* __restrict__ inten,
                              char* __restrict__ scratch, size_t scratch_stride,
                              double2* __restrict__ out, uint8_t* __restrict__ mask_out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= H * W) return;
  const size_t px = (size_t)H * W;
  const FrameScratch fs = frame_scratch(scratch, scratch_stride, px);
  const double* __restrict__ d = fs.d;
  const double* __restrict__ n = fs.n;
  const uint8_t* __restrict__ flags = fs.flags;
  inten += blockIdx.y * px;
  out += blockIdx.y * (px * (kTexelBytes / sizeof(double2)));
  mask_out += blockIdx.y * px;
  const int r = p / W, c = p - r * W;
  const uint8_t f = flags[p];
  double g[10];
  bool core_ok = false, norm_ok = false;
  const bool interior = r > 0 && r < H - 1 && c > 0 && c < W - 1;
  if (interior) {
    const uint8_t fr = flags[p + 1], fl = flags[p - 1], fd = flags[p + W], fu = flags[p - W];
    core_ok = (f & fr & fl & fd & fu & kDV) != 0;                // cues.py:72-79 on depth_valid
    norm_ok = (f & fr & fl & fd & fu & kCoherent) != 0;          // ... on the coherent mask
  }
  // cues.py:70-71: 0.5 * (right - left), 0.5 * (down - up); zero where invalid (:80).
  if (core_ok) {
    g[0] = __dmul_rn(0.5, __dsub_rn(inten[p + 1], inten[p - 1]));
    g[1] = __dmul_rn(0.5, __dsub_rn(inten[p + W], inten[p - W]));
    g[2] = __dmul_rn(0.5, __dsub_rn(d[p + 1], d[p - 1]));
    g[3] = __dmul_rn(0.5, __dsub_rn(d[p + W], d[p - W]));
  } else {
    g[0] = g[1] = g[2] = g[3] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (norm_ok) {
      g[4 + 2 * k] = __dmul_rn(0.5, __dsub_rn(n[3 * (p + 1) + k], n[3 * (p - 1) + k]));
      g[5 + 2 * k] = __dmul_rn(0.5, __dsub_rn(n[3 * (p + W) + k], n[3 * (p - W) + k]));
    } else {
      g[4 + 2 * k] = g[5 + 2 * k] = 0.0;
    }
  }
  const uint32_t m = (f & (kDV | kNV)) | (core_ok ? PBA_MASK_SAMP_CORE : 0u) |
                     (norm_ok ? PBA_MASK_SAMP_NORMAL : 0u);
  const int64_t np = (int64_t)H * W;
  out[kPairID * np + p] = make_double2(inten[p], d[p]);
  out[kPairNxy * np + p] = make_double2(n[3 * p + 0], n[3 * p + 1]);
  out[kPairNzM * np + p] = make_double2(n[3 * p + 2], __longlong_as_double((long long)m));
#pragma unroll
  for (int k = 0; k < 5; ++k) out[(kPairGI + k) * np + p] = make_double2(g[2 * k], g[2 * k + 1]);
  mask_out[p] = (uint8_t)m;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

}  // namespace pba

using namespace pba;

extern "C" size_t pba_texel_bytes(void) { return kTexelBytes; }

extern "C" size_t pba_ray_table_doubles(const pba_camera* cam) {
  if (!cam) return 0;
  return 2 * (size_t)cam->width + 2 * (size_t)cam->height;
}

extern "C" size_t pba_build_texels_scratch_bytes(const pba_camera* cam) {
  if (!cam) return 0;
  const size_t px = (size_t)cam->width * cam->height;
  return align_up(px * sizeof(double), 256) + align_up(px * 3 * sizeof(double), 256) +
         align_up(px, 256);
}

extern "C" int pba_build_texels_batch(const pba_camera* cam, int32_t n_frames,
                                      const double* intensity, const double* depth,
                                      const double* normals, void* texels, uint8_t* mask,
                                      void* scratch, void* stream) {
  PBA_ARG_CHECK(cam != nullptr, "cam is NULL");
  PBA_ARG_CHECK(cam->width >= 2 && cam->height >= 2, "image must be at least 2x2");
  PBA_ARG_CHECK(n_frames >= 0 && n_frames <= 65535, "n_frames must lie in [0, 65535]");
  if (n_frames == 0) return PBA_OK;
  PBA_ARG_CHECK(intensity && depth && normals && texels && mask && scratch, "NULL buffer");
  const int H = cam->height, W = cam->width;
  const size_t px = (size_t)W * H;
  const size_t stride = pba_build_texels_scratch_bytes(cam);
  char* s = static_cast<char*>(scratch);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int threads = 256;
  const dim3 grid((unsigned)((px + threads - 1) / threads), (unsigned)n_frames);
  clean_pass<<<grid, threads, 0, st>>>(H, W, cam->depth_min, cam->depth_max, depth, normals, s,
                                        stride);
  PBA_LAUNCH_CHECK();
  coherence_pass<<<grid, threads, 0, st>>>(H, W, s, stride);
  PBA_LAUNCH_CHECK();
  gradient_pass<<<grid, threads, 0, st>>>(H, W, intensity, s, stride,
                                           static_cast<double2*>(texels), mask);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

extern "C" int pba_build_texels(const pba_camera* cam, const double* intensity,
                                const double* depth, const double* normals, void* texels,
                                uint8_t* mask, void* scratch, void* stream) {
  return pba_build_texels_batch(cam, 1, intensity, depth, normals, texels, mask, scratch, stream);
}
