// K7: raster decode for dataset loading.
// Reference: read_raster / read_intensity / read_depth (dataset_io.py:74-136)
// and the PGM P5 format (pkg/docs/formats.md:7-20).  The host parses the
// headers and gathers every frame's payload into one pinned buffer; this
// kernel turns the big-endian 16-bit (or 8-bit) samples into fp64 in the
// (n, H, W) planes the pyramid builder (K6) consumes, with the reference's
// arithmetic: intensity raw / 65535 (raw / 255 for 8-bit) as an IEEE
// division, depth raw * depth_scale as one rounded multiply.

#include "pba_common.cuh"

namespace pba {
namespace {

__global__ void __launch_bounds__(256) decode_kernel(const uint8_t* __restrict__ raw,
                                                     int64_t n, int32_t kind, double scale,
                                                     double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v;
  if (kind == PBA_RASTER_U8_INTENSITY) {
    v = __ddiv_rn((double)raw[i], 255.0);
  } else {
    const uint32_t s = ((uint32_t)raw[2 * i] << 8) | (uint32_t)raw[2 * i + 1];
    v = kind == PBA_RASTER_U16_DEPTH ? __dmul_rn((double)s, scale) : __ddiv_rn((double)s, 65535.0);
  }
  out[i] = v;
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" int pba_decode_raster(const uint8_t* raw, int64_t n_samples, int32_t kind,
                                 double depth_scale, double* out, void* stream) {
  PBA_ARG_CHECK(n_samples >= 0, "n_samples < 0");
  PBA_ARG_CHECK(kind == PBA_RASTER_U8_INTENSITY || kind == PBA_RASTER_U16_INTENSITY ||
                    kind == PBA_RASTER_U16_DEPTH,
                "unknown raster kind");
  PBA_ARG_CHECK(kind != PBA_RASTER_U16_DEPTH || depth_scale > 0.0, "depth_scale must be > 0");
  if (n_samples == 0) return PBA_OK;
  PBA_ARG_CHECK(raw && out, "NULL buffer");
  decode_kernel<<<(unsigned)((n_samples + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      raw, n_samples, kind, depth_scale, out);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
