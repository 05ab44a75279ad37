// Shared device-side definitions for the B200 photometric-BA kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pba.h"

namespace pba {

constexpr int kRec = PBA_RECORD_DOUBLES;

// One (frame, level) pixel as the linearisation kernel reads it: the five
// cue values and their ten central-difference gradients in fp64 plus the
// validity bits, 128 B = one L2 line, so the four bilinear corners of a
// destination sample are four aligned lines.  Field order follows the
// reference channels [intensity, depth, nx, ny, nz] (solver.py:340) and the
// gradient order [d/dcol, d/drow] (cues.py:63-71); every (col,row) gradient
// pair and the (I,D), (nx,ny) value pairs sit on 16-byte boundaries so they
// load as one 128-bit access.
struct __align__(16) Texel {
  double v[5];   // I, D, nx, ny, nz                                   0..39
  uint32_t mask; // PBA_MASK_*                                         40
  uint32_t pad;  //                                                    44
  double g[10];  // gI(c,r), gD(c,r), gnx(c,r), gny(c,r), gnz(c,r)   48..127
};
static_assert(sizeof(Texel) == 128, "texel must be one 128-byte line");

// Thread-local error message for pba_last_error().
void set_error(const char* fmt, ...);
// Process-wide count of kernels launched by the library (pba_kernel_launches()).
void count_launch();

}  // namespace pba

#define PBA_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::pba::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),      \
                       __FILE__, __LINE__);                                         \
      return PBA_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

#define PBA_LAUNCH_CHECK()                                                          \
  do {                                                                              \
    ::pba::count_launch();                                                          \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) {                                                        \
      ::pba::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e),  \
                       __FILE__, __LINE__);                                         \
      return PBA_ERR_CUDA;                                                          \
    }                                                                               \
  } while (0)

#define PBA_ARG_CHECK(cond, msg)                                                    \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      ::pba::set_error("invalid argument: %s", msg);                                \
      return PBA_ERR_ARG;                                                           \
    }                                                                               \
  } while (0)
