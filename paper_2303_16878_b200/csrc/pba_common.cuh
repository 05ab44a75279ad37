// Shared device-side definitions for the B200 photometric-BA kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "pba.h"

namespace pba {

constexpr int kRec = PBA_RECORD_DOUBLES;

// One (frame, level) image as the linearisation kernel reads it: eight
// planes of 16-byte pairs (128 B per pixel in total), plane-major, so the
// 32 lanes of a warp reading the same pair of 32 neighbouring pixels touch
// 4-5 consecutive 128-byte lines (L1 wavefronts) instead of 32 — with a
// 128-byte per-pixel record every gather lane was its own wavefront and the
// L1 data pipe was the bottleneck.  Pair k of pixel p is at
// base[k * W * H + p].  Field order follows the reference channels
// [intensity, depth, nx, ny, nz] (solver.py:340) and the gradient order
// [d/dcol, d/drow] (cues.py:63-71).
enum TexelPair : int {
  kPairID = 0,    // I, D
  kPairNxy = 1,   // nx, ny
  kPairNzM = 2,   // nz, (mask u32, pad u32) — mask in the low word of .y
  kPairGI = 3,    // dI/dcol, dI/drow
  kPairGD = 4,    // dD/dcol, dD/drow
  kPairGN = 5,    // 5, 6, 7: d(nx,ny,nz)/dcol, /drow
  kTexelPairs = 8
};
constexpr int kTexelBytes = 16 * kTexelPairs;

// Checked build (-DPBA_CHECKED -> _lib/libpba_b200_checked.so, selected by
// PBA_CHECKED=1): device-side bounds assertions standing in for
// compute-sanitizer memcheck, which is closed on this GPU pool.  A failed
// check prints one "PBA_CHECK" line and clamps the index, so the kernel
// never touches memory outside the buffer it was checking.
#ifdef PBA_CHECKED
__device__ __forceinline__ long long checked_index(long long i, long long n, const char* file,
                                                   int line) {
  if (i < 0 || i >= n) {
    printf("PBA_CHECK %s:%d index %lld outside [0, %lld)\n", file, line, i, n);
    return i < 0 ? 0 : (n > 0 ? n - 1 : 0);
  }
  return i;
}
#define PBA_DCHECK_INDEX(idx, n) ::pba::checked_index((long long)(idx), (long long)(n), __FILE__, __LINE__)
#else
#define PBA_DCHECK_INDEX(idx, n) (idx)
#endif

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
