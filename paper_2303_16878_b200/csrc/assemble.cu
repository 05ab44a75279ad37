// K2: fixed-edge-order assembly of per-pair records into the dense normal
// equations — the loop of _LevelProblem.evaluate (solver.py:428-449).
//
// The reference adds, for every edge in order, H_ii into the i slot, H_jj
// into the j slot, H_ij / H_ij^T into the two off-diagonal blocks, and the
// b blocks likewise; gauge contributions are dropped (solver.py:433-448).
// Here the host builds (once per level) a CSR plan listing, per target
// block, the contributing records in edge order; one thread per target
// entry then sums its list sequentially, which reproduces the reference
// order for every entry and is independent of how records were produced.

#include <map>
#include <utility>
#include <vector>

#include "pba_common.cuh"

namespace pba {
namespace {

__device__ __forceinline__ double upper_get(const double* u, int k, int l) {
  if (k > l) {
    const int t = k;
    k = l;
    l = t;
  }
  return u[k * 6 - (k * (k - 1)) / 2 + (l - k)];
}

// Threads [0, n_free*42): diagonal targets (36 H entries + 6 b entries each).
// Threads [n_free*42, n_free*42 + n_off*36): off-diagonal block entries.
__global__ void assemble_kernel(const double* __restrict__ rec, int n_free,
                                const int32_t* __restrict__ diag_ptr,
                                const int32_t* __restrict__ diag_items, int n_off,
                                const int32_t* __restrict__ off_ptr,
                                const int32_t* __restrict__ off_rc,
                                const int32_t* __restrict__ off_items, double* __restrict__ H,
                                double* __restrict__ b) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long dim = 6L * n_free;
  const long n_diag = 42L * n_free;
  if (t < n_diag) {
    const int s = (int)(t / 42), e = (int)(t - 42L * s);
    const int i0 = diag_ptr[s], i1 = diag_ptr[s + 1];
    double acc = 0.0;
    if (e < 36) {
      const int k = e / 6, l = e - 6 * (e / 6);
      for (int it = i0; it < i1; ++it) {
        const int item = diag_items[it];
        const double* r = rec + (long)(item >> 1) * kRec;
        acc += upper_get(r + ((item & 1) ? PBA_REC_HJJ : PBA_REC_HII), k, l);
      }
      H[PBA_DCHECK_INDEX((6L * s + k) * dim + 6L * s + l, dim * dim)] = acc;
    } else {
      const int k = e - 36;
      for (int it = i0; it < i1; ++it) {
        const int item = diag_items[it];
        const double* r = rec + (long)(item >> 1) * kRec;
        acc += r[((item & 1) ? PBA_REC_BJ : PBA_REC_BI) + k];
      }
      b[6L * s + k] = acc;
    }
    return;
  }
  const long u = t - n_diag;
  if (u >= 36L * n_off) return;
  const int o = (int)(u / 36), e = (int)(u - 36L * o);
  const int k = e / 6, l = e - 6 * (e / 6);
  double acc = 0.0;
  for (int it = off_ptr[o]; it < off_ptr[o + 1]; ++it) {
    const int item = off_items[it];
    const double* hij = rec + (long)(item >> 1) * kRec + PBA_REC_HIJ;
    acc += (item & 1) ? hij[6 * l + k] : hij[6 * k + l];
  }
  const long r = off_rc[2 * o], c = off_rc[2 * o + 1];
  H[PBA_DCHECK_INDEX((6 * r + k) * dim + 6 * c + l, dim * dim)] = acc;
  H[PBA_DCHECK_INDEX((6 * c + l) * dim + 6 * r + k, dim * dim)] = acc;
}

// The same sums into the block-sparse (BSR) normal matrix: block-row CSR of
// 6x6 blocks (the diagonal and both orientations of every off-diagonal
// block, full symmetric storage), Hb[blk * 36 + 6 k + l].  diag_blk[s] /
// off_blk[2 o], off_blk[2 o + 1] are the CSR positions of the diagonal block
// of slot s and of the (r, c) / (c, r) blocks of off-diagonal target o.
// Entry by entry the sums run in the same edge order as assemble_kernel,
// so Hb holds exactly the dense H's non-zero blocks.
__device__ __forceinline__ void assemble_bsr_entry(long t, const double* __restrict__ rec,
                                                   int n_free,
                                                   const int32_t* __restrict__ diag_ptr,
                                                   const int32_t* __restrict__ diag_items,
                                                   int n_off,
                                                   const int32_t* __restrict__ off_ptr,
                                                   const int32_t* __restrict__ off_items,
                                                   const int32_t* __restrict__ diag_blk,
                                                   const int32_t* __restrict__ off_blk,
                                                   double* __restrict__ Hb,
                                                   double* __restrict__ b) {
  const long n_diag = 42L * n_free;
  if (t < n_diag) {
    const int s = (int)(t / 42), e = (int)(t - 42L * s);
    const int i0 = diag_ptr[s], i1 = diag_ptr[s + 1];
    double acc = 0.0;
    if (e < 36) {
      const int k = e / 6, l = e - 6 * (e / 6);
      for (int it = i0; it < i1; ++it) {
        const int item = diag_items[it];
        const double* r = rec + (long)(item >> 1) * kRec;
        acc += upper_get(r + ((item & 1) ? PBA_REC_HJJ : PBA_REC_HII), k, l);
      }
      Hb[(long)diag_blk[s] * 36 + 6 * k + l] = acc;
    } else {
      const int k = e - 36;
      for (int it = i0; it < i1; ++it) {
        const int item = diag_items[it];
        const double* r = rec + (long)(item >> 1) * kRec;
        acc += r[((item & 1) ? PBA_REC_BJ : PBA_REC_BI) + k];
      }
      b[6L * s + k] = acc;
    }
    return;
  }
  const long u = t - n_diag;
  if (u >= 36L * n_off) return;
  const int o = (int)(u / 36), e = (int)(u - 36L * o);
  const int k = e / 6, l = e - 6 * (e / 6);
  double acc = 0.0;
  for (int it = off_ptr[o]; it < off_ptr[o + 1]; ++it) {
    const int item = off_items[it];
    const double* hij = rec + (long)(item >> 1) * kRec + PBA_REC_HIJ;
    acc += (item & 1) ? hij[6 * l + k] : hij[6 * k + l];
  }
  Hb[(long)off_blk[2 * o] * 36 + 6 * k + l] = acc;      // block (r, c)
  Hb[(long)off_blk[2 * o + 1] * 36 + 6 * l + k] = acc;  // block (c, r) = (r, c)^T
}

// cost and count summed over pairs: each thread a contiguous edge range in
// order, then a fixed tree — deterministic for a given pair count.
__device__ __forceinline__ void totals_block(const double* __restrict__ rec, int n_pairs,
                                             double* __restrict__ totals) {
  __shared__ double sc[256], sn[256];
  const int tid = threadIdx.x;
  const int per = (n_pairs + 255) / 256;
  const int p0 = tid * per, p1 = min(p0 + per, n_pairs);
  double c = 0.0, n = 0.0;
  for (int p = p0; p < p1; ++p) {
    c += rec[(long)p * kRec + PBA_REC_COST];
    n += rec[(long)p * kRec + PBA_REC_COUNT];
  }
  sc[tid] = c;
  sn[tid] = n;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (tid < s) {
      sc[tid] += sc[tid + s];
      sn[tid] += sn[tid + s];
    }
    __syncthreads();
  }
  if (tid == 0) {
    totals[0] = sc[0];
    totals[1] = sn[0];
  }
}

__global__ void totals_kernel(const double* __restrict__ rec, int n_pairs,
                              double* __restrict__ totals) {
  totals_block(rec, n_pairs, totals);
}

// The block-sparse assembly with the totals as one more CTA of the same
// launch (the last one; 256 threads, the same fixed tree as totals_kernel),
// so an LM step issues one launch for both.
__global__ void __launch_bounds__(256) assemble_bsr_kernel(
    const double* __restrict__ rec, int n_free, const int32_t* __restrict__ diag_ptr,
    const int32_t* __restrict__ diag_items, int n_off, const int32_t* __restrict__ off_ptr,
    const int32_t* __restrict__ off_items, const int32_t* __restrict__ diag_blk,
    const int32_t* __restrict__ off_blk, double* __restrict__ Hb, double* __restrict__ b,
    int n_pairs, double* __restrict__ totals) {
  if (blockIdx.x == gridDim.x - 1) {
    totals_block(rec, n_pairs, totals);
    return;
  }
  assemble_bsr_entry((long)blockIdx.x * blockDim.x + threadIdx.x, rec, n_free, diag_ptr,
                     diag_items, n_off, off_ptr, off_items, diag_blk, off_blk, Hb, b);
}

}  // namespace
}  // namespace pba

using namespace pba;

extern "C" int pba_plan_assembly(const int32_t* slot_of_pose, int32_t n_poses,
                                 const int32_t* pair_pose_i, const int32_t* pair_pose_j,
                                 int32_t n_pairs, int32_t* diag_ptr, int32_t* diag_items,
                                 int32_t* off_ptr, int32_t* off_rc, int32_t* off_items,
                                 int32_t* n_off_out) {
  PBA_ARG_CHECK(n_poses >= 1 && n_pairs >= 0, "bad sizes");
  PBA_ARG_CHECK(slot_of_pose && (n_pairs == 0 || (pair_pose_i && pair_pose_j)), "NULL input");
  int n_free = 0;
  for (int k = 0; k < n_poses; ++k) n_free = slot_of_pose[k] >= 0 ? n_free + 1 : n_free;
  std::vector<std::vector<int32_t>> diag(n_free);
  std::map<std::pair<int, int>, int> block_of;
  std::vector<std::pair<int, int>> blocks;
  std::vector<std::vector<int32_t>> off;
  for (int e = 0; e < n_pairs; ++e) {
    const int pi = pair_pose_i[e], pj = pair_pose_j[e];
    PBA_ARG_CHECK(pi >= 0 && pi < n_poses && pj >= 0 && pj < n_poses, "pose index out of range");
    const int si = slot_of_pose[pi], sj = slot_of_pose[pj];
    PBA_ARG_CHECK(si < n_free && sj < n_free, "slot out of range");
    if (si >= 0) diag[si].push_back(e << 1);
    if (sj >= 0) diag[sj].push_back((e << 1) | 1);
    if (si >= 0 && sj >= 0) {
      PBA_ARG_CHECK(si != sj, "pair connects a pose to itself");
      const int r = si < sj ? si : sj, c = si < sj ? sj : si;
      auto key = std::make_pair(r, c);
      auto it = block_of.find(key);
      int o;
      if (it == block_of.end()) {
        o = (int)blocks.size();
        block_of.emplace(key, o);
        blocks.push_back(key);
        off.emplace_back();
      } else {
        o = it->second;
      }
      off[o].push_back((e << 1) | (si > sj ? 1 : 0));
    }
  }
  if (n_off_out) *n_off_out = (int32_t)blocks.size();
  if (diag_ptr && diag_items) {
    int32_t pos = 0;
    for (int s = 0; s < n_free; ++s) {
      diag_ptr[s] = pos;
      for (int32_t it : diag[s]) diag_items[pos++] = it;
    }
    diag_ptr[n_free] = pos;
  }
  if (off_ptr && off_rc && off_items) {
    int32_t pos = 0;
    for (size_t o = 0; o < blocks.size(); ++o) {
      off_ptr[o] = pos;
      off_rc[2 * o] = blocks[o].first;
      off_rc[2 * o + 1] = blocks[o].second;
      for (int32_t it : off[o]) off_items[pos++] = it;
    }
    off_ptr[blocks.size()] = pos;
  }
  return PBA_OK;
}

extern "C" int pba_assemble(const double* records, int32_t n_pairs, int32_t n_free,
                            const int32_t* diag_ptr, const int32_t* diag_items, int32_t n_off,
                            const int32_t* off_ptr, const int32_t* off_rc,
                            const int32_t* off_items, double* H, double* b, double* totals,
                            void* stream) {
  PBA_ARG_CHECK(n_free >= 0 && n_off >= 0 && n_pairs >= 0, "bad sizes");
  PBA_ARG_CHECK(totals != nullptr, "NULL totals");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_free > 0) {
    PBA_ARG_CHECK(H && b && diag_ptr && (n_off == 0 || (off_ptr && off_rc && off_items)),
                  "NULL buffer");
    const size_t dim = 6 * (size_t)n_free;
    PBA_CUDA_TRY(cudaMemsetAsync(H, 0, dim * dim * sizeof(double), st));
    const long threads = 42L * n_free + 36L * n_off;
    assemble_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
        records, n_free, diag_ptr, diag_items, n_off, off_ptr, off_rc, off_items, H, b);
    PBA_LAUNCH_CHECK();
  }
  totals_kernel<<<1, 256, 0, st>>>(records, n_pairs, totals);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

extern "C" int pba_sum_totals(const double* records, int32_t n_pairs, double* totals,
                              void* stream) {
  PBA_ARG_CHECK(totals != nullptr && n_pairs >= 0, "bad arguments");
  totals_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(records, n_pairs, totals);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}

extern "C" int pba_assemble_bsr(const double* records, int32_t n_pairs, int32_t n_free,
                                const int32_t* diag_ptr, const int32_t* diag_items, int32_t n_off,
                                const int32_t* off_ptr, const int32_t* off_items,
                                const int32_t* diag_blk, const int32_t* off_blk, double* Hb,
                                double* b, double* totals, void* stream) {
  PBA_ARG_CHECK(n_free >= 0 && n_off >= 0 && n_pairs >= 0, "bad sizes");
  PBA_ARG_CHECK(totals != nullptr, "NULL totals");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_free > 0)
    PBA_ARG_CHECK(Hb && b && diag_ptr && diag_blk && (n_off == 0 || (off_ptr && off_items &&
                                                                     off_blk)),
                  "NULL buffer");
  const long threads = n_free > 0 ? 42L * n_free + 36L * n_off : 0;  // every block written
  assemble_bsr_kernel<<<(unsigned)((threads + 255) / 256 + 1), 256, 0, st>>>(
      records, n_free, diag_ptr, diag_items, n_off, off_ptr, off_items, diag_blk, off_blk, Hb, b,
      n_pairs, totals);
  PBA_LAUNCH_CHECK();
  return PBA_OK;
}
