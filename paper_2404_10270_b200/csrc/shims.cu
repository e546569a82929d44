// Parity shims with the reference kernel signatures, on the reference's own
// packed cell-sorted layout (per-cell segments addressed by offs/counts,
// pkg/src/picmc/core.py:100-132).  These let `picmc.backends`-style callers
// (and the reference's test_backends.py comparisons) run on the GPU; the
// engine itself uses the flat layout of push_deposit.cu.
//
// One warp per cell: lanes stride the cell's live slots (coalesced within
// the segment); cells are grid-strided over warps.
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace pb {

constexpr int kShimThreads = 256;
constexpr int kWarps = kShimThreads / 32;

// fused_move (pkg/src/picmc/backends/_kernels.pyx:60-102).
__global__ void k_fused_move(const double *__restrict__ accel, double *x,
                             double *vx, const double *__restrict__ vy,
                             double *yp, const int64_t *__restrict__ offs,
                             const int64_t *__restrict__ counts, int64_t nc,
                             double fnstep) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t j = w0; j < nc; j += nw) {
    const int64_t base = offs[j];
    const int64_t cnt = counts[j];
    double aj = 0.0, daj = 0.0;
    if (accel) {
      aj = accel[j];
      daj = __dsub_rn(accel[j + 1], aj);
    }
    for (int64_t i = lane; i < cnt; i += 32) {
      const int64_t k = base + i;
      double v;
      if (accel) {
        const double atemp = __dadd_rn(aj, __dmul_rn(x[k], daj));
        v = __dadd_rn(vx[k], atemp);
        vx[k] = v;
      } else {
        v = vx[k];
      }
      x[k] = __dadd_rn(x[k], __dmul_rn(fnstep, v));
      if (yp) yp[k] = __dadd_rn(yp[k], __dmul_rn(fnstep, vy[k]));
    }
  }
}

// deposit_partials (_kernels.pyx:14-34): strictly sequential per cell in
// slot order, so the result is bitwise the reference's.  One thread per
// cell: the sequential add chain is the
// latency, so 32 cells per warp in flight (loads issued four ahead) beat a
// warp replaying one cell's chain.
__global__ void k_deposit_partials_tpc(const double *__restrict__ x,
                                       const int64_t *__restrict__ offs,
                                       const int64_t *__restrict__ counts, int64_t nc,
                                       double *__restrict__ left, double *__restrict__ right) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double *p = x + offs[j];
    const int64_t cnt = counts[j];
    double sl = 0.0, sr = 0.0;
    int64_t k = 0;
    for (; k + 4 <= cnt; k += 4) {
      const double a = p[k], b = p[k + 1], c = p[k + 2], d = p[k + 3];
      sl = __dadd_rn(sl, __dsub_rn(1.0, a));
      sr = __dadd_rn(sr, a);
      sl = __dadd_rn(sl, __dsub_rn(1.0, b));
      sr = __dadd_rn(sr, b);
      sl = __dadd_rn(sl, __dsub_rn(1.0, c));
      sr = __dadd_rn(sr, c);
      sl = __dadd_rn(sl, __dsub_rn(1.0, d));
      sr = __dadd_rn(sr, d);
    }
    for (; k < cnt; ++k) {
      const double a = p[k];
      sl = __dadd_rn(sl, __dsub_rn(1.0, a));
      sr = __dadd_rn(sr, a);
    }
    left[j] = sl;
    right[j] = sr;
  }
}

// gather (_kernels.pyx:37-57): live order output, start[j] = sum(counts[:j]).
__global__ void k_gather(const double *__restrict__ nodes,
                         const double *__restrict__ x,
                         const int64_t *__restrict__ offs,
                         const int64_t *__restrict__ counts,
                         const int64_t *__restrict__ start, int64_t nc,
                         double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t j = w0; j < nc; j += nw) {
    const int64_t base = offs[j];
    const int64_t cnt = counts[j];
    const int64_t o = start[j];
    const double aj = nodes[j];
    const double daj = __dsub_rn(nodes[j + 1], aj);
    for (int64_t i = lane; i < cnt; i += 32)
      out[o + i] = __dadd_rn(aj, __dmul_rn(x[base + i], daj));
  }
}

static unsigned shim_grid(int64_t nc) {
  int64_t blocks = (nc + kWarps - 1) / kWarps;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

// fused_move_aos / fused_move_table (pkg/src/picmc/backends/_kernels.pyx:105-152):
// the same arithmetic on a row-major table with columns x, vx, vy, vz[, yp].
__global__ void k_fused_move_aos(double *tab, int64_t ncols, const int64_t *__restrict__ starts,
                                 const int64_t *__restrict__ counts, int64_t nc,
                                 const double *__restrict__ accel, double fnstep, int has_yp) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t j = w0; j < nc; j += nw) {
    const int64_t base = starts[j];
    const int64_t cnt = counts[j];
    double aj = 0.0, daj = 0.0;
    if (accel) {
      aj = accel[j];
      daj = __dsub_rn(accel[j + 1], aj);
    }
    for (int64_t i = lane; i < cnt; i += 32) {
      double *r = tab + (base + i) * ncols;
      double v;
      if (accel) {
        const double atemp = __dadd_rn(aj, __dmul_rn(r[0], daj));
        v = __dadd_rn(r[1], atemp);
        r[1] = v;
      } else {
        v = r[1];
      }
      r[0] = __dadd_rn(r[0], __dmul_rn(fnstep, v));
      if (has_yp) r[4] = __dadd_rn(r[4], __dmul_rn(fnstep, r[2]));
    }
  }
}

}  // namespace pb

extern "C" int pb_fused_move(const double *accel_or_null, double *x,
                             double *vx, const double *vy, double *yp_or_null,
                             const int64_t *offs, const int64_t *counts,
                             int64_t nc, double fnstep, void *stream) {
  if (nc < 0) {
    pb::set_error("nc=%lld must be >= 0", (long long)nc);
    return PB_ERR_INVALID;
  }
  if (nc == 0) return PB_OK;
  if (!x || !vx || !offs || !counts || (yp_or_null && !vy)) {
    pb::set_error("pb_fused_move: NULL array argument");
    return PB_ERR_INVALID;
  }
  pb::k_fused_move<<<pb::shim_grid(nc), pb::kShimThreads, 0, (cudaStream_t)stream>>>(
      accel_or_null, x, vx, vy, yp_or_null, offs, counts, nc, fnstep);
  PB_CHECK_LAUNCH("k_fused_move");
  return PB_OK;
}

extern "C" int pb_deposit_partials(const double *x, const int64_t *offs,
                                   const int64_t *counts, int64_t nc,
                                   double *left, double *right, void *stream) {
  if (nc < 0) {
    pb::set_error("nc=%lld must be >= 0", (long long)nc);
    return PB_ERR_INVALID;
  }
  if (nc == 0) return PB_OK;
  if (!offs || !counts || !left || !right) {
    pb::set_error("pb_deposit_partials: NULL array argument");
    return PB_ERR_INVALID;
  }
  int64_t blocks = (nc + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  pb::k_deposit_partials_tpc<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      x, offs, counts, nc, left, right);
  PB_CHECK_LAUNCH("k_deposit_partials_tpc");
  return PB_OK;
}

extern "C" int pb_gather(const double *nodes, const double *x,
                         const int64_t *offs, const int64_t *counts, int64_t nc,
                         double *out, void *stream) {
  if (nc < 0) {
    pb::set_error("nc=%lld must be >= 0", (long long)nc);
    return PB_ERR_INVALID;
  }
  if (nc == 0) return PB_OK;
  if (!nodes || !offs || !counts) {
    pb::set_error("pb_gather: NULL array argument");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts,
                                                (int64_t *)nullptr, (int)nc, st);
  if (e != cudaSuccess) return pb::cuda_status(e, "DeviceScan size");
  void *buf = nullptr;
  const size_t start_bytes = ((size_t)nc * sizeof(int64_t) + 255) & ~(size_t)255;
  e = cudaMallocAsync(&buf, start_bytes + tmp_bytes, st);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaMallocAsync");
  int64_t *start = (int64_t *)buf;
  void *tmp = (char *)buf + start_bytes;
  e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, start, (int)nc, st);
  if (e != cudaSuccess) {
    cudaFreeAsync(buf, st);
    return pb::cuda_status(e, "DeviceScan");
  }
  pb::k_gather<<<pb::shim_grid(nc), pb::kShimThreads, 0, st>>>(nodes, x, offs, counts,
                                                              start, nc, out);
  cudaError_t le = cudaGetLastError();
  cudaFreeAsync(buf, st);
  if (le != cudaSuccess) return pb::cuda_status(le, "k_gather");
  return PB_OK;
}

extern "C" int pb_fused_move_aos(double *tab, int64_t ncols, const int64_t *starts,
                                 const int64_t *counts, int64_t nc, const double *accel_or_null,
                                 double fnstep, int has_yp, void *stream) {
  if (nc < 0 || (nc > 0 && (!tab || !starts || !counts)) || ncols < (has_yp ? 5 : 4)) {
    pb::set_error("pb_fused_move_aos: bad arguments (ncols=%lld)", (long long)ncols);
    return PB_ERR_INVALID;
  }
  if (nc == 0) return PB_OK;
  int64_t blocks = (nc + pb::kWarps - 1) / pb::kWarps;
  if (blocks > 148 * 32) blocks = 148 * 32;
  pb::k_fused_move_aos<<<(unsigned)blocks, pb::kShimThreads, 0, (cudaStream_t)stream>>>(
      tab, ncols, starts, counts, nc, accel_or_null, fnstep, has_yp);
  PB_CHECK_LAUNCH("k_fused_move_aos");
  return PB_OK;
}
