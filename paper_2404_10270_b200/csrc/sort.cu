// Periodic sort by cell and absorbing-wall compaction.
//
// The reference keeps particles "naturally sorted" in per-cell segments and
// pays for it every step in resort/commit (pkg/src/picmc/mover.py:113-195,
// pkg/src/picmc/core.py:192-240: ~133 ns/particle on the CPU).  The flat
// device store instead carries a cell index per particle and restores cell
// order only every S steps with a counting sort: a cell histogram
// (warp-aggregated atomics), an exclusive scan into per-cell cursors, and one
// scatter pass that writes every field to its cell's range of the ping-pong
// buffers (lanes of a warp sharing a cell take consecutive slots, so the
// writes of nearly-sorted data stay coalesced).  Order within a cell is
// arbitrary; particle state is unchanged by the sort and the fixed-point
// deposit is order independent, so physics is bitwise identical for any sort
// period.  ~0.8 GB of traffic for 10M electrons, vs ~1.7 GB for the LSD
// radix sort + gather it replaced.
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "compact.cuh"

#include <cstring>

namespace pb {

static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Per-cell counts; lanes holding the same cell add once per warp.
// n_dev (absorbing species): the live count on device, bounded by n, so the
// sort needs no host read of it.
__device__ __forceinline__ int64_t live_n(int64_t n, const int64_t *n_dev) {
  if (!n_dev) return n;
  const int64_t m = *n_dev;
  return m < n ? m : n;
}

__global__ void k_cell_count(const int32_t *__restrict__ cell, int64_t n, const int64_t *n_dev,
                             uint32_t *counts) {
  n = live_n(n, n_dev);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < n; b += stride) {
    const int64_t i = b + threadIdx.x;
    const int32_t c = i < n ? __ldg(cell + i) : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    if (c >= 0 && (threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1))
      atomicAdd(&counts[c], (uint32_t)__popc(grp));
  }
}

struct ScatterArgs {
  const double *src[5];
  double *dst[5];
  int nf;
  const int32_t *cell;
  int32_t *cell_out;
  uint32_t *cursor;
  int64_t n;
  const int64_t *n_dev;
};

__global__ void k_cell_scatter(const __grid_constant__ ScatterArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const unsigned lane = threadIdx.x & 31;
  const int64_t n = live_n(a.n, a.n_dev);
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < n; b += stride) {
    const int64_t i = b + threadIdx.x;
    const int32_t c = i < n ? __ldg(a.cell + i) : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    const unsigned leader = (unsigned)(__ffs(grp) - 1);
    uint32_t base = 0;
    if (c >= 0 && lane == leader) base = atomicAdd(&a.cursor[c], (uint32_t)__popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (c < 0) continue;
    const uint32_t pos = base + (uint32_t)__popc(grp & lanemask_lt());
#pragma unroll
    for (int f = 0; f < 5; ++f)
      if (f < a.nf) a.dst[f][pos] = __ldg(a.src[f] + i);
    a.cell_out[pos] = c;
  }
}


// chunk_base = first cell of each PB_CELL8_CHUNK-slot chunk minus a margin
// (cell-sorted chunks then fit in int8 offsets with room for drift);
// cell8 = cell - chunk_base or the escape.
__global__ void k_cell8_build(const int32_t *__restrict__ cell, int64_t n,
                              int8_t *__restrict__ cell8, int32_t *__restrict__ chunk_base) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c0 = (i / PB_CELL8_CHUNK) * PB_CELL8_CHUNK;
    const int32_t first = __ldg(cell + c0);
    const int32_t base = (first >= 0 ? first : 0) - PB_CELL8_MARGIN;
    if (i == c0) chunk_base[i / PB_CELL8_CHUNK] = base;
    cell8[i] = cell8_of(cell[i], base);
  }
}

static size_t scan_temp_bytes(int64_t nc) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                (int)nc);
  return t;
}

// ---- absorbing-wall compaction (compact.cuh) -------------------------------
constexpr int kCompactThreads = 1024;

__global__ void __launch_bounds__(kCompactThreads)
    k_compact(const __grid_constant__ CompactArgs a) {
  pdl_enter();
  __shared__ CompactSmem<kCompactThreads> sm;
  if ((int)blockIdx.x < a.nsp) compact_species<kCompactThreads>(a, blockIdx.x, sm);
}

int compact_args(const pb_species *sp, int nsp, pb_status *status, void *scratch, size_t scratch_bytes,
                 CompactArgs &a) {
  memset(&a, 0, sizeof(a));
  if (nsp < 0 || nsp > PB_MAX_SPECIES || !status) {
    set_error("pb_compact: bad arguments");
    return PB_ERR_INVALID;
  }
  int64_t nmax = 1;
  for (int k = 0; k < nsp; ++k) {
    if (sp[k].kind == PB_KIND_INACTIVE || sp[k].n <= 0) continue;
    if (!sp[k].n_dev || !sp[k].holes) {
      set_error("pb_compact: species %d lacks n_dev/holes", k);
      return PB_ERR_INVALID;
    }
    a.sp[a.nsp] = sp[k];
    a.id[a.nsp] = k;
    a.nsp++;
    if (sp[k].n > nmax) nmax = sp[k].n;
  }
  if (a.nsp == 0) return PB_OK;
  if (!scratch || scratch_bytes < (size_t)a.nsp * (size_t)nmax * sizeof(int64_t)) {
    set_error("pb_compact: scratch too small");
    return PB_ERR_INVALID;
  }
  a.tail = (int64_t *)scratch;
  a.tail_stride = nmax;
  a.st = status;
  return PB_OK;
}

}  // namespace pb

extern "C" size_t pb_sort_scratch_bytes(int64_t n, int64_t nc) {
  (void)n;
  if (nc < 1) nc = 1;
  return 2 * pb::align256((size_t)nc * sizeof(uint32_t)) + pb::align256(pb::scan_temp_bytes(nc));
}

extern "C" int pb_sort_by_cell(const pb_species *src, const pb_species *dst, int64_t nc,
                               void *scratch, size_t scratch_bytes, void *stream) {
  if (!src || !dst) {
    pb::set_error("pb_sort_by_cell: NULL species");
    return PB_ERR_INVALID;
  }
  const int64_t n = src->n;
  if (n <= 0) return PB_OK;
  if (n > 0xffffffffLL || nc < 1 || nc > 0x7fffffffLL) {
    pb::set_error("pb_sort_by_cell: n=%lld nc=%lld out of range", (long long)n,
                  (long long)nc);
    return PB_ERR_INVALID;
  }
  if (scratch_bytes < pb_sort_scratch_bytes(n, nc) || !scratch) {
    pb::set_error("pb_sort_by_cell: scratch too small");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char *p = (char *)scratch;
  uint32_t *counts = (uint32_t *)p;
  p += pb::align256((size_t)nc * sizeof(uint32_t));
  uint32_t *cursor = (uint32_t *)p;
  p += pb::align256((size_t)nc * sizeof(uint32_t));
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)nc * sizeof(uint32_t), st);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaMemsetAsync");
  pb::k_cell_count<<<148 * 8, 256, 0, st>>>(src->cell, n, src->n_dev, counts);
  PB_CHECK_LAUNCH("k_cell_count");
  size_t tb = pb::scan_temp_bytes(nc);
  e = cub::DeviceScan::ExclusiveSum(p, tb, counts, cursor, (int)nc, st);
  if (e != cudaSuccess) return pb::cuda_status(e, "DeviceScan::ExclusiveSum");
  pb::ScatterArgs a;
  int nf = 0;
  a.src[nf] = src->x; a.dst[nf++] = dst->x;
  a.src[nf] = src->vx; a.dst[nf++] = dst->vx;
  a.src[nf] = src->vy; a.dst[nf++] = dst->vy;
  a.src[nf] = src->vz; a.dst[nf++] = dst->vz;
  if (src->yp && dst->yp) {
    a.src[nf] = src->yp;
    a.dst[nf++] = dst->yp;
  }
  a.nf = nf;
  a.cell = src->cell;
  a.cell_out = dst->cell;
  a.cursor = cursor;
  a.n = n;
  a.n_dev = src->n_dev;
  pb::k_cell_scatter<<<148 * 8, 256, 0, st>>>(a);
  PB_CHECK_LAUNCH("k_cell_scatter");
  return PB_OK;
}

extern "C" size_t pb_compact_scratch_bytes(int64_t n) {
  if (n < 1) n = 1;
  return (size_t)PB_MAX_SPECIES * (size_t)n * sizeof(int64_t);
}

extern "C" int pb_compact(const pb_species *sp, int nsp, pb_status *status,
                          void *scratch, size_t scratch_bytes, void *stream) {
  pb::CompactArgs a;
  const int rc = pb::compact_args(sp, nsp, status, scratch, scratch_bytes, a);
  if (rc || a.nsp == 0) return rc;
  cudaError_t le = pb::launch_pdl(pb::k_compact, dim3(a.nsp), dim3(pb::kCompactThreads), 0,
                                  (cudaStream_t)stream, a);
  if (le != cudaSuccess) return pb::cuda_status(le, "k_compact");
  PB_CHECK_LAUNCH("k_compact");
  return PB_OK;
}

extern "C" int pb_cell8_build(const pb_species *sp, void *stream) {
  if (!sp || !sp->cell) {
    pb::set_error("pb_cell8_build: NULL species/cell");
    return PB_ERR_INVALID;
  }
  if (!sp->cell8 || !sp->chunk_base || sp->n <= 0) return PB_OK;
  pb::k_cell8_build<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(sp->cell, sp->n, sp->cell8,
                                                                sp->chunk_base);
  PB_CHECK_LAUNCH("k_cell8_build");
  return PB_OK;
}
