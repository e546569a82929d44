// Periodic sort by cell and absorbing-wall compaction.
//
// The reference keeps particles "naturally sorted" in per-cell segments and
// pays for it every step in resort/commit (pkg/src/picmc/mover.py:113-195,
// pkg/src/picmc/core.py:192-240: ~133 ns/particle on the CPU).  The flat
// device store instead carries a cell index per particle and restores cell
// order only every S steps: a stable LSD radix sort of (cell, slot) over
// ceil(log2 nc) bits, then one gather pass that permutes every field into
// the ping-pong buffers.  Particle state is unchanged by the sort, and the
// fixed-point deposit is order independent, so physics is bitwise identical
// for any sort period.
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace pb {

static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

static int key_bits(int64_t nc) {
  int b = 1;
  while (b < 31 && ((int64_t)1 << b) < nc) ++b;
  return b;
}

__global__ void k_iota(uint32_t *v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)i;
}

struct PermArgs {
  const double *src[5];
  double *dst[5];
  int nf;
};

__global__ void k_permute(PermArgs pa, const uint32_t *__restrict__ perm,
                          int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[i];
#pragma unroll
    for (int f = 0; f < 5; ++f)
      if (f < pa.nf) pa.dst[f][i] = __ldg(pa.src[f] + p);
  }
}

static size_t radix_temp_bytes(int64_t n, int64_t nc) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint32_t *)nullptr,
                                  (uint32_t *)nullptr, (const uint32_t *)nullptr,
                                  (uint32_t *)nullptr, (int)(n > 0 ? n : 1), 0,
                                  key_bits(nc));
  return t;
}

// ---- absorbing-wall compaction -------------------------------------------
constexpr int kCompactThreads = 1024;

struct CompactArgs {
  pb_species sp[PB_MAX_SPECIES];
  int id[PB_MAX_SPECIES];
  int nsp;
  int64_t *tail;  // scratch: per species, cap entries
  int64_t tail_stride;
  pb_status *st;
};

// One block per species: the survivors in the tail [n-k, n) fill the holes
// below n-k.  Tail survivors are enumerated in slot order with a block scan
// over warp ballots; holes are consumed through a cursor.
__global__ void __launch_bounds__(kCompactThreads)
    k_compact(const __grid_constant__ CompactArgs a) {
  using Scan = cub::BlockScan<int, kCompactThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t s_cnt;
  __shared__ unsigned long long s_cursor;
  const int isp = blockIdx.x;
  if (isp >= a.nsp) return;
  const pb_species &s = a.sp[isp];
  const int sid = a.id[isp];
  const int64_t n = *s.n_dev;
  const int64_t k = a.st->n_holes[sid];
  if (k <= 0) return;
  const int64_t n2 = n - k;
  int64_t *tail = a.tail + (size_t)isp * a.tail_stride;
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_cursor = 0;
  }
  __syncthreads();
  for (int64_t b = n2; b < n; b += kCompactThreads) {
    const int64_t i = b + threadIdx.x;
    const int alive = (i < n && s.cell[i] >= 0) ? 1 : 0;
    int pos, total;
    Scan(tmp).ExclusiveSum(alive, pos, total);
    if (alive) tail[s_cnt + pos] = i;
    __syncthreads();
    if (threadIdx.x == 0) s_cnt += total;
    __syncthreads();
  }
  for (int64_t j = threadIdx.x; j < k; j += kCompactThreads) {
    const int64_t h = s.holes[j];
    if (h >= n2) continue;
    const unsigned long long t = atomicAdd(&s_cursor, 1ull);
    const int64_t src = tail[t];
    s.x[h] = s.x[src];
    s.vx[h] = s.vx[src];
    s.vy[h] = s.vy[src];
    s.vz[h] = s.vz[src];
    if (s.yp) s.yp[h] = s.yp[src];
    s.cell[h] = s.cell[src];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *s.n_dev = n2;
    a.st->n_holes[sid] = 0;
  }
}

}  // namespace pb

extern "C" size_t pb_sort_scratch_bytes(int64_t n, int64_t nc) {
  if (n < 1) n = 1;
  return 2 * pb::align256((size_t)n * sizeof(uint32_t)) +
         pb::align256(pb::radix_temp_bytes(n, nc));
}

extern "C" int pb_sort_by_cell(const pb_species *src, const pb_species *dst,
                               int64_t nc, void *scratch, size_t scratch_bytes,
                               void *stream) {
  if (!src || !dst) {
    pb::set_error("pb_sort_by_cell: NULL species");
    return PB_ERR_INVALID;
  }
  const int64_t n = src->n;
  if (n <= 0) return PB_OK;
  if (n > 0x7fffffffLL || nc < 1 || nc > 0x7fffffffLL) {
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
  uint32_t *iota = (uint32_t *)p;
  p += pb::align256((size_t)n * sizeof(uint32_t));
  uint32_t *perm = (uint32_t *)p;
  p += pb::align256((size_t)n * sizeof(uint32_t));
  size_t tb = pb::radix_temp_bytes(n, nc);
  pb::k_iota<<<148 * 8, 256, 0, st>>>(iota, n);
  PB_CHECK_LAUNCH("k_iota");
  cudaError_t e = cub::DeviceRadixSort::SortPairs(
      p, tb, (const uint32_t *)src->cell, (uint32_t *)dst->cell, iota, perm,
      (int)n, 0, pb::key_bits(nc), st);
  if (e != cudaSuccess) return pb::cuda_status(e, "DeviceRadixSort::SortPairs");
  pb::PermArgs pa;
  int nf = 0;
  pa.src[nf] = src->x; pa.dst[nf++] = dst->x;
  pa.src[nf] = src->vx; pa.dst[nf++] = dst->vx;
  pa.src[nf] = src->vy; pa.dst[nf++] = dst->vy;
  pa.src[nf] = src->vz; pa.dst[nf++] = dst->vz;
  if (src->yp && dst->yp) {
    pa.src[nf] = src->yp;
    pa.dst[nf++] = dst->yp;
  }
  pa.nf = nf;
  pb::k_permute<<<148 * 8, 256, 0, st>>>(pa, perm, n);
  PB_CHECK_LAUNCH("k_permute");
  return PB_OK;
}

extern "C" size_t pb_compact_scratch_bytes(int64_t n) {
  if (n < 1) n = 1;
  return (size_t)PB_MAX_SPECIES * (size_t)n * sizeof(int64_t);
}

extern "C" int pb_compact(const pb_species *sp, int nsp, pb_status *status,
                          void *scratch, size_t scratch_bytes, void *stream) {
  if (nsp < 0 || nsp > PB_MAX_SPECIES || !status) {
    pb::set_error("pb_compact: bad arguments");
    return PB_ERR_INVALID;
  }
  pb::CompactArgs a;
  memset(&a, 0, sizeof(a));
  int64_t nmax = 1;
  for (int k = 0; k < nsp; ++k) {
    if (sp[k].kind == PB_KIND_INACTIVE || sp[k].n <= 0) continue;
    if (!sp[k].n_dev || !sp[k].holes) {
      pb::set_error("pb_compact: species %d lacks n_dev/holes", k);
      return PB_ERR_INVALID;
    }
    a.sp[a.nsp] = sp[k];
    a.id[a.nsp] = k;
    a.nsp++;
    if (sp[k].n > nmax) nmax = sp[k].n;
  }
  if (a.nsp == 0) return PB_OK;
  if (!scratch || scratch_bytes < (size_t)a.nsp * (size_t)nmax * sizeof(int64_t)) {
    pb::set_error("pb_compact: scratch too small");
    return PB_ERR_INVALID;
  }
  a.tail = (int64_t *)scratch;
  a.tail_stride = nmax;
  a.st = status;
  pb::k_compact<<<a.nsp, pb::kCompactThreads, 0, (cudaStream_t)stream>>>(a);
  PB_CHECK_LAUNCH("k_compact");
  return PB_OK;
}
