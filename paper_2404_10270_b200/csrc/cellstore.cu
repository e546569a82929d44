// Mover-level API on the reference's packed cell-segmented store
// (CellSortedStore, pkg/src/picmc/core.py:100-264: per cell j, live slots
// [offs[j], offs[j]+counts[j]) of packed float64 field arrays, zeroed free
// space up to offs[j]+caps[j]).
//
// These back paper_2404_10270_b200/mover.py, the twin of
// pkg/src/picmc/mover.py (push_velocity, resort_collect, commit_incomers):
//   pb_push_velocity   vx[live] += coef * E_p               (mover.py:43-54)
//   pb_resort_count    movers per cell + CFL check          (mover.py:136-148)
//   pb_resort_collect  movers out in (src_cell, src_slot) order, survivors
//                      compacted in slot order, vacated slots zeroed,
//                      counts updated                       (mover.py:149-181)
//   pb_commit_place    incomers appended per destination cell in
//                      lexsort(dest, src_cell, src_slot) order (mover.py:185-195)
//
// One warp per cell, cells grid-strided over warps (the layout's natural
// unit: a cell segment is contiguous, so a warp's loads coalesce).
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "mover.cuh"

namespace pb {

constexpr int kCsThreads = 256;
constexpr int kCsWarps = kCsThreads / 32;

static unsigned cs_grid(int64_t nc) {
  int64_t blocks = (nc + kCsWarps - 1) / kCsWarps;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

__device__ __forceinline__ unsigned lanes_below() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// push_velocity: E_p is aligned with the live order (cell-major), so cell
// j's particles read E_p[start[j] + i]; numpy's `vx[idx] += coef * e_p`
// rounds the product, then the sum.
__global__ void k_push_velocity(const double *__restrict__ e_p, double coef, double *vx,
                                const int64_t *__restrict__ offs,
                                const int64_t *__restrict__ counts,
                                const int64_t *__restrict__ start, int64_t nc) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kCsWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kCsWarps;
  for (int64_t j = w0; j < nc; j += nw) {
    const int64_t base = offs[j], o = start[j], cnt = counts[j];
    for (int64_t i = lane; i < cnt; i += 32)
      vx[base + i] = __dadd_rn(vx[base + i], __dmul_rn(coef, e_p[o + i]));
  }
}

// Movers per cell; the first CFL offender in live order (= slot order: the
// segments are laid out in cell order) is kept with atomicMin.
__global__ void k_resort_count(const double *__restrict__ x, const int64_t *__restrict__ offs,
                               const int64_t *__restrict__ counts, int64_t nc,
                               int64_t nc_global, int64_t *__restrict__ movers,
                               unsigned long long *cfl_slot) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kCsWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kCsWarps;
  for (int64_t j = w0; j < nc; j += nw) {
    const int64_t base = offs[j], cnt = counts[j];
    int64_t m = 0;
    for (int64_t i0 = 0; i0 < cnt; i0 += 32) {
      const int64_t i = i0 + lane;
      bool mv = false;
      if (i < cnt) {
        const double d = floor(x[base + i]);
        mv = d != 0.0;
        if (mv && fabs(d) >= (double)nc_global)
          atomicMin(cfl_slot, (unsigned long long)(base + i));
      }
      m += __popc(__ballot_sync(0xffffffffu, mv));
    }
    if (lane == 0) movers[j] = m;
  }
}

struct CollectArgs {
  double *f[PB_CS_MAX_FIELDS];  // f[0] = x
  double *mf[PB_CS_MAX_FIELDS];  // mover fields out
  int nf;
  const int64_t *offs;
  int64_t *counts;
  const int64_t *mover_base;  // exclusive scan of the per-cell mover counts
  int64_t nc, lo, nc_global;
  int64_t *dest, *src_cell, *src_slot;
};

// The warp walks its cell in 32-slot chunks: every lane loads its slot's
// fields before any lane stores (a survivor's new slot is never above its
// old one, and chunks are visited in order), so the compaction is in place.
__global__ void k_resort_collect(const __grid_constant__ CollectArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kCsWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kCsWarps;
  const unsigned below = lanes_below();
  for (int64_t j = w0; j < a.nc; j += nw) {
    const int64_t base = a.offs[j], cnt = a.counts[j];
    const int64_t gcell = j + a.lo;
    int64_t kept = 0, moved = 0;
    const int64_t mbase = a.mover_base[j];
    for (int64_t i0 = 0; i0 < cnt; i0 += 32) {
      const int64_t i = i0 + lane;
      const bool live = i < cnt;
      double v[PB_CS_MAX_FIELDS];
#pragma unroll
      for (int f = 0; f < PB_CS_MAX_FIELDS; ++f)
        v[f] = (live && f < a.nf) ? a.f[f][base + i] : 0.0;
      double x = v[0];
      MoveOut o{(int32_t)gcell, false, -1, false};
      if (live) o = transfer<PB_BC_PERIODIC>(x, (int32_t)gcell, a.nc_global);
      const bool mv = live && o.moved;  // CFL offenders were rejected by the count pass
      const unsigned mball = __ballot_sync(0xffffffffu, mv);
      const unsigned sball = __ballot_sync(0xffffffffu, live && !mv);
      __syncwarp();
      if (mv) {
        const int64_t p = mbase + moved + __popc(mball & below);
        a.dest[p] = o.cell;
        a.src_cell[p] = gcell;
        a.src_slot[p] = i;
        a.mf[0][p] = x;
#pragma unroll
        for (int f = 1; f < PB_CS_MAX_FIELDS; ++f)
          if (f < a.nf) a.mf[f][p] = v[f];
      } else if (live) {
        const int64_t p = base + kept + __popc(sball & below);
#pragma unroll
        for (int f = 0; f < PB_CS_MAX_FIELDS; ++f)
          if (f < a.nf) a.f[f][p] = v[f];
      }
      moved += __popc(mball);
      kept += __popc(sball);
    }
    __syncwarp();
    // vacated tail slots back to zero (core.py:103-106)
    for (int64_t i = kept + lane; i < cnt; i += 32) {
#pragma unroll
      for (int f = 0; f < PB_CS_MAX_FIELDS; ++f)
        if (f < a.nf) a.f[f][base + i] = 0.0;
    }
    if (lane == 0) a.counts[j] = kept;
  }
}

struct PlaceArgs {
  double *f[PB_CS_MAX_FIELDS];
  const double *mf[PB_CS_MAX_FIELDS];
  int nf;
  const int64_t *offs;
  const int64_t *counts;
  const int64_t *order;  // movers in lexsort(dest, src_cell, src_slot) order
  const int64_t *dest;
  const int64_t *rank;   // position within its destination cell's incomers
  int64_t n, lo;
};

__global__ void k_commit_place(const __grid_constant__ PlaceArgs a) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < a.n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = a.order[t];
    const int64_t j = a.dest[k] - a.lo;
    const int64_t p = a.offs[j] + a.counts[j] + a.rank[t];
#pragma unroll
    for (int f = 0; f < PB_CS_MAX_FIELDS; ++f)
      if (f < a.nf) a.f[f][p] = a.mf[f][k];
  }
}

// Repack a species into new per-cell offsets (capacity growth, core.py:220-240):
// live segments copied, everything else zero (the destination is pre-zeroed).
__global__ void k_repack(const double *__restrict__ src, double *__restrict__ dst,
                         const int64_t *__restrict__ offs_old,
                         const int64_t *__restrict__ offs_new,
                         const int64_t *__restrict__ counts, int64_t nc) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * kCsWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kCsWarps;
  for (int64_t j = w0; j < nc; j += nw) {
    const int64_t a = offs_old[j], b = offs_new[j], cnt = counts[j];
    for (int64_t i = lane; i < cnt; i += 32) dst[b + i] = src[a + i];
  }
}

}  // namespace pb

extern "C" size_t pb_cs_scratch_bytes(int64_t nc) {
  if (nc < 1) nc = 1;
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int64_t *)nullptr, (int64_t *)nullptr,
                                (int)(nc + 1));
  return pb::align256((size_t)(nc + 1) * sizeof(int64_t)) + pb::align256(t);
}

static int cs_scan(const int64_t *in, int64_t *out, int64_t n, void *scratch, size_t bytes,
                   cudaStream_t st) {
  size_t t = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, t, in, out, (int)n, st);
  if (e != cudaSuccess) return pb::cuda_status(e, "DeviceScan size");
  if (t > bytes) {
    pb::set_error("cell store scratch too small");
    return PB_ERR_INVALID;
  }
  e = cub::DeviceScan::ExclusiveSum(scratch, t, in, out, (int)n, st);
  if (e != cudaSuccess) return pb::cuda_status(e, "DeviceScan");
  return PB_OK;
}

extern "C" int pb_push_velocity(const double *e_p, double coef, double *vx, const int64_t *offs,
                                const int64_t *counts, int64_t nc, void *scratch,
                                size_t scratch_bytes, void *stream) {
  if (nc < 0 || (nc > 0 && (!vx || !offs || !counts || !scratch))) {
    pb::set_error("pb_push_velocity: bad arguments");
    return PB_ERR_INVALID;
  }
  if (nc == 0) return PB_OK;
  if (scratch_bytes < pb_cs_scratch_bytes(nc)) {
    pb::set_error("pb_push_velocity: scratch too small");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int64_t *start = (int64_t *)scratch;
  const size_t head = pb::align256((size_t)(nc + 1) * sizeof(int64_t));
  int rc = cs_scan(counts, start, nc, (char *)scratch + head, scratch_bytes - head, st);
  if (rc) return rc;
  pb::k_push_velocity<<<pb::cs_grid(nc), pb::kCsThreads, 0, st>>>(e_p, coef, vx, offs, counts,
                                                                  start, nc);
  PB_CHECK_LAUNCH("k_push_velocity");
  return PB_OK;
}

extern "C" int pb_resort_count(const double *x, const int64_t *offs, const int64_t *counts,
                               int64_t nc, int64_t nc_global, int64_t *mover_counts,
                               int64_t *mover_base, uint64_t *cfl_slot, void *scratch,
                               size_t scratch_bytes, void *stream) {
  if (nc < 0 || nc_global < 1 || (nc > 0 && (!x || !offs || !counts || !mover_counts ||
                                             !mover_base || !cfl_slot || !scratch))) {
    pb::set_error("pb_resort_count: bad arguments");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(cfl_slot, 0xff, sizeof(uint64_t), st);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaMemsetAsync");
  e = cudaMemsetAsync(mover_counts, 0, (size_t)(nc + 1) * sizeof(int64_t), st);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaMemsetAsync");
  if (nc > 0) {
    pb::k_resort_count<<<pb::cs_grid(nc), pb::kCsThreads, 0, st>>>(
        x, offs, counts, nc, nc_global, mover_counts, (unsigned long long *)cfl_slot);
    PB_CHECK_LAUNCH("k_resort_count");
  }
  // mover_counts has nc+1 entries (the last one zero): base[nc] = total
  return cs_scan(mover_counts, mover_base, nc + 1, scratch, scratch_bytes, st);
}

extern "C" int pb_resort_collect(const pb_cell_fields *s, const pb_movers *m, int64_t lo,
                                 int64_t nc_global, const int64_t *mover_base, void *stream) {
  if (!s || !m || s->nf < 1 || s->nf > PB_CS_MAX_FIELDS || s->nc < 0 || nc_global < 1) {
    pb::set_error("pb_resort_collect: bad arguments");
    return PB_ERR_INVALID;
  }
  if (s->nc == 0) return PB_OK;
  pb::CollectArgs a;
  a.nf = s->nf;
  for (int f = 0; f < PB_CS_MAX_FIELDS; ++f) {
    a.f[f] = f < s->nf ? s->field[f] : nullptr;
    a.mf[f] = f < s->nf ? m->field[f] : nullptr;
  }
  a.offs = s->offs;
  a.counts = s->counts;
  a.mover_base = mover_base;
  a.nc = s->nc;
  a.lo = lo;
  a.nc_global = nc_global;
  a.dest = m->dest;
  a.src_cell = m->src_cell;
  a.src_slot = m->src_slot;
  pb::k_resort_collect<<<pb::cs_grid(s->nc), pb::kCsThreads, 0, (cudaStream_t)stream>>>(a);
  PB_CHECK_LAUNCH("k_resort_collect");
  return PB_OK;
}

extern "C" int pb_commit_place(const pb_cell_fields *s, const pb_movers *m, const int64_t *order,
                               const int64_t *rank, int64_t n, int64_t lo, void *stream) {
  if (!s || !m || s->nf < 1 || s->nf > PB_CS_MAX_FIELDS || n < 0 ||
      (n > 0 && (!order || !rank || !m->dest))) {
    pb::set_error("pb_commit_place: bad arguments");
    return PB_ERR_INVALID;
  }
  if (n == 0) return PB_OK;
  pb::PlaceArgs a;
  a.nf = s->nf;
  for (int f = 0; f < PB_CS_MAX_FIELDS; ++f) {
    a.f[f] = f < s->nf ? s->field[f] : nullptr;
    a.mf[f] = f < s->nf ? m->field[f] : nullptr;
  }
  a.offs = s->offs;
  a.counts = s->counts;
  a.order = order;
  a.dest = m->dest;
  a.rank = rank;
  a.n = n;
  a.lo = lo;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  pb::k_commit_place<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a);
  PB_CHECK_LAUNCH("k_commit_place");
  return PB_OK;
}

extern "C" int pb_repack(const double *src, double *dst, const int64_t *offs_old,
                         const int64_t *offs_new, const int64_t *counts, int64_t nc,
                         void *stream) {
  if (nc < 0 || (nc > 0 && (!src || !dst || !offs_old || !offs_new || !counts))) {
    pb::set_error("pb_repack: bad arguments");
    return PB_ERR_INVALID;
  }
  if (nc == 0) return PB_OK;
  pb::k_repack<<<pb::cs_grid(nc), pb::kCsThreads, 0, (cudaStream_t)stream>>>(
      src, dst, offs_old, offs_new, counts, nc);
  PB_CHECK_LAUNCH("k_repack");
  return PB_OK;
}
