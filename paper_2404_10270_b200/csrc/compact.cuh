// Absorbing-wall compaction (config 3 extension; the reference always wraps,
// pkg/src/picmc/mover.py:156): the survivors in the tail [n-k, n) of a
// species fill the k holes the mover recorded below n-k.  Shared by the
// standalone k_compact (sort.cu) and the compaction blocks of the
// single-launch field step (k_field_fused, fields.cu), which fills the
// previous step's holes in the same launch.
#pragma once

#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace pb {

struct CompactArgs {
  pb_species sp[PB_MAX_SPECIES];
  int id[PB_MAX_SPECIES];
  int nsp;
  int64_t *tail;  // scratch: per species, tail_stride entries
  int64_t tail_stride;
  pb_status *st;
};

__device__ __forceinline__ int8_t cell8_of(int32_t cell, int32_t base) {
  const int32_t d = cell - base;
  return (cell >= 0 && d > PB_CELL8_ESCAPE && d <= 127) ? (int8_t)d : (int8_t)PB_CELL8_ESCAPE;
}

template <int NT>
struct CompactSmem {
  typename cub::BlockScan<int, NT>::TempStorage scan;
  int64_t cnt;
  unsigned long long cursor;
};

// One block of NT threads per species slot isp: tail survivors are
// enumerated in slot order with a block scan, holes consumed through a
// shared cursor (the pairing order is free: stores compare as multisets).
template <int NT>
__device__ void compact_species(const CompactArgs &a, int isp, CompactSmem<NT> &sm) {
  using Scan = cub::BlockScan<int, NT>;
  const pb_species &s = a.sp[isp];
  const int sid = a.id[isp];
  const int64_t n = *s.n_dev;
  const int64_t k = a.st->n_holes[sid];
  if (k <= 0) return;  // uniform across the block
  const int64_t n2 = n - k;
  int64_t *tail = a.tail + (size_t)isp * a.tail_stride;
  if (threadIdx.x == 0) {
    sm.cnt = 0;
    sm.cursor = 0;
  }
  __syncthreads();
  for (int64_t b = n2; b < n; b += NT) {
    const int64_t i = b + threadIdx.x;
    const int alive = (i < n && s.cell[i] >= 0) ? 1 : 0;
    int pos, total;
    Scan(sm.scan).ExclusiveSum(alive, pos, total);
    if (alive) tail[sm.cnt + pos] = i;
    __syncthreads();
    if (threadIdx.x == 0) sm.cnt += total;
    __syncthreads();
  }
  for (int64_t j = threadIdx.x; j < k; j += NT) {
    const int64_t h = s.holes[j];
    if (h >= n2) continue;
    const unsigned long long t = atomicAdd(&sm.cursor, 1ull);
    const int64_t src = tail[t];
    s.x[h] = s.x[src];
    s.vx[h] = s.vx[src];
    s.vy[h] = s.vy[src];
    s.vz[h] = s.vz[src];
    if (s.yp) s.yp[h] = s.yp[src];
    s.cell[h] = s.cell[src];
    if (s.cell8) s.cell8[h] = cell8_of(s.cell[src], s.chunk_base[h / PB_CELL8_CHUNK]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *s.n_dev = n2;
    a.st->n_holes[sid] = 0;
  }
}

// Host: fill CompactArgs from the species that take part (active, n > 0,
// absorbing: n_dev and holes set).  Returns PB_OK, or PB_ERR_INVALID with
// the error text set.
int compact_args(const pb_species *sp, int nsp, pb_status *status, void *scratch, size_t scratch_bytes,
                 CompactArgs &a);

}  // namespace pb
