// Multi-GPU density exchange fused with the density epilogue, over peer
// memory (NVLink 5 / NVSwitch on a B200 node; CUDA IPC mappings between the
// per-GPU processes).
//
// The reference stitches worker density pieces with fixed-order seam sums
// (pkg/src/picmc/decomposition.py:147-174, harness.py:97-102); the NCCL path
// of this engine all-reduces the fixed-point bins and then runs the epilogue.
// Here one kernel does both: every rank owns a contiguous slice of the nodes,
// sums the bins of its slice (and one halo cell) straight out of every
// rank's memory -- integer adds, so the reduction is exact and order free --,
// turns them into left/right/rho with the epilogue arithmetic and stores its
// slice into every rank's left/right/rho buffers.  Net NVLink traffic per
// rank and step: the bins once (reduce-scatter volume) plus 1/N of the
// outputs to each peer (all-gather volume), with no separate collective
// launch and no host synchronisation.
//
// Cross-GPU ordering uses flag words in each rank's memory (system-scope
// release stores / acquire loads, monotonically increasing epochs):
//   A  arrive   -- every rank's bins of this step are final (the kernel runs
//                  after the rank's push on its stream);
//   B  done     -- every block of every rank has read the bins and written
//                  its slice: the own bins may be cleared and rho is
//                  complete on every rank.
// The grid is persistent (<= resident capacity, checked at launch) so that
// every block of every rank can reach the barriers.  Waits are bounded by a
// wall-clock timeout (%globaltimer; pb_peer_density.timeout_ns, default
// 60 s).  A rank that times out publishes the failing epoch in the error word
// of EVERY rank's flag block, sets PB_ERR_PEER in its status and leaves its
// bins alone; every rank polls its own error word inside its waits, so all
// ranks -- including one that arrives after the timeout -- flag the step
// PB_ERR_PEER instead of computing rho from bins a peer may already have
// cleared.  The error is sticky for the run: every later exchange fails too.
#include <cstring>

#include "common.cuh"

namespace pb {

// 64-thread blocks, at most one per SM: small enough (2.5K registers) to be
// co-resident with the persistent mover (3 x 256 threads x 80 registers =
// 61K of the SM's 64K), so in field-free steps the exchange runs beside the
// push instead of waiting for SM slots in its tail.
constexpr int kPeerThreads = 64;
constexpr int kErrWord = 2 * PB_MAX_RANKS;  // index of the error word in a flag block

struct PeerArgs {
  const uint64_t *bins[PB_MAX_RANKS];
  double *left[PB_MAX_RANKS], *right[PB_MAX_RANKS], *rho[PB_MAX_RANKS];
  unsigned long long *flags[PB_MAX_RANKS];  // [0, N): arrive epochs, [N, 2N): done counts,
                                            // [kErrWord]: first failed epoch (0 = none)
  uint64_t *clear_next;
  double coef[PB_MAX_SPECIES];
  int ndep, rank, world, field_bc;
  int64_t nc;
  unsigned long long epoch;
  const unsigned long long *epoch_dev;  // device epoch counter (graph replay), or null
  unsigned long long timeout_ns;
  pb_status *st;
};

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Mark the exchange failed on every rank (first failed epoch wins per rank).
__device__ void peer_fail(const PeerArgs &a, unsigned long long epoch) {
  for (int r = 0; r < a.world; ++r) atomicCAS_system(a.flags[r] + kErrWord, 0ull, epoch);
  __threadfence_system();
  atomicCAS(&a.st->code, PB_OK, PB_ERR_PEER);
}

// thread 0 of the block waits until flags[slot0 + r] >= target for every
// rank r; false on timeout or when any rank has reported a failure.
__device__ bool peer_wait(const PeerArgs &a, int slot0, unsigned long long target,
                          unsigned long long epoch) {
  const unsigned long long *f = a.flags[a.rank];
  const unsigned long long t0 = global_ns();
  for (int r = 0; r < a.world; ++r) {
    while (ld_acquire_sys(f + slot0 + r) < target) {
      if (ld_acquire_sys(f + kErrWord) != 0) {
        atomicCAS(&a.st->code, PB_OK, PB_ERR_PEER);
        return false;
      }
      __nanosleep(64);
      if (global_ns() - t0 > a.timeout_ns) {  // a peer is gone or far behind
        peer_fail(a, epoch);
        return false;
      }
    }
  }
  if (ld_acquire_sys(f + kErrWord) != 0) {  // sticky: an earlier exchange failed
    atomicCAS(&a.st->code, PB_OK, PB_ERR_PEER);
    return false;
  }
  return true;
}

// summed (count << 48) - R and R of cell c over all ranks, weighted in
// species order from 0.0: weighted_partials of the reduced bins
__device__ __forceinline__ void reduced_partials(const PeerArgs &a, int64_t c, double &left,
                                                 double &right) {
  double l = 0.0, r = 0.0;
  for (int s = 0; s < a.ndep; ++s) {
    uint64_t R = 0, C = 0;
    const size_t o = (size_t)s * 2 * a.nc + c;
    for (int k = 0; k < a.world; ++k) {
      R += a.bins[k][o];
      C += a.bins[k][o + a.nc];
    }
    if (C >= kMaxCellCount) flag_overflow(a.st, C);
    const uint64_t L = (C << kFracBits) - R;
    const double lraw = __dmul_rn(__ull2double_rn(L), kFracInv);
    const double rraw = __dmul_rn(__ull2double_rn(R), kFracInv);
    l = __dadd_rn(l, __dmul_rn(a.coef[s], lraw));
    r = __dadd_rn(r, __dmul_rn(a.coef[s], rraw));
  }
  left = l;
  right = r;
}

__global__ void __launch_bounds__(kPeerThreads) k_peer_density(const __grid_constant__ PeerArgs a) {
  pdl_enter();
  // bumped by k_peer_epoch after this grid
  const unsigned long long epoch = a.epoch_dev ? *a.epoch_dev + 1 : a.epoch;
  const int64_t nc = a.nc;
  // A: announce that this rank's bins are final, wait for every rank
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int r = 0; r < a.world; ++r) st_release_sys(a.flags[r] + a.rank, epoch);
  }
  __shared__ int ok;
  __shared__ double s_right[kPeerThreads + 1];  // right partials of cells g0-1 .. g0+63
  if (threadIdx.x == 0) ok = peer_wait(a, 0, epoch, epoch);
  __syncthreads();
  // this rank's cells [c0, c1) and nodes [c0, c1) (the last rank also node nc)
  const int64_t c0 = nc * a.rank / a.world, c1 = nc * (a.rank + 1) / a.world;
  const int64_t n1 = a.rank == a.world - 1 ? nc + 1 : c1;
  if (ok) {
    // Each cell's reduced partials are computed once: a block covers 64
    // consecutive nodes g0..g0+63 and cells g0-1..g0+63 (one halo cell,
    // computed by thread 0), sharing the right partials through shared
    // memory; only the periodic / wall end nodes recompute an end cell.
    for (int64_t g0 = c0 + (int64_t)blockIdx.x * kPeerThreads; g0 < n1;
         g0 += (int64_t)gridDim.x * kPeerThreads) {
      const int64_t g = g0 + threadIdx.x;
      double lg = 0.0, rg = 0.0;
      if (g < nc && g < n1) {
        reduced_partials(a, g, lg, rg);
        for (int r = 0; r < a.world; ++r) {
          a.left[r][g] = lg;
          a.right[r][g] = rg;
        }
      }
      s_right[threadIdx.x + 1] = rg;
      if (threadIdx.x == 0) {
        double lh = 0.0, rh = 0.0;
        if (g0 > 0) reduced_partials(a, g0 - 1, lh, rh);
        s_right[0] = rh;
      }
      __syncthreads();
      if (g < n1) {
        double v;
        if (g > 0 && g < nc) {
          v = __dadd_rn(s_right[threadIdx.x], lg);  // rho[g] = R[g-1] + L[g] (fields.py:85)
        } else if (a.field_bc == PB_FIELD_PERIODIC) {
          double l0, r0, ll, rl;  // rho[0] = rho[nc] = R[nc-1] + L[0]
          reduced_partials(a, 0, l0, r0);
          reduced_partials(a, nc - 1, ll, rl);
          v = __dadd_rn(rl, l0);
        } else if (g == 0) {
          v = __dmul_rn(lg, 2.0);  // walls own half a cell (fields.py:115-117)
        } else {
          v = __dmul_rn(s_right[threadIdx.x], 2.0);  // g == nc: cell nc-1 is g-1
        }
        for (int r = 0; r < a.world; ++r) a.rho[r][g] = v;
      }
      __syncthreads();
    }
  }
  // B: this block has read every rank's bins and stored its outputs.  The
  // done count is added even after a failure, so the counts of all ranks stay
  // aligned with epoch * blocks.
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int r = 0; r < a.world; ++r)
      atomicAdd_system(a.flags[r] + a.world + a.rank, 1ull);
    ok = ok && peer_wait(a, a.world, epoch * (unsigned long long)gridDim.x, epoch);
  }
  __syncthreads();
  if (!ok) return;  // a peer may still read these bins: leave them
  // every rank is past its reads: clear this rank's bins (and, if asked, the
  // set the coming push deposits into)
  uint64_t *mine = const_cast<uint64_t *>(a.bins[a.rank]);
  const int64_t words = (int64_t)a.ndep * 2 * nc;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    mine[w] = 0;
    if (a.clear_next) a.clear_next[w] = 0;
  }
}

// The device epoch advances once per exchange, stream-ordered after the
// exchange kernel (so a captured step replays with a fresh epoch each time).
__global__ void k_peer_epoch(unsigned long long *epoch) {
  pdl_enter();
  *epoch += 1;
}

}  // namespace pb

extern "C" int pb_peer_alloc(size_t bytes, void **ptr, void *handle_out) {
  if (!ptr || !handle_out || bytes == 0) {
    pb::set_error("pb_peer_alloc: bad arguments");
    return PB_ERR_INVALID;
  }
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaMalloc");
  e = cudaMemset(*ptr, 0, bytes);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaMemset");
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaIpcGetMemHandle");
  memcpy(handle_out, &h, sizeof(h));
  return PB_OK;
}

extern "C" int pb_peer_open(const void *handle, void **ptr) {
  if (!handle || !ptr) {
    pb::set_error("pb_peer_open: bad arguments");
    return PB_ERR_INVALID;
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaIpcOpenMemHandle");
  return PB_OK;
}

extern "C" int pb_peer_close(void *ptr, int owned) {
  cudaError_t e = owned ? cudaFree(ptr) : cudaIpcCloseMemHandle(ptr);
  if (e != cudaSuccess) return pb::cuda_status(e, owned ? "cudaFree" : "cudaIpcCloseMemHandle");
  return PB_OK;
}

extern "C" int pb_peer_density_step(const pb_peer_density *p, uint64_t *bins_next,
                                    const double *coef, int ndep, int64_t nc, int field_bc,
                                    pb_status *status, void *stream) {
  if (!p || p->world < 1 || p->world > PB_MAX_RANKS || p->rank < 0 || p->rank >= p->world ||
      ndep < 0 || ndep > PB_MAX_SPECIES || nc < 2 || !status || (p->epoch == 0 && !p->epoch_dev) ||
      (ndep > 0 && !coef) ||
      (field_bc != PB_FIELD_PERIODIC && field_bc != PB_FIELD_DIRICHLET)) {
    pb::set_error("pb_peer_density_step: bad arguments");
    return PB_ERR_INVALID;
  }
  pb::PeerArgs a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < p->world; ++r) {
    if (!p->bins[r] || !p->left[r] || !p->right[r] || !p->rho[r] || !p->flags[r]) {
      pb::set_error("pb_peer_density_step: NULL buffer of rank %d", r);
      return PB_ERR_INVALID;
    }
    a.bins[r] = p->bins[r];
    a.left[r] = p->left[r];
    a.right[r] = p->right[r];
    a.rho[r] = p->rho[r];
    a.flags[r] = (unsigned long long *)p->flags[r];
  }
  for (int s = 0; s < ndep; ++s) a.coef[s] = coef[s];
  a.ndep = ndep;
  a.rank = p->rank;
  a.world = p->world;
  a.field_bc = field_bc;
  a.nc = nc;
  a.epoch = p->epoch;
  a.epoch_dev = (const unsigned long long *)p->epoch_dev;
  a.clear_next = bins_next;
  a.timeout_ns = p->timeout_ns ? p->timeout_ns : 60000000000ull;
  a.st = status;
  // persistent grid: every block must be resident to reach the barriers
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t per_rank = (nc + 1 + p->world - 1) / p->world;
  int64_t blocks = (per_rank + pb::kPeerThreads - 1) / pb::kPeerThreads;
  if (blocks > sms) blocks = sms;
  if (blocks < 1) blocks = 1;
  // co-residency: the barriers need every block of the grid resident at once
  int per_sm = 0;
  cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pb::k_peer_density,
                                                                 pb::kPeerThreads, 0);
  if (oe != cudaSuccess) return pb::cuda_status(oe, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if ((int64_t)per_sm * sms < blocks) {
    pb::set_error("pb_peer_density_step: %lld blocks cannot be co-resident (%d per SM x %d SMs)",
                  (long long)blocks, per_sm, sms);
    return PB_ERR_INVALID;
  }
  // the done count target is epoch * blocks on every rank: same grid everywhere
  cudaError_t e = pb::launch_pdl(pb::k_peer_density, dim3((unsigned)blocks), dim3(pb::kPeerThreads),
                                 0, (cudaStream_t)stream, a);
  if (e != cudaSuccess) return pb::cuda_status(e, "k_peer_density");
  if (p->epoch_dev) {
    e = pb::launch_pdl(pb::k_peer_epoch, dim3(1), dim3(1), 0, (cudaStream_t)stream,
                       (unsigned long long *)p->epoch_dev);
    if (e != cudaSuccess) return pb::cuda_status(e, "k_peer_epoch");
  }
  return PB_OK;
}
