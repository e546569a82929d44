// Fused particle mover + charge deposition for sm_100a.
//
// One persistent-style launch covers every species of a step.  Blocks are
// split across species in proportion to their HBM bytes; each block owns a
// contiguous chunk of its species' flat SoA arrays and streams it once:
//
//   load (x, vx[, vy, vz, yp], cell)        128-bit, evict-first
//   gather a[j], a[j+1] = coef*E            read-only path, L1/L2 resident
//   kick / Boris / drift                     reference op order, no FMA
//   floor / carry / wrap or absorb           pkg/src/picmc/mover.py:136-163
//   store x, vx[, ...]; cell only if moved
//   fixed-point deposit of the new position  warp segmented scan -> smem
//                                            window -> global u64 atomics
//
// Reference arithmetic per particle (pkg/src/picmc/backends/_kernels.pyx:81-101):
//   atemp = aj + x*(aj1 - aj); v = vx + atemp; vx = v; x = x + fnstep*v
//   yp = yp + fnstep*vy
// with aj = coef*E[j] (accel_nodes_for_species, pkg/src/picmc/mover.py:221).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "mover.cuh"

namespace pb {

constexpr int kThreads = 256;
constexpr int kPairsPerThread = 2;
constexpr int kTile = kThreads * 2 * kPairsPerThread;  // 1024 particles
constexpr int kWin = 1024;    // shared-memory deposit window, cells
constexpr int kMargin = 64;   // cells kept left of the chunk's first cell

// A chunk list over some of the launch's species: round-robin over them for
// the first rr_chunks chunks (rr_each per species), then species by species.
struct ChunkList {
  int nsp;
  int order[PB_MAX_SPECIES];  // slots in LaunchArgs::sp
  int64_t tile_start[PB_MAX_SPECIES + 1];
  int64_t rr_chunks, rr_each;
  int64_t tail_start[PB_MAX_SPECIES + 1];
};

struct LaunchArgs {
  pb_species sp[PB_MAX_SPECIES];
  int blk_start[PB_MAX_SPECIES + 1];
  int id[PB_MAX_SPECIES];  // caller species index (status arrays)
  int nsp;
  int push;  // 0: deposit only (no mover)
  int order[PB_MAX_SPECIES];             // chunk list over all species (quad/ring kernels)
  int64_t tile_start[PB_MAX_SPECIES + 1];
  // quad kernel chunk interleave: the first rr_chunks chunks go round-robin
  // over the species (rr_each per species), the rest species by species
  int64_t rr_chunks, rr_each;
  int64_t tail_start[PB_MAX_SPECIES + 1];
  int64_t chunk;  // particles per claimed chunk (power of two dividing PB_CELL8_CHUNK)
  // split mover: list 0 = ring-staged charged species, list 1 = the rest
  ChunkList lists[2];
  const double *e;
  int64_t nc;
  uint64_t *bins;
  pb_status *st;
};

// ---------------------------------------------------------------------------
// Deposit emission: warp segmented reduction of packed (count, R) words keyed
// by cell, then shared-memory window atomics or global atomics.
// ---------------------------------------------------------------------------
struct Window {
  uint64_t *sR;
  uint32_t *sC;
  int64_t base;
  int64_t lim;  // window width in use (0: global atomics only)
  uint64_t *gR;
  uint64_t *gC;

  __device__ __forceinline__ void emit(int32_t key, uint64_t w) const {
    const uint64_t r = w & kRMask;
    const uint32_t c = (uint32_t)(w >> kCountShift);
    const int64_t b = (int64_t)key - base;
    if (b >= 0 && b < lim) {
      atomicAdd((unsigned long long *)&sR[b], (unsigned long long)r);
      atomicAdd(&sC[b], c);
    } else {
      atomicAdd((unsigned long long *)&gR[key], (unsigned long long)r);
      atomicAdd((unsigned long long *)&gC[key], (unsigned long long)c);
    }
  }
};

// Every lane of the warp must call this (it shuffles).  key < 0 = nothing.
__device__ __forceinline__ void warp_segmented_emit(int32_t key, uint64_t w,
                                                    const Window &win) {
  const unsigned full = 0xffffffffu;
  const unsigned lane = lane_id();
  const int32_t kprev = __shfl_up_sync(full, key, 1);
  const int32_t knext = __shfl_down_sync(full, key, 1);
  const bool head = (lane == 0) || (kprev != key);
  const bool tail = (lane == 31) || (knext != key);
  int f = head;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t wu = __shfl_up_sync(full, w, d);
    const int fu = __shfl_up_sync(full, f, d);
    if ((int)lane >= d) {
      if (!f) w += wu;
      f |= fu;
    }
  }
  if (tail && key >= 0) win.emit(key, w);
}

// Two consecutive particles of one lane: merge locally, emit the first
// directly if it starts a different cell, scan the second.
__device__ __forceinline__ void deposit_pair(int32_t k0, double x0, int32_t k1,
                                             double x1, const Window &win) {
  uint64_t w0 = k0 >= 0 ? deposit_word(x0) : 0;
  uint64_t w1 = k1 >= 0 ? deposit_word(x1) : 0;
  if (k0 == k1) {
    w1 += w0;
  } else if (k0 >= 0) {
    win.emit(k0, w0);
  }
  warp_segmented_emit(k1, w1, win);
}

// ---------------------------------------------------------------------------
// Block-level accumulators for the step status.
// ---------------------------------------------------------------------------
struct Tally {
  int moved = 0;
  int absorbed[2] = {0, 0};
};

// Register image of two consecutive particles.
struct Pair {
  double x0 = 0, x1 = 0, vx0 = 0, vx1 = 0, vy0 = 0, vy1 = 0, vz0 = 0, vz1 = 0,
         y0 = 0, y1 = 0;
  int32_t c0 = -1, c1 = -1;
};

template <int KIND, bool YP>
struct Fields {
  static constexpr bool kNeedV = (KIND == PB_KIND_KICK || is_boris(KIND) ||
                                  KIND == PB_KIND_DRIFT);
  static constexpr bool kVy = YP || is_boris(KIND);
  static constexpr bool kVz = is_boris(KIND);
};

// Push, cell transfer, stores, tallies and deposit for particles i, i+1
// (v0/v1: which of them exist).  Warp-collective when BC == ABSORBING or
// DEP: every lane of the warp must call it.
template <int KIND, bool YP, int BC, bool PUSH, bool DEP>
__device__ __forceinline__ void handle_pair(const LaunchArgs &a,
                                            const pb_species &s, int sid,
                                            int64_t i, bool v0, bool v1,
                                            Pair &q, const Window &win,
                                            Tally &t) {
  const unsigned full = 0xffffffffu;
  const int64_t nc = a.nc;
  constexpr bool kEagerCell = (KIND != PB_KIND_DRIFT) || DEP;
  int32_t n0 = q.c0, n1 = q.c1;
  if (PUSH) {
    bool m0 = false, m1 = false, cfl0 = false, cfl1 = false;
    int8_t w0 = -1, w1 = -1;
    if (v0) {
      kick_drift<KIND>(q.x0, q.vx0, q.vy0, q.vz0, q.c0, s, a.e);
      if (YP) q.y0 = __dadd_rn(q.y0, __dmul_rn(s.fnstep, q.vy0));
      if (!kEagerCell && floor(q.x0) != 0.0) q.c0 = s.cell[i];
      const MoveOut o = transfer<BC>(q.x0, q.c0, nc);
      n0 = o.cell;
      m0 = o.moved;
      w0 = o.wall;
      cfl0 = o.cfl;
    }
    if (v1) {
      kick_drift<KIND>(q.x1, q.vx1, q.vy1, q.vz1, q.c1, s, a.e);
      if (YP) q.y1 = __dadd_rn(q.y1, __dmul_rn(s.fnstep, q.vy1));
      if (!kEagerCell && floor(q.x1) != 0.0) q.c1 = s.cell[i + 1];
      const MoveOut o = transfer<BC>(q.x1, q.c1, nc);
      n1 = o.cell;
      m1 = o.moved;
      w1 = o.wall;
      cfl1 = o.cfl;
    }
    double *X = s.x, *VX = s.vx, *VY = s.vy, *VZ = s.vz, *YPp = s.yp;
    if (v1) {
      __stcs(reinterpret_cast<double2 *>(X + i), make_double2(q.x0, q.x1));
      if (KIND != PB_KIND_DRIFT)
        __stcs(reinterpret_cast<double2 *>(VX + i), make_double2(q.vx0, q.vx1));
      if (is_boris(KIND)) {
        __stcs(reinterpret_cast<double2 *>(VY + i), make_double2(q.vy0, q.vy1));
        __stcs(reinterpret_cast<double2 *>(VZ + i), make_double2(q.vz0, q.vz1));
      }
      if (YP) __stcs(reinterpret_cast<double2 *>(YPp + i), make_double2(q.y0, q.y1));
    } else if (v0) {
      X[i] = q.x0;
      if (KIND != PB_KIND_DRIFT) VX[i] = q.vx0;
      if (is_boris(KIND)) {
        VY[i] = q.vy0;
        VZ[i] = q.vz0;
      }
      if (YP) YPp[i] = q.y0;
    }
    if (m0) {
      s.cell[i] = n0;
      if (s.cell8) s.cell8[i] = (int8_t)PB_CELL8_ESCAPE;
    }
    if (m1) {
      s.cell[i + 1] = n1;
      if (s.cell8) s.cell8[i + 1] = (int8_t)PB_CELL8_ESCAPE;
    }
    t.moved += (int)m0 + (int)m1;
    if (BC == PB_BC_ABSORBING) {
      t.absorbed[0] += (int)(w0 == 0) + (int)(w1 == 0);
      t.absorbed[1] += (int)(w0 == 1) + (int)(w1 == 1);
      // Warp-ballot stream compaction of removed slots into the hole list.
      const bool r0 = w0 >= 0, r1 = w1 >= 0;
      const unsigned b0 = __ballot_sync(full, r0);
      const unsigned b1 = __ballot_sync(full, r1);
      const int tot = __popc(b0) + __popc(b1);
      if (tot) {
        const unsigned lane = lane_id();
        unsigned long long base = 0;
        if (lane == 0)
          base = atomicAdd((unsigned long long *)&a.st->n_holes[sid], (unsigned long long)tot);
        base = __shfl_sync(full, base, 0);
        const unsigned lt = (1u << lane) - 1u;
        if (r0) s.holes[base + __popc(b0 & lt)] = i;
        if (r1) s.holes[base + __popc(b0) + __popc(b1 & lt)] = i + 1;
      }
    }
    if (cfl0 || cfl1) {
      const uint64_t key = ((uint64_t)sid << 56) | (uint64_t)(cfl0 ? i : i + 1);
      atomicMin((unsigned long long *)&a.st->cfl_index, (unsigned long long)key);
      atomicCAS(&a.st->code, PB_OK, PB_ERR_CFL);
      if (cfl0) n0 = -1;
      if (cfl1) n1 = -1;
    }
  }
  if (DEP) deposit_pair(v0 ? n0 : -1, q.x0, v1 ? n1 : -1, q.x1, win);
}

// LDG path: used for chunk tails, deposit-only launches and PB_PUSH_PATH=ldg.
// Consumer threads only (threadIdx.x < kThreads).
template <int KIND, bool YP, int BC, bool PUSH, bool DEP>
__device__ __forceinline__ void process_chunk(const LaunchArgs &a, int isp,
                                              int64_t beg, int64_t end,
                                              const Window &win, Tally &t) {
  using F = Fields<KIND, YP>;
  const pb_species &s = a.sp[isp];
  const int sid = a.id[isp];
  constexpr bool kEagerCell = (KIND != PB_KIND_DRIFT) || DEP;
  for (int64_t tb = beg; tb < end; tb += kTile) {
#pragma unroll
    for (int p = 0; p < kPairsPerThread; ++p) {
      const int64_t i = tb + (int64_t)p * (2 * kThreads) + 2 * threadIdx.x;
      const bool v0 = i < end;
      const bool v1 = (i + 1) < end;
      Pair q;
      if (v1) {
        const double2 xx = __ldcs(reinterpret_cast<const double2 *>(s.x + i));
        q.x0 = xx.x;
        q.x1 = xx.y;
        if (PUSH && F::kNeedV) {
          const double2 v = __ldcs(reinterpret_cast<const double2 *>(s.vx + i));
          q.vx0 = v.x;
          q.vx1 = v.y;
        }
        if (PUSH && F::kVy) {
          const double2 v = __ldcs(reinterpret_cast<const double2 *>(s.vy + i));
          q.vy0 = v.x;
          q.vy1 = v.y;
        }
        if (PUSH && F::kVz) {
          const double2 v = __ldcs(reinterpret_cast<const double2 *>(s.vz + i));
          q.vz0 = v.x;
          q.vz1 = v.y;
        }
        if (PUSH && YP) {
          const double2 v = __ldcs(reinterpret_cast<const double2 *>(s.yp + i));
          q.y0 = v.x;
          q.y1 = v.y;
        }
        if (kEagerCell) {
          const int2 c = __ldcs(reinterpret_cast<const int2 *>(s.cell + i));
          q.c0 = c.x;
          q.c1 = c.y;
        }
      } else if (v0) {
        q.x0 = s.x[i];
        if (PUSH && F::kNeedV) q.vx0 = s.vx[i];
        if (PUSH && F::kVy) q.vy0 = s.vy[i];
        if (PUSH && F::kVz) q.vz0 = s.vz[i];
        if (PUSH && YP) q.y0 = s.yp[i];
        if (kEagerCell) q.c0 = s.cell[i];
      }
      handle_pair<KIND, YP, BC, PUSH, DEP>(a, s, sid, i, v0, v1, q, win, t);
    }
  }
}

// ---------------------------------------------------------------------------
// LDG kernel: static contiguous chunks per block, shared-memory deposit
// window.  Used for deposit-only launches and as the PB_PUSH_PATH=ldg mover.
// ---------------------------------------------------------------------------
template <int KIND, bool YP, int BC, bool PUSH>
__device__ __forceinline__ void ldg_dispatch(const LaunchArgs &a, int isp, int64_t beg,
                                             int64_t end, const Window &win, Tally &t,
                                             bool dep) {
  if (dep)
    process_chunk<KIND, YP, BC, PUSH, true>(a, isp, beg, end, win, t);
  else
    process_chunk<KIND, YP, BC, PUSH, false>(a, isp, beg, end, win, t);
}

template <int BC, bool PUSH>
__device__ __forceinline__ void run_any(const LaunchArgs &a, int isp, int64_t beg, int64_t end,
                                        const Window &win, Tally &t, bool dep) {
  const pb_species &s = a.sp[isp];
  const bool yp = s.yp != nullptr;
  const int kind = PUSH ? s.kind : PB_KIND_INACTIVE;
  switch (kind) {
    case PB_KIND_KICK:
      if (yp) ldg_dispatch<PB_KIND_KICK, true, BC, PUSH>(a, isp, beg, end, win, t, dep);
      else ldg_dispatch<PB_KIND_KICK, false, BC, PUSH>(a, isp, beg, end, win, t, dep);
      break;
    case PB_KIND_BORIS:
      if (s.b_nodes) {
        if (yp) ldg_dispatch<kKindBorisB, true, BC, PUSH>(a, isp, beg, end, win, t, dep);
        else ldg_dispatch<kKindBorisB, false, BC, PUSH>(a, isp, beg, end, win, t, dep);
      } else {
        if (yp) ldg_dispatch<PB_KIND_BORIS, true, BC, PUSH>(a, isp, beg, end, win, t, dep);
        else ldg_dispatch<PB_KIND_BORIS, false, BC, PUSH>(a, isp, beg, end, win, t, dep);
      }
      break;
    case PB_KIND_DRIFT:
      if (yp) ldg_dispatch<PB_KIND_DRIFT, true, BC, PUSH>(a, isp, beg, end, win, t, dep);
      else ldg_dispatch<PB_KIND_DRIFT, false, BC, PUSH>(a, isp, beg, end, win, t, dep);
      break;
    default:  // not pushed: deposit current positions only
      if (dep) process_chunk<PB_KIND_INACTIVE, false, BC, false, true>(a, isp, beg, end, win, t);
      break;
  }
}

// Block reduction of the tallies into the step status (all threads call).
__device__ __forceinline__ void flush_tally(const LaunchArgs &a, int sid, const Tally &t,
                                            int *sTally) {
  int mv = t.moved, al = t.absorbed[0], ar = t.absorbed[1];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mv += __shfl_down_sync(0xffffffffu, mv, d);
    al += __shfl_down_sync(0xffffffffu, al, d);
    ar += __shfl_down_sync(0xffffffffu, ar, d);
  }
  if (lane_id() == 0) {
    if (mv) atomicAdd((unsigned long long *)&a.st->moved[sid], (unsigned long long)mv);
    if (al) atomicAdd((unsigned long long *)&a.st->absorbed[sid][0], (unsigned long long)al);
    if (ar) atomicAdd((unsigned long long *)&a.st->absorbed[sid][1], (unsigned long long)ar);
  }
  (void)sTally;
}

template <int BC, bool PUSH>
__global__ void __launch_bounds__(kThreads)
    k_push_deposit(const __grid_constant__ LaunchArgs a) {
  __shared__ uint64_t sR[kWin];
  __shared__ uint32_t sC[kWin];

  int isp = 0;
  while (isp + 1 < a.nsp && (int)blockIdx.x >= a.blk_start[isp + 1]) ++isp;
  const pb_species &s = a.sp[isp];
  const int lb = (int)blockIdx.x - a.blk_start[isp];
  const int nb = a.blk_start[isp + 1] - a.blk_start[isp];
  const int64_t n = s.n_dev ? *s.n_dev : s.n;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  const int64_t t0 = ntiles * lb / nb, t1 = ntiles * (lb + 1) / nb;
  if (t0 >= t1) return;  // uniform across the block
  const int64_t beg = t0 * kTile;
  const int64_t end = t1 * kTile < n ? t1 * kTile : n;
  const bool dep = s.deposit >= 0 && a.bins != nullptr;

  for (int b = threadIdx.x; b < kWin; b += kThreads) {
    sR[b] = 0;
    sC[b] = 0;
  }
  Window win{sR, sC, 0, kWin, nullptr, nullptr};
  if (dep) {
    win.gR = a.bins + (size_t)s.deposit * 2 * (size_t)a.nc;
    win.gC = win.gR + a.nc;
    win.base = (int64_t)s.cell[beg] - kMargin;
  }
  __syncthreads();
  Tally t;
  run_any<BC, PUSH>(a, isp, beg, end, win, t, dep);
  if (PUSH) flush_tally(a, a.id[isp], t, nullptr);
  __syncthreads();
  if (dep) {
    for (int b = threadIdx.x; b < kWin; b += kThreads) {
      const uint32_t c = sC[b];
      if (c) {
        const int64_t cell = win.base + b;
        atomicAdd((unsigned long long *)&win.gR[cell], (unsigned long long)sR[b]);
        atomicAdd((unsigned long long *)&win.gC[cell], (unsigned long long)c);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA) + mbarrier helpers of the per-warp rings (k_push_ring,
// k_push_split).
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Self-cleaning work counter: every claimer (a warp, or a TMA producer lane)
// reports once when it has stopped claiming; the last one resets the counter,
// so no separate reset has to be ordered before the next launch (the density
// epilogue can then run concurrently with the mover).
// A claimer's last claim has returned (it is what ended its loop) before its
// done-increment is issued, so the reset is ordered after every claim without
// a fence (a __threadfence here costs a full L1 invalidate per exiting warp).
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// In-kernel launch clock (pb_status.mover_t0/mover_ns/mover_launches): one
// RED.MIN per block at its start...
// PB_MOVER_TRACE builds: every block's start and every warp's finish
// (scripts/mover_tail_trace.py, pb_debug_warp_ends)
#ifdef PB_MOVER_TRACE
__device__ unsigned long long g_blk_start[2048];
__device__ unsigned long long g_warp_end[8192];
__device__ unsigned long long g_mlog[512][2];  // per launch: first block start, last warp end
__device__ unsigned long long g_mlog_n;
#endif
__device__ __forceinline__ void mover_clock_start(pb_status *st) {
  if (threadIdx.x == 0) {
    const unsigned long long t = global_ns();
    atomicMin((unsigned long long *)&st->mover_t0, t);
#ifdef PB_MOVER_TRACE
    if (blockIdx.x < 2048) g_blk_start[blockIdx.x] = t;
#endif
  }
}

__device__ __forceinline__ void release_work_counter(pb_status *st, unsigned long long claimers) {
#ifdef PB_RELEASE_FENCE
  __threadfence();
#endif
#ifdef PB_MOVER_TRACE
  {
    const unsigned w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w < 8192) g_warp_end[w] = global_ns();
  }
#endif
  const unsigned long long d = atomicAdd((unsigned long long *)&st->tile_done, 1ull);
  if (d == claimers - 1) {
    // ...and the last claimer to finish closes the launch's interval
    const unsigned long long t1 = global_ns();
    const unsigned long long t0 = atomicExch((unsigned long long *)&st->mover_t0, ~0ull);
#ifdef PB_MOVER_TRACE
    {
      const unsigned long long k = atomicAdd(&g_mlog_n, 1ull) % 512;
      g_mlog[k][0] = t0;
      g_mlog[k][1] = t1;
    }
#endif
    if (t0 != ~0ull && t1 > t0) {
      atomicAdd((unsigned long long *)&st->mover_ns, t1 - t0);
      atomicAdd((unsigned long long *)&st->mover_launches, 1ull);
    }
    atomicExch((unsigned long long *)&st->tile_next, 0ull);
    atomicExch((unsigned long long *)&st->tile_next2, 0ull);
    atomicExch((unsigned long long *)&st->tile_done, 0ull);
  }
}

// Thread-local run of equal cells, flushed to the window when the cell changes.
struct RunAcc {
  int32_t key = -1;
  uint64_t w = 0;
  __device__ __forceinline__ void add(int32_t k, double x, const Window &win) {
    if (k < 0) return;
    const uint64_t d = deposit_word(x);
    if (k == key) {
      w += d;
    } else {
      if (key >= 0) win.emit(key, w);
      key = k;
      w = d;
    }
  }
};

#ifndef PB_ST4
#define PB_ST4 "st.global.cs.v4.f64"
#endif
__device__ __forceinline__ void st4(double *p, double a, double b, double c, double d) {
  asm volatile(PB_ST4 " [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}

// ---------------------------------------------------------------------------
#ifndef PB_CHUNK
#define PB_CHUNK 2048
#endif
constexpr int kChunk = PB_CHUNK;

#ifndef PB_LD4
#define PB_LD4 "ld.global.cs.v4.f64"
#endif
__device__ __forceinline__ void ld4(const double *p, double &a, double &b, double &c, double &d) {
  asm volatile(PB_LD4 " {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// Register image of one lane's 4 consecutive particles.
template <int KIND, bool YP>
struct Quad {
  double x[4], vx[4], vy[4], vz[4], y[4];
  int32_t c[4];
  int32_t base;  // chunk_base of the quad's chunk (cell8 in use)
  int packed;    // 4 cell8 bytes, not yet decoded when c[0] == kPackedCells
  int nv;
};

constexpr int32_t kPackedCells = -2;  // c[0] marker: cells still in q.packed

template <int KIND, bool YP>
__device__ __forceinline__ void quad_cells(const pb_species &s, int64_t i, Quad<KIND, YP> &q) {
  if (q.c[0] != kPackedCells) return;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int8_t o = (int8_t)((q.packed >> (8 * k)) & 0xff);
    q.c[k] = o == PB_CELL8_ESCAPE ? s.cell[i + k] : q.base + (int32_t)o;
  }
}

__device__ __forceinline__ int8_t cell8_encode(int32_t cell, int32_t base) {
  const int32_t d = cell - base;
  return (d > PB_CELL8_ESCAPE && d <= 127) ? (int8_t)d : (int8_t)PB_CELL8_ESCAPE;
}

template <int KIND, bool YP>
__device__ __forceinline__ void quad_load(const pb_species &s, int64_t i, int64_t end,
                                          Quad<KIND, YP> &q) {
  using F = Fields<KIND, YP>;
  constexpr bool kCell = KIND != PB_KIND_DRIFT;
  q.nv = i >= end ? 0 : (end - i >= 4 ? 4 : (int)(end - i));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    q.x[k] = q.vx[k] = q.vy[k] = q.vz[k] = q.y[k] = 0.0;
    q.c[k] = -1;
  }
  q.base = 0;
  q.packed = 0;
  if (q.nv == 4) {
    ld4(s.x + i, q.x[0], q.x[1], q.x[2], q.x[3]);
    ld4(s.vx + i, q.vx[0], q.vx[1], q.vx[2], q.vx[3]);
    if (F::kVy) ld4(s.vy + i, q.vy[0], q.vy[1], q.vy[2], q.vy[3]);
    if (F::kVz) ld4(s.vz + i, q.vz[0], q.vz[1], q.vz[2], q.vz[3]);
    if (YP) ld4(s.yp + i, q.y[0], q.y[1], q.y[2], q.y[3]);
    if (kCell) {
      if (s.cell8) {
        // 4 compressed cells in one 32-bit load, decoded at first use
        // (quad_cells) so a prefetched slice does not stall here
        q.base = __ldg(s.chunk_base + i / PB_CELL8_CHUNK);
        q.packed = __ldcs(reinterpret_cast<const int *>(s.cell8 + i));
        q.c[0] = kPackedCells;
      } else {
        const int4 cc = __ldcs(reinterpret_cast<const int4 *>(s.cell + i));
        q.c[0] = cc.x;
        q.c[1] = cc.y;
        q.c[2] = cc.z;
        q.c[3] = cc.w;
      }
    }
  } else {
    if (kCell && s.cell8 && q.nv > 0) q.base = __ldg(s.chunk_base + i / PB_CELL8_CHUNK);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < q.nv) {
        q.x[k] = s.x[i + k];
        q.vx[k] = s.vx[i + k];
        if (F::kVy) q.vy[k] = s.vy[i + k];
        if (F::kVz) q.vz[k] = s.vz[i + k];
        if (YP) q.y[k] = s.yp[i + k];
        if (kCell) q.c[k] = s.cell[i + k];
      }
    }
  }
}

#ifndef PB_FULL_SLICES
#define PB_FULL_SLICES 1
#endif
// Push, transfer, store, tallies and deposit of one lane's quad at slot i
// (every lane of the warp calls this: the deposit scan shuffles).  FULL: the
// quad is known to hold 4 particles (a full TMA slice) -- no per-particle
// validity predicates.  The rare events (cell transfers, CFL, wall removal)
// are tested once per quad / warp and handled off the common path.
template <int KIND, bool YP, int BC, bool DEP, bool FULL = false>
__device__ __forceinline__ void quad_process(const LaunchArgs &a, int isp, int64_t i,
                                             Quad<KIND, YP> &q, const Window &win, Tally &t) {
  const pb_species &s = a.sp[isp];
  const int sid = a.id[isp];
  const unsigned full = 0xffffffffu;
  const int64_t nc = a.nc;
  constexpr bool kCell = KIND != PB_KIND_DRIFT;
  const int lane = (int)lane_id();
  const int nv = FULL ? 4 : q.nv;
  if (kCell) quad_cells<KIND, YP>(s, i, q);
  int32_t nn[4];
  int8_t wall[4];
  bool mv[4], cfl[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    nn[k] = -1;
    wall[k] = -1;
    mv[k] = false;
    cfl[k] = false;
    if (FULL || k < nv) {
      kick_drift<KIND>(q.x[k], q.vx[k], q.vy[k], q.vz[k], q.c[k], s, a.e);
      if (YP) q.y[k] = __dadd_rn(q.y[k], __dmul_rn(s.fnstep, q.vy[k]));
      if (!kCell && floor(q.x[k]) != 0.0) q.c[k] = s.cell[i + k];
      const MoveOut o = transfer<BC>(q.x[k], q.c[k], nc);
      nn[k] = o.cell;
      mv[k] = o.moved;
      wall[k] = o.wall;
      cfl[k] = o.cfl;
    }
  }
  if (FULL || nv == 4) {
    st4(s.x + i, q.x[0], q.x[1], q.x[2], q.x[3]);
    if (KIND != PB_KIND_DRIFT) st4(s.vx + i, q.vx[0], q.vx[1], q.vx[2], q.vx[3]);
    if (is_boris(KIND)) {
      st4(s.vy + i, q.vy[0], q.vy[1], q.vy[2], q.vy[3]);
      st4(s.vz + i, q.vz[0], q.vz[1], q.vz[2], q.vz[3]);
    }
    if (YP) st4(s.yp + i, q.y[0], q.y[1], q.y[2], q.y[3]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < nv) {
        s.x[i + k] = q.x[k];
        if (KIND != PB_KIND_DRIFT) s.vx[i + k] = q.vx[k];
        if (is_boris(KIND)) {
          s.vy[i + k] = q.vy[k];
          s.vz[i + k] = q.vz[k];
        }
        if (YP) s.yp[i + k] = q.y[k];
      }
    }
  }
  t.moved += (int)mv[0] + (int)mv[1] + (int)mv[2] + (int)mv[3];
  if (mv[0] | mv[1] | mv[2] | mv[3]) {  // a cell transfer: ~0.6% of electron pushes
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (mv[k]) {
        s.cell[i + k] = nn[k];
        if (kCell && s.cell8)
          s.cell8[i + k] = nn[k] >= 0 ? cell8_encode(nn[k], q.base) : (int8_t)PB_CELL8_ESCAPE;
      }
    }
  }
  if (cfl[0] | cfl[1] | cfl[2] | cfl[3]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (cfl[k]) {
        const uint64_t key = ((uint64_t)sid << 56) | (uint64_t)(i + k);
        atomicMin((unsigned long long *)&a.st->cfl_index, (unsigned long long)key);
        atomicCAS(&a.st->code, PB_OK, PB_ERR_CFL);
        nn[k] = -1;
      }
    }
  }
  if (BC == PB_BC_ABSORBING) {
    // Warp-ballot stream compaction of removed slots into the hole list,
    // entered only by warps that removed something.
    if (__any_sync(full, (wall[0] >= 0) | (wall[1] >= 0) | (wall[2] >= 0) | (wall[3] >= 0))) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        t.absorbed[0] += (int)(wall[k] == 0);
        t.absorbed[1] += (int)(wall[k] == 1);
        const bool r = wall[k] >= 0;
        const unsigned b = __ballot_sync(full, r);
        if (b) {
          unsigned long long hb = 0;
          if (lane == 0)
            hb = atomicAdd((unsigned long long *)&a.st->n_holes[sid], (unsigned long long)__popc(b));
          hb = __shfl_sync(full, hb, 0);
          if (r) s.holes[hb + __popc(b & ((1u << lane) - 1u))] = i + k;
        }
      }
    }
  }
  if (DEP) {
    int32_t key;
    uint64_t w;
    if (nn[0] >= 0 && nn[0] == nn[1] && nn[1] == nn[2] && nn[2] == nn[3]) {
      // the quad stays in one cell (sorted stores: the common case)
      key = nn[0];
      w = (uint64_t(4) << kCountShift) +
          ((quantize(q.x[0]) + quantize(q.x[1])) + (quantize(q.x[2]) + quantize(q.x[3])));
    } else {
      RunAcc run;
#pragma unroll
      for (int k = 0; k < 4; ++k) run.add(nn[k], q.x[k], win);
      key = run.key;
      w = run.w;
    }
    warp_segmented_emit(key, w, win);
  }
}

#ifndef PB_QUAD_PREFETCH
#define PB_QUAD_PREFETCH 1
#endif

template <int KIND, bool YP, int BC, bool DEP>
__device__ __forceinline__ void quad_chunk(const LaunchArgs &a, int isp, int64_t beg, int64_t end,
                                           const Window &win, Tally &t) {
  const pb_species &s = a.sp[isp];
  const int lane = (int)lane_id();
  // Charged (KICK, no yp) slices: software-pipeline the next 128 particles'
  // loads under this slice's gather / push / deposit scan, doubling the bytes
  // each warp keeps in flight (the neutral path already runs at copy rate;
  // wider kinds would spill at the 80-register budget).
  constexpr bool kPrefetch = PB_QUAD_PREFETCH && KIND == PB_KIND_KICK && !YP;
  Quad<KIND, YP> q;
  quad_load<KIND, YP>(s, beg + 4 * lane, end, q);
#pragma unroll 1
  for (int64_t q0 = beg; q0 < end; q0 += 128) {
    const int64_t i = q0 + 4 * lane;
    Quad<KIND, YP> nq;
    if (kPrefetch) quad_load<KIND, YP>(s, i + 128, end, nq);
    // warp-uniform: every lane holds 4 particles (periodic launches only: the
    // absorbing register path would spill with both bodies inlined)
    if (PB_FULL_SLICES && BC == PB_BC_PERIODIC && end - q0 >= 128)
      quad_process<KIND, YP, BC, DEP, true>(a, isp, i, q, win, t);
    else
      quad_process<KIND, YP, BC, DEP>(a, isp, i, q, win, t);
    if (kPrefetch)
      q = nq;
    else
      quad_load<KIND, YP>(s, i + 128, end, q);
  }
}

// Chunk c -> (species slot, [beg, end)).  end <= beg for empty chunks.
__device__ __forceinline__ int chunk_species(const LaunchArgs &a, int64_t c, int64_t &beg,
                                             int64_t &end) {
  int kk = 0;
  int64_t local;
  if (c < a.rr_chunks) {
    kk = (int)(c % a.nsp);
    local = c / a.nsp;
  } else {
    const int64_t r = c - a.rr_chunks;
    while (kk + 1 < a.nsp && r >= a.tail_start[kk + 1]) ++kk;
    local = a.rr_each + (r - a.tail_start[kk]);
  }
  const int isp = a.order[kk];
  const pb_species &s = a.sp[isp];
  const int64_t n = s.n_dev ? *s.n_dev : s.n;
  beg = local * a.chunk;
  end = beg + a.chunk < n ? beg + a.chunk : n;
  return isp;
}

__device__ __forceinline__ int64_t claim_chunk(const LaunchArgs &a) {
  unsigned long long c = 0;
  if (lane_id() == 0) c = atomicAdd((unsigned long long *)&a.st->tile_next, 1ull);
  return (int64_t)__shfl_sync(0xffffffffu, c, 0);
}

// BMODE: 0 no Boris species, 1 uniform-B Boris, 2 every charged mover a
// Boris species with B nodes (pb_species.b_nodes), 3 any mix with B nodes --
// separate kernels, so the gathered-B path's extra registers do not cost the
// uniform one.
template <int BC, int BMODE>
__device__ __forceinline__ void quad_dispatch(const LaunchArgs &a, int isp, int64_t beg,
                                              int64_t end, const Window &win, Tally &t) {
  const pb_species &s = a.sp[isp];
  const bool yp = s.yp != nullptr;
  const bool dep = s.deposit >= 0 && a.bins != nullptr;
#define PB_Q(K, Y)                                                  \
  do {                                                              \
    if (dep) quad_chunk<K, Y, BC, true>(a, isp, beg, end, win, t);  \
    else quad_chunk<K, Y, BC, false>(a, isp, beg, end, win, t);     \
  } while (0)
  // BMODE 2 launches hold only gathered-B Boris and neutral species (the
  // host checks): the kick and uniform-Boris bodies are not compiled in, so
  // the kernel's code -- which runs cold in the instruction cache, the two
  // live paths interleaved across warps -- stays small
  if (BMODE != 2 && s.kind == PB_KIND_KICK) {
    if (yp) PB_Q(PB_KIND_KICK, true); else PB_Q(PB_KIND_KICK, false);
  } else if (BMODE >= 2 && s.kind == PB_KIND_BORIS && s.b_nodes) {
    if (yp) PB_Q(kKindBorisB, true); else PB_Q(kKindBorisB, false);
  } else if (BMODE != 0 && BMODE != 2 && s.kind == PB_KIND_BORIS) {
    if (yp) PB_Q(PB_KIND_BORIS, true); else PB_Q(PB_KIND_BORIS, false);
  } else {
    if (yp) PB_Q(PB_KIND_DRIFT, true); else PB_Q(PB_KIND_DRIFT, false);
  }
#undef PB_Q
}

#ifndef PB_QUAD_MINBLOCKS
#define PB_QUAD_MINBLOCKS 3
#endif

constexpr int kWarpsPerBlock = kThreads / 32;

// The gathered-B kernel (BMODE 2) runs at 2 blocks/SM: its per-particle B
// gather + divisions would spill at the 3-block register budget.
template <int BC, int BMODE>
__global__ void __launch_bounds__(kThreads, BMODE >= 2 ? 2 : PB_QUAD_MINBLOCKS)
    k_push_quad(const __grid_constant__ LaunchArgs a) {
  pdl_enter();
  mover_clock_start(a.st);
  const int64_t total = a.tile_start[a.nsp];
  Window win{nullptr, nullptr, 0, 0, nullptr, nullptr};
  Tally t;
  int cur = -1;
  for (int64_t c = claim_chunk(a); c < total; c = claim_chunk(a)) {
    int64_t beg, end;
    const int isp = chunk_species(a, c, beg, end);
    const pb_species &s = a.sp[isp];
    if (isp != cur) {
      if (cur >= 0) flush_tally(a, a.id[cur], t, nullptr);
      t = Tally();
      cur = isp;
      if (s.deposit >= 0 && a.bins) {
        win.gR = a.bins + (size_t)s.deposit * 2 * (size_t)a.nc;
        win.gC = win.gR + a.nc;
      }
    }
    quad_dispatch<BC, BMODE>(a, isp, beg, end, win, t);
  }
  if (cur >= 0) flush_tally(a, a.id[cur], t, nullptr);
  if (lane_id() == 0) release_work_counter(a.st, (unsigned long long)gridDim.x * kWarpsPerBlock);
}

// ---------------------------------------------------------------------------
// Charged-only launches (e.g. config 3: no neutral slices to interleave
// with): a per-warp TMA ring.  Each warp streams its 128-particle slices
// (x, vx, cell = 2.5 KB) through kRing shared-memory stages with
// cp.async.bulk issued by one lane (mbarrier completion), claiming the next
// chunk before the current one runs out.  A stage is released as soon as the
// warp has copied its slice to registers, so the next slice streams in while
// the current one is computed and stored.  One stage is the fastest
// (config 3 push: 1 stage 93.9 us, 2 stages 94.7, 3 stages 96.2, 4 stages
// 115 -- two blocks per SM; a smaller carve-out leaves more L1 for the E
// gather).  Mixed launches use k_push_split.
// ---------------------------------------------------------------------------
#ifndef PB_RING_STAGES
#define PB_RING_STAGES 1
#endif
constexpr int kRing = PB_RING_STAGES;
constexpr int kSlice = 128;
constexpr int kSliceBytes = kSlice * 8 * 2 + kSlice * 4;  // x, vx, cell

struct SliceMeta {
  int64_t base;
  int32_t isp;
  int32_t cnt;  // kSlice: staged by TMA; fewer: loaded directly
};

struct WarpRing {
  unsigned char *buf;
  uint64_t *bar;
  SliceMeta *meta;
};

// Intra-block slice sharing (k_push_ring): each warp's claimed chunk is
// handed out slice by slice through a shared word, generation:16 |
// next slice:24 | slices:24, with the chunk's [base, end) and species in a
// two-generation buffer.  The owner takes its slices with the same atomic,
// so once the global chunk counter runs dry the warps that finish first take
// the remaining slices of their block's busy warps: a block ends when its
// eight warps' leftovers are done, not when its slowest warp finishes its
// whole last chunk (profiles/r02_mover_tail.txt: 24 us of warp finishing
// spread in a 91 us config-3 launch).
struct ShareChunk {
  int64_t base, end;
  int32_t isp, pad;
};
struct ShareState {
  unsigned long long word[kWarpsPerBlock];
  ShareChunk gen[kWarpsPerBlock][2];
};
constexpr int kShareSliceShift = 24;
constexpr unsigned long long kShareMask = (1ull << 24) - 1;

static constexpr int ring_smem_bytes() {
  return kWarpsPerBlock * kRing * (kSliceBytes + (int)sizeof(uint64_t) + (int)sizeof(SliceMeta)) +
         (int)sizeof(ShareState);
}

// Take the next slice of warp v's shared chunk in two halves: share_fetch
// issues the atomic (lane 0 keeps the raw word, not yet waited on), and
// share_decode broadcasts it -- true with [sb, sb + cnt) of species isp,
// false when that chunk was exhausted.  The owner fetches its next take one
// slice ahead, so the shared-memory atomic's latency stays off the issue
// path (taken back to back it cost config 3 ~3% of the push).  Warp-collective.
__device__ __forceinline__ unsigned long long share_fetch(ShareState *sh, int v) {
  unsigned long long old = 0;
  if (lane_id() == 0) old = atomicAdd(&sh->word[v], 1ull << kShareSliceShift);
  return old;
}
__device__ __forceinline__ bool share_decode(const ShareState *sh, int v, unsigned long long raw, int64_t &sb,
                                             int &cnt, int &isp, uint32_t &gen) {
  const unsigned long long old = __shfl_sync(0xffffffffu, raw, 0);
  gen = (uint32_t)(old >> 48);
  const unsigned long long idx = (old >> kShareSliceShift) & kShareMask, n = old & kShareMask;
  if (idx >= n) return false;
  const ShareChunk c = sh->gen[v][gen & 1];
  sb = c.base + (int64_t)idx * kSlice;
  cnt = (int)(c.end - sb < kSlice ? c.end - sb : kSlice);
  isp = c.isp;
  return true;
}
__device__ __forceinline__ bool share_take(ShareState *sh, int v, int64_t &sb, int &cnt, int &isp,
                                           uint32_t &gen) {
  return share_decode(sh, v, share_fetch(sh, v), sb, cnt, isp, gen);
}

// Owner: publish [beg, end) of species isp as warp w's next chunk generation.
__device__ __forceinline__ void share_install(ShareState *sh, int w, uint32_t gen, int64_t beg, int64_t end,
                                              int isp) {
  if (lane_id() == 0) {
    ShareChunk &c = sh->gen[w][(gen + 1) & 1];
    c.base = beg;
    c.end = end;
    c.isp = isp;
    __threadfence_block();
    const unsigned long long n = (unsigned long long)((end - beg + kSlice - 1) / kSlice);
    atomicExch(&sh->word[w], ((unsigned long long)((gen + 1) & 0xffff) << 48) | n);
  }
  __syncwarp();
}

// Once the work lists are drained: the leftover ring slices of the block's
// ring warps [0, nring), through the register path (any warp of the block).
template <int BC>
__device__ __forceinline__ void steal_ring_slices(const LaunchArgs &a, ShareState *share, int w, int nring,
                                                  Window &win, Tally &t, int &cur) {
  const int lane = (int)lane_id();
  for (int v = 1; v <= nring; ++v) {
    const int victim = (w + v) % kWarpsPerBlock;
    if (victim >= nring || victim == w) continue;
    int64_t sb;
    int cnt, isp;
    uint32_t gen;
    while (share_take(share, victim, sb, cnt, isp, gen)) {
      const pb_species &s = a.sp[isp];
      if (isp != cur) {
        if (cur >= 0) flush_tally(a, a.id[cur], t, nullptr);
        t = Tally();
        cur = isp;
        win.gR = a.bins + (size_t)s.deposit * 2 * (size_t)a.nc;
        win.gC = win.gR + a.nc;
      }
      Quad<PB_KIND_KICK, false> q;
      const int64_t i = sb + 4 * lane;
      quad_load<PB_KIND_KICK, false>(s, i, sb + cnt, q);
      if (PB_FULL_SLICES && cnt == kSlice)
        quad_process<PB_KIND_KICK, false, BC, true, true>(a, isp, i, q, win, t);
      else
        quad_process<PB_KIND_KICK, false, BC, true>(a, isp, i, q, win, t);
    }
  }
}

template <int BC>
__global__ void __launch_bounds__(kThreads, PB_QUAD_MINBLOCKS)
    k_push_ring(const __grid_constant__ LaunchArgs a) {
  pdl_enter();
  mover_clock_start(a.st);
  extern __shared__ __align__(128) unsigned char r_smem[];
  const int lane = (int)lane_id();
  const int w = threadIdx.x >> 5;
  uint64_t *bars = reinterpret_cast<uint64_t *>(r_smem + (size_t)kWarpsPerBlock * kRing * kSliceBytes);
  SliceMeta *metas = reinterpret_cast<SliceMeta *>(bars + kWarpsPerBlock * kRing);
  ShareState *share = reinterpret_cast<ShareState *>(metas + kWarpsPerBlock * kRing);
  const WarpRing r{r_smem + (size_t)w * kRing * kSliceBytes, bars + w * kRing, metas + w * kRing};
  if (lane == 0) {
    for (int k = 0; k < kRing; ++k) mbar_init(&r.bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    share->word[w] = 0;  // generation 0, no slices: the first take claims
  }
  __syncthreads();  // every warp's share word is initialised before any thief reads it
  const int64_t total = a.tile_start[a.nsp];
  Window win{nullptr, nullptr, 0, 0, nullptr, nullptr};
  Tally t;
  int cur = -1;
  bool issuing = true;
  uint32_t head = 0, tail = 0;
  unsigned long long pend = share_fetch(share, w);  // lane 0: the take of the next slice
  auto issue = [&]() {
    int64_t ibeg;
    int cnt, iisp;
    uint32_t gen;
    while (!share_decode(share, w, pend, ibeg, cnt, iisp, gen)) {  // own chunk exhausted: claim the next
      const int64_t c = claim_chunk(a);
      if (c >= total) {
        issuing = false;
        return;
      }
      int64_t beg, end;
      const int isp = chunk_species(a, c, beg, end);
      if (end > beg) share_install(share, w, gen, beg, end, isp);
      pend = share_fetch(share, w);
    }
    pend = share_fetch(share, w);  // one slice ahead: waited on at the next issue
    const uint32_t st = head % kRing;
    if (lane == 0) {
      r.meta[st].base = ibeg;
      r.meta[st].isp = iisp;
      r.meta[st].cnt = cnt;
      if (cnt == kSlice) {
        const pb_species &s = a.sp[iisp];
        unsigned char *b = r.buf + st * kSliceBytes;
        mbar_expect_tx(&r.bar[st], (uint32_t)kSliceBytes);
        tma_load_1d(b, s.x + ibeg, kSlice * 8, &r.bar[st]);
        tma_load_1d(b + kSlice * 8, s.vx + ibeg, kSlice * 8, &r.bar[st]);
        tma_load_1d(b + kSlice * 16, s.cell + ibeg, kSlice * 4, &r.bar[st]);
      } else {
        mbar_arrive(&r.bar[st]);  // partial slice: loaded directly, phase still completes
      }
    }
    ++head;
  };
  while (issuing && head - tail < (uint32_t)kRing) issue();
  while (tail != head) {
    const uint32_t st = tail % kRing;
    mbar_wait(&r.bar[st], (tail / kRing) & 1u);
    const SliceMeta m = r.meta[st];
    const pb_species &s = a.sp[m.isp];
    if (m.isp != cur) {
      if (cur >= 0) flush_tally(a, a.id[cur], t, nullptr);
      t = Tally();
      cur = m.isp;
      win.gR = a.bins + (size_t)s.deposit * 2 * (size_t)a.nc;
      win.gC = win.gR + a.nc;
    }
    Quad<PB_KIND_KICK, false> q;
    const int64_t i = m.base + 4 * lane;
    if (m.cnt == kSlice) {
      const unsigned char *b = r.buf + st * kSliceBytes;
      const double2 *px = reinterpret_cast<const double2 *>(b) + 2 * lane;
      const double2 *pv = reinterpret_cast<const double2 *>(b + kSlice * 8) + 2 * lane;
      const int4 cc = reinterpret_cast<const int4 *>(b + kSlice * 16)[lane];
      const double2 x01 = px[0], x23 = px[1], v01 = pv[0], v23 = pv[1];
      q.x[0] = x01.x; q.x[1] = x01.y; q.x[2] = x23.x; q.x[3] = x23.y;
      q.vx[0] = v01.x; q.vx[1] = v01.y; q.vx[2] = v23.x; q.vx[3] = v23.y;
      q.c[0] = cc.x; q.c[1] = cc.y; q.c[2] = cc.z; q.c[3] = cc.w;
#pragma unroll
      for (int k = 0; k < 4; ++k) q.vy[k] = q.vz[k] = q.y[k] = 0.0;
      q.base = 0;
      q.packed = 0;
      q.nv = 4;
    } else {
      quad_load<PB_KIND_KICK, false>(s, i, m.base + m.cnt, q);
    }
    __syncwarp();  // every lane holds its slice in registers: the stage may be refilled
    ++tail;
    if (issuing) issue();
    if (PB_FULL_SLICES && m.cnt == kSlice)
      quad_process<PB_KIND_KICK, false, BC, true, true>(a, m.isp, i, q, win, t);
    else
      quad_process<PB_KIND_KICK, false, BC, true>(a, m.isp, i, q, win, t);
  }
  // the global counter is dry and this warp's ring is drained: take the
  // leftover slices of the block's other warps
  steal_ring_slices<BC>(a, share, w, kWarpsPerBlock, win, t, cur);
  if (cur >= 0) flush_tally(a, a.id[cur], t, nullptr);
  if (lane == 0) release_work_counter(a.st, (unsigned long long)gridDim.x * kWarpsPerBlock);
}

// ---------------------------------------------------------------------------
// Split mover for mixed launches: warps w < kSplitRingWarps of every block
// stream the ring-eligible charged species (list 0) through their private
// TMA rings; the other warps run the register path over the rest (list 1,
// the neutral slices).  Both kinds stay resident on every SM; a warp whose
// list runs dry moves on to the other list (register path), so the tails
// balance.  The ring stages the 1-byte cell index where the species has one.
// ---------------------------------------------------------------------------
#ifndef PB_SPLIT_RING_WARPS
#define PB_SPLIT_RING_WARPS 6
#endif
#ifndef PB_SPLIT_STAGES
#define PB_SPLIT_STAGES 2
#endif
constexpr int kSplitRingWarps = PB_SPLIT_RING_WARPS;
constexpr int kSplitStages = PB_SPLIT_STAGES;

// (No slice sharing here: the per-slice shared-memory atomic on the ring
// warps' issue path cost config 2 3.5% of the push, more than its tail
// gained -- profiles/r02_mover_tail.txt.)
static constexpr int split_smem_bytes() {
  return kSplitRingWarps * kSplitStages * (kSliceBytes + (int)sizeof(uint64_t) + (int)sizeof(SliceMeta));
}


__device__ __forceinline__ int list_chunk(const LaunchArgs &a, const ChunkList &L, int64_t c,
                                          int64_t &beg, int64_t &end) {
  int kk = 0;
  int64_t local;
  if (c < L.rr_chunks) {
    kk = (int)(c % L.nsp);
    local = c / L.nsp;
  } else {
    const int64_t r = c - L.rr_chunks;
    while (kk + 1 < L.nsp && r >= L.tail_start[kk + 1]) ++kk;
    local = L.rr_each + (r - L.tail_start[kk]);
  }
  const int isp = L.order[kk];
  const pb_species &s = a.sp[isp];
  const int64_t n = s.n_dev ? *s.n_dev : s.n;
  beg = local * a.chunk;
  end = beg + a.chunk < n ? beg + a.chunk : n;
  return isp;
}

__device__ __forceinline__ int64_t claim_from(unsigned long long *ctr) {
  unsigned long long c = 0;
  if (lane_id() == 0) c = atomicAdd(ctr, 1ull);
  return (int64_t)__shfl_sync(0xffffffffu, c, 0);
}

template <int BC>
__device__ __forceinline__ void split_register_list(const LaunchArgs &a, int g, Window &win,
                                                    Tally &t, int &cur) {
  const ChunkList &L = a.lists[g];
  unsigned long long *ctr = (unsigned long long *)(g == 0 ? &a.st->tile_next : &a.st->tile_next2);
  const int64_t total = L.tile_start[L.nsp];
  for (int64_t c = claim_from(ctr); c < total; c = claim_from(ctr)) {
    int64_t beg, end;
    const int isp = list_chunk(a, L, c, beg, end);
    const pb_species &s = a.sp[isp];
    if (isp != cur) {
      if (cur >= 0) flush_tally(a, a.id[cur], t, nullptr);
      t = Tally();
      cur = isp;
      if (s.deposit >= 0 && a.bins) {
        win.gR = a.bins + (size_t)s.deposit * 2 * (size_t)a.nc;
        win.gC = win.gR + a.nc;
      }
    }
    if (g == 0)  // list 0 is ring-eligible by construction: KICK, no yp, depositing
      quad_chunk<PB_KIND_KICK, false, BC, true>(a, isp, beg, end, win, t);
    else
      quad_dispatch<BC, false>(a, isp, beg, end, win, t);
  }
}

template <int BC>
__global__ void __launch_bounds__(kThreads, PB_QUAD_MINBLOCKS)
    k_push_split(const __grid_constant__ LaunchArgs a) {
  pdl_enter();
  mover_clock_start(a.st);
  extern __shared__ __align__(128) unsigned char s_smem[];
  const int lane = (int)lane_id();
  const int w = threadIdx.x >> 5;
  Window win{nullptr, nullptr, 0, 0, nullptr, nullptr};
  Tally t;
  int cur = -1;
  if (w < kSplitRingWarps) {
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_smem + (size_t)kSplitRingWarps * kSplitStages * kSliceBytes);
    SliceMeta *metas = reinterpret_cast<SliceMeta *>(bars + kSplitRingWarps * kSplitStages);
    const WarpRing r{s_smem + (size_t)w * kSplitStages * kSliceBytes, bars + w * kSplitStages,
                     metas + w * kSplitStages};
    if (lane == 0) {
      for (int k = 0; k < kSplitStages; ++k) mbar_init(&r.bar[k], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const ChunkList &L = a.lists[0];
    const int64_t total = L.tile_start[L.nsp];
    unsigned long long *ctr = (unsigned long long *)&a.st->tile_next;
    int64_t ibeg = 0, iend = 0;
    int iisp = 0;
    bool issuing = true;
    uint32_t head = 0, tail = 0;
    auto issue = [&]() {
      while (ibeg >= iend) {
        const int64_t c = claim_from(ctr);
        if (c >= total) {
          issuing = false;
          return;
        }
        iisp = list_chunk(a, L, c, ibeg, iend);
      }
      const int cnt = (int)(iend - ibeg < kSlice ? iend - ibeg : kSlice);
      const uint32_t st = head % kSplitStages;
      if (lane == 0) {
        r.meta[st].base = ibeg;
        r.meta[st].isp = iisp;
        r.meta[st].cnt = cnt;
        if (cnt == kSlice) {
          const pb_species &s = a.sp[iisp];
          unsigned char *b = r.buf + st * kSliceBytes;
          const uint32_t cb = s.cell8 ? kSlice : kSlice * 4;
          mbar_expect_tx(&r.bar[st], (uint32_t)(kSlice * 16) + cb);
          tma_load_1d(b, s.x + ibeg, kSlice * 8, &r.bar[st]);
          tma_load_1d(b + kSlice * 8, s.vx + ibeg, kSlice * 8, &r.bar[st]);
          if (s.cell8)
            tma_load_1d(b + kSlice * 16, s.cell8 + ibeg, kSlice, &r.bar[st]);
          else
            tma_load_1d(b + kSlice * 16, s.cell + ibeg, kSlice * 4, &r.bar[st]);
        } else {
          mbar_arrive(&r.bar[st]);
        }
      }
      ibeg += cnt;
      ++head;
    };
    while (issuing && head - tail < (uint32_t)kSplitStages) issue();
    while (tail != head) {
      const uint32_t st = tail % kSplitStages;
      mbar_wait(&r.bar[st], (tail / kSplitStages) & 1u);
      const SliceMeta m = r.meta[st];
      const pb_species &s = a.sp[m.isp];
      if (m.isp != cur) {
        if (cur >= 0) flush_tally(a, a.id[cur], t, nullptr);
        t = Tally();
        cur = m.isp;
        win.gR = a.bins + (size_t)s.deposit * 2 * (size_t)a.nc;
        win.gC = win.gR + a.nc;
      }
      Quad<PB_KIND_KICK, false> q;
      const int64_t i = m.base + 4 * lane;
      if (m.cnt == kSlice) {
        const unsigned char *b = r.buf + st * kSliceBytes;
        const double2 *px = reinterpret_cast<const double2 *>(b) + 2 * lane;
        const double2 *pv = reinterpret_cast<const double2 *>(b + kSlice * 8) + 2 * lane;
        const double2 x01 = px[0], x23 = px[1], v01 = pv[0], v23 = pv[1];
        q.x[0] = x01.x; q.x[1] = x01.y; q.x[2] = x23.x; q.x[3] = x23.y;
        q.vx[0] = v01.x; q.vx[1] = v01.y; q.vx[2] = v23.x; q.vx[3] = v23.y;
        if (s.cell8) {
          q.base = __ldg(s.chunk_base + i / PB_CELL8_CHUNK);
          q.packed = reinterpret_cast<const int *>(b + kSlice * 16)[lane];
          q.c[0] = kPackedCells;
          q.c[1] = q.c[2] = q.c[3] = 0;
        } else {
          const int4 cc = reinterpret_cast<const int4 *>(b + kSlice * 16)[lane];
          q.c[0] = cc.x; q.c[1] = cc.y; q.c[2] = cc.z; q.c[3] = cc.w;
          q.base = 0;
          q.packed = 0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) q.vy[k] = q.vz[k] = q.y[k] = 0.0;
        q.nv = 4;
      } else {
        quad_load<PB_KIND_KICK, false>(s, i, m.base + m.cnt, q);
      }
      __syncwarp();
      ++tail;
      if (issuing) issue();
      if (PB_FULL_SLICES && m.cnt == kSlice)
        quad_process<PB_KIND_KICK, false, BC, true, true>(a, m.isp, i, q, win, t);
      else
        quad_process<PB_KIND_KICK, false, BC, true>(a, m.isp, i, q, win, t);
    }
    split_register_list<BC>(a, 1, win, t, cur);
  } else {
    split_register_list<BC>(a, 1, win, t, cur);
    split_register_list<BC>(a, 0, win, t, cur);
  }
  if (cur >= 0) flush_tally(a, a.id[cur], t, nullptr);
  if (lane == 0) release_work_counter(a.st, (unsigned long long)gridDim.x * kWarpsPerBlock);
}

// ---------------------------------------------------------------------------
// Host side.
//
// Kernel choice (measured on configs 2-5):
//   every species pushed, mixed charged + other kinds  -> k_push_split
//   every species pushed, all KICK without yp (config 3) -> k_push_ring
//   every species pushed, otherwise (Boris, config 4)    -> k_push_quad
//   deposit-only launches, or inactive depositing species -> k_push_deposit
// Compile-time A/B switches (scripts/variants.txt builds them with EXTRA=-D...):
//   PB_SPLIT (1), PB_RING (1), PB_SPLIT_SOLO (0), PB_INTERLEAVE (1),
//   PB_CLAIM_CHUNK (0 = by launch size).
// ---------------------------------------------------------------------------
#ifndef PB_SPLIT
#define PB_SPLIT 1
#endif
#ifndef PB_RING
#define PB_RING 1
#endif
#ifndef PB_SPLIT_SOLO
#define PB_SPLIT_SOLO 0
#endif
#ifndef PB_INTERLEAVE
#define PB_INTERLEAVE 1
#endif
#ifndef PB_CLAIM_CHUNK
#define PB_CLAIM_CHUNK 0
#endif

static int g_sm_count = 0;
typedef void (*KernFn)(LaunchArgs);
static const char *g_last_kernel = "";

static int sm_count() {
  if (g_sm_count == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_sm_count;
}

static int occupancy(const void *fn, int threads, int smem, int *bps) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
  // Pin the L1 / shared-memory split to the smallest shared carve-out that
  // holds PB_QUAD_MINBLOCKS blocks: the rest stays L1, which the register-
  // path loads need for their in-flight sectors (left to the driver, the
  // split varied between processes and so did the mover's speed).
  {
    const int per_sm = (smem + 1024) * PB_QUAD_MINBLOCKS;
    int pct = smem > 0 ? (per_sm * 100 + 233471) / 233472 : 0;  // of 228 KB
    if (pct > 100) pct = 100;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(carveout)");
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, fn, threads, smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (*bps < 1) *bps = 1;
  return PB_OK;
}

// Approximate HBM bytes per particle, used to balance blocks and order chunks.
static double bytes_per_particle(const pb_species &s, bool push) {
  if (!push) return 12.0;
  const bool yp = s.yp != nullptr;
  switch (s.kind) {
    case PB_KIND_KICK: return 36.0 + (yp ? 24.0 : 0.0);
    case PB_KIND_BORIS: return 68.0 + (yp ? 24.0 : 0.0);
    case PB_KIND_DRIFT: return 24.0 + (yp ? 24.0 : 0.0) + (s.deposit >= 0 ? 4.0 : 0.0);
    default: return s.deposit >= 0 ? 12.0 : 0.0;
  }
}

// Chunk list over the species slots gs[0..n) (heaviest bytes first): the
// first rr_each chunks of every species round-robin (charged chunks are
// latency-heavier than neutral ones; a mix keeps the memory system busy),
// then species by species.
static void build_list(const LaunchArgs &a, const int *gs, int n, ChunkList &L) {
  L.nsp = n;
  L.tile_start[0] = 0;
  int64_t mn = -1;
  for (int k = 0; k < n; ++k) {
    L.order[k] = gs[k];
    const int64_t nk = (a.sp[gs[k]].n + a.chunk - 1) / a.chunk;
    L.tile_start[k + 1] = L.tile_start[k] + nk;
    if (mn < 0 || nk < mn) mn = nk;
  }
  L.rr_each = PB_INTERLEAVE ? mn : 0;
  L.rr_chunks = L.rr_each * n;
  L.tail_start[0] = 0;
  for (int k = 0; k < n; ++k)
    L.tail_start[k + 1] = L.tail_start[k] + (L.tile_start[k + 1] - L.tile_start[k]) - L.rr_each;
}

static int launch_persistent(KernFn fn, const char *name, int smem, const LaunchArgs &a,
                             cudaStream_t stream) {
  int bps = 0;
  int rc = occupancy((const void *)fn, kThreads, smem, &bps);
  if (rc) return rc;
  cudaError_t le = launch_pdl(fn, dim3(sm_count() * bps), dim3(kThreads), smem, stream, a);
  if (le != cudaSuccess) return cuda_status(le, name);
  g_last_kernel = name;
  return PB_OK;
}

static int launch(const pb_species *sp, int nsp, const double *e, int64_t nc, int bc, bool push,
                  uint64_t *bins, pb_status *st, cudaStream_t stream) {
  if (nsp < 0 || nsp > PB_MAX_SPECIES) {
    set_error("nsp=%d outside [0, %d]", nsp, PB_MAX_SPECIES);
    return PB_ERR_INVALID;
  }
  if (nc < 1 || nc > 0x7fffffffLL) {
    set_error("nc=%lld outside [1, 2^31)", (long long)nc);
    return PB_ERR_INVALID;
  }
  if (bc != PB_BC_PERIODIC && bc != PB_BC_ABSORBING) {
    set_error("unknown particle boundary %d", bc);
    return PB_ERR_INVALID;
  }
  if (st == nullptr) {
    set_error("status pointer is NULL");
    return PB_ERR_INVALID;
  }
  LaunchArgs a;
  memset(&a, 0, sizeof(a));
  a.chunk = kChunk;
  a.push = push ? 1 : 0;
  a.e = e;
  a.nc = nc;
  a.bins = bins;
  a.st = st;
  double w[PB_MAX_SPECIES];
  double wsum = 0.0;
  bool all_move = true;
  for (int k = 0; k < nsp; ++k) {
    const pb_species &s = sp[k];
    const bool dep = s.deposit >= 0 && bins != nullptr;
    const bool moves = push && s.kind != PB_KIND_INACTIVE;
    if (s.n <= 0 || (!moves && !dep)) continue;
    if (!s.x || !s.cell) {
      set_error("species %d: x/cell pointers are NULL", k);
      return PB_ERR_INVALID;
    }
    if (moves && (s.kind == PB_KIND_KICK || s.kind == PB_KIND_BORIS) && !e) {
      set_error("species %d is charged but e_nodes is NULL", k);
      return PB_ERR_INVALID;
    }
    if (moves && !s.vx) {
      set_error("species %d: vx pointer is NULL", k);
      return PB_ERR_INVALID;
    }
    if (moves && (s.yp || s.kind == PB_KIND_BORIS) && !s.vy) {
      set_error("species %d: vy pointer is NULL", k);
      return PB_ERR_INVALID;
    }
    if (moves && s.kind == PB_KIND_BORIS && !s.vz) {
      set_error("species %d: vz pointer is NULL", k);
      return PB_ERR_INVALID;
    }
    if (bc == PB_BC_ABSORBING && moves && (!s.holes || !s.n_dev)) {
      set_error("species %d: absorbing walls need holes and n_dev", k);
      return PB_ERR_INVALID;
    }
    if (((uintptr_t)s.x | (uintptr_t)s.vx | (uintptr_t)s.vy | (uintptr_t)s.vz | (uintptr_t)s.yp |
         (uintptr_t)s.cell) & 15u) {
      set_error("species %d: arrays must be 16-byte aligned", k);
      return PB_ERR_INVALID;
    }
    a.id[a.nsp] = k;
    a.sp[a.nsp] = s;
    if (!moves) {
      a.sp[a.nsp].kind = PB_KIND_INACTIVE;
      all_move = false;
    }
    w[a.nsp] = (double)s.n * bytes_per_particle(a.sp[a.nsp], push);
    wsum += w[a.nsp];
    a.nsp++;
  }
  if (a.nsp == 0) return PB_OK;
  const int sms = sm_count();
  if (sms == 0) return cuda_status(cudaGetLastError(), "device query");

  if (push && all_move) {
    // Chunk list: species by descending bytes/particle.
    int order[PB_MAX_SPECIES];
    bool boris = false, bgather = false, bonly = true;
    for (int k = 0; k < a.nsp; ++k) {
      order[k] = k;
      boris |= a.sp[k].kind == PB_KIND_BORIS;
      bgather |= a.sp[k].kind == PB_KIND_BORIS && a.sp[k].b_nodes != nullptr;
      // gathered-B only: every charged mover a gathered-B Boris species
      if (a.sp[k].kind == PB_KIND_KICK || (a.sp[k].kind == PB_KIND_BORIS && !a.sp[k].b_nodes)) bonly = false;
    }
    for (int i = 1; i < a.nsp; ++i)
      for (int j = i; j > 0 && bytes_per_particle(a.sp[order[j]], true) >
                                   bytes_per_particle(a.sp[order[j - 1]], true); --j) {
        const int tmp = order[j];
        order[j] = order[j - 1];
        order[j - 1] = tmp;
      }
    // Claim granularity: 1024-particle chunks (a shorter tail) unless the
    // launch is large enough that 2048 still gives every warp >= 64 chunks.
    // Measured (profiles/r01h_claim_chunk_ab.jsonl): 1024 is -1.4% push on
    // config 2, -1.4% config 3 (ring), -1.4% config 4; config 5 (1B
    // particles, ~140 chunks per warp at 2048) is +5% slower at 1024.
    // PB_CLAIM_CHUNK (compile time) pins it (a power of two from 256 to
    // 2048: chunks never straddle a cell8 chunk).
    {
      int64_t work = 0;
      for (int k = 0; k < a.nsp; ++k) work += a.sp[k].n;
      const int64_t warps = (int64_t)sms * 3 * kWarpsPerBlock;
      constexpr int claim = PB_CLAIM_CHUNK;
      if (claim >= 256 && claim <= kChunk && (claim & (claim - 1)) == 0)
        a.chunk = claim;
      else
        a.chunk = work < warps * 64 * (int64_t)kChunk ? kChunk / 2 : kChunk;
    }
    ChunkList all;
    build_list(a, order, a.nsp, all);
    for (int k = 0; k < a.nsp; ++k) a.order[k] = all.order[k];
    for (int k = 0; k <= a.nsp; ++k) {
      a.tile_start[k] = all.tile_start[k];
      a.tail_start[k] = all.tail_start[k];
    }
    a.rr_each = all.rr_each;
    a.rr_chunks = all.rr_chunks;
    // mixed launches with ring-eligible charged species and other species:
    // the warp-specialised split kernel, measured 3-4% faster than the quad
    // kernel on config 2
    if (PB_SPLIT && !boris) {
      int g0[PB_MAX_SPECIES], g1[PB_MAX_SPECIES], n0 = 0, n1 = 0;
      for (int k = 0; k < a.nsp; ++k) {
        const int sk = order[k];  // heaviest bytes first within each list
        const pb_species &sp2 = a.sp[sk];
        const bool elig = sp2.kind == PB_KIND_KICK && !sp2.yp && sp2.deposit >= 0 && bins;
        if (elig) g0[n0++] = sk; else g1[n1++] = sk;
      }
      if (n0 > 0 && (n1 > 0 || PB_SPLIT_SOLO)) {
        build_list(a, g0, n0, a.lists[0]);
        build_list(a, g1, n1, a.lists[1]);
        return launch_persistent(bc == PB_BC_PERIODIC ? k_push_split<PB_BC_PERIODIC>
                                                      : k_push_split<PB_BC_ABSORBING>,
                                 "k_push_split", split_smem_bytes(), a, stream);
      }
    }
    // charged-only launches (every species KICK without yp, depositing, on
    // the full int32 cell index): the per-warp TMA ring kernel
    bool ring = PB_RING;
    for (int k = 0; k < a.nsp && ring; ++k)
      ring = a.sp[k].kind == PB_KIND_KICK && !a.sp[k].yp && a.sp[k].deposit >= 0 && bins &&
             !a.sp[k].cell8;
    if (ring)
      return launch_persistent(bc == PB_BC_PERIODIC ? k_push_ring<PB_BC_PERIODIC>
                                                    : k_push_ring<PB_BC_ABSORBING>,
                               "k_push_ring", ring_smem_bytes(), a, stream);
    KernFn fn = bc == PB_BC_PERIODIC
                    ? (bgather ? (bonly ? k_push_quad<PB_BC_PERIODIC, 2> : k_push_quad<PB_BC_PERIODIC, 3>)
                               : boris ? k_push_quad<PB_BC_PERIODIC, 1> : k_push_quad<PB_BC_PERIODIC, 0>)
                    : (bgather ? (bonly ? k_push_quad<PB_BC_ABSORBING, 2> : k_push_quad<PB_BC_ABSORBING, 3>)
                               : boris ? k_push_quad<PB_BC_ABSORBING, 1> : k_push_quad<PB_BC_ABSORBING, 0>);
    return launch_persistent(fn, "k_push_quad", 0, a, stream);
  }
  // Deposit-only launches and launches with inactive depositing species:
  // static contiguous chunks per block, shared-memory deposit window.
  KernFn fn = bc == PB_BC_PERIODIC
                  ? (push ? k_push_deposit<PB_BC_PERIODIC, true> : k_push_deposit<PB_BC_PERIODIC, false>)
                  : (push ? k_push_deposit<PB_BC_ABSORBING, true> : k_push_deposit<PB_BC_ABSORBING, false>);
  int bps = 0;
  int rc = occupancy((const void *)fn, kThreads, 0, &bps);
  if (rc) return rc;
  const int grid = sms * bps;
  int start = 0;
  for (int k = 0; k < a.nsp; ++k) {
    const int64_t tiles = (a.sp[k].n + kTile - 1) / kTile;
    int64_t nb = (int64_t)(grid * (w[k] / wsum) + 0.5);
    if (nb < 1) nb = 1;
    if (nb > tiles) nb = tiles;
    a.blk_start[k] = start;
    start += (int)nb;
  }
  a.blk_start[a.nsp] = start;
  fn<<<start, kThreads, 0, stream>>>(a);
  PB_CHECK_LAUNCH("k_push_deposit");
  g_last_kernel = "k_push_deposit";
  return PB_OK;
}

}  // namespace pb

extern "C" int pb_push_deposit(const pb_species *sp, int nsp, const double *e_nodes, int64_t nc,
                               int particle_bc, uint64_t *bins, pb_status *status, void *stream) {
  return pb::launch(sp, nsp, e_nodes, nc, particle_bc, true, bins, status, (cudaStream_t)stream);
}

extern "C" int pb_deposit_only(const pb_species *sp, int nsp, int64_t nc, uint64_t *bins,
                               pb_status *status, void *stream) {
  if (!bins) {
    pb::set_error("bins pointer is NULL");
    return PB_ERR_INVALID;
  }
  return pb::launch(sp, nsp, nullptr, nc, PB_BC_PERIODIC, false, bins, status, (cudaStream_t)stream);
}

extern "C" const char *pb_last_mover_kernel(void) { return pb::g_last_kernel; }

#ifdef PB_MOVER_TRACE
// debug: the last launch's block starts and per-warp finish times (globaltimer ns)
extern "C" int pb_debug_warp_ends(unsigned long long *out, int n, unsigned long long *starts, int nb) {
  if (n > 8192) n = 8192;
  if (nb > 2048) nb = 2048;
  if (cudaMemcpyFromSymbol(out, pb::g_warp_end, (size_t)n * sizeof(unsigned long long)) != cudaSuccess)
    return PB_ERR_CUDA;
  return cudaMemcpyFromSymbol(starts, pb::g_blk_start, (size_t)nb * sizeof(unsigned long long)) == cudaSuccess
             ? PB_OK
             : PB_ERR_CUDA;
}
// debug: the mover launch log (first block start, last warp end) and its count
extern "C" int pb_debug_mover_log(unsigned long long *out, unsigned long long *count) {
  if (cudaMemcpyFromSymbol(out, pb::g_mlog, sizeof(pb::g_mlog)) != cudaSuccess) return PB_ERR_CUDA;
  return cudaMemcpyFromSymbol(count, pb::g_mlog_n, sizeof(unsigned long long)) == cudaSuccess ? PB_OK
                                                                                            : PB_ERR_CUDA;
}
#endif
