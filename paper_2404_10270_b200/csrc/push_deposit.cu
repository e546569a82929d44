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
#include <cstring>

#include "common.cuh"

namespace pb {

constexpr int kThreads = 256;
constexpr int kPairsPerThread = 2;
constexpr int kTile = kThreads * 2 * kPairsPerThread;  // 1024 particles
constexpr int kWin = 1024;    // shared-memory deposit window, cells
constexpr int kMargin = 64;   // cells kept left of the chunk's first cell

struct LaunchArgs {
  pb_species sp[PB_MAX_SPECIES];
  int blk_start[PB_MAX_SPECIES + 1];
  int id[PB_MAX_SPECIES];  // caller species index (status arrays)
  int nsp;
  int push;  // 0: deposit only (no mover)
  const double *e;
  int64_t nc;
  uint64_t *bins;
  pb_status *st;
};

// ---------------------------------------------------------------------------
// Per-particle mover arithmetic.  Returns the new state in place.
// ---------------------------------------------------------------------------
struct MoveOut {
  int32_t cell;
  bool moved;      // cell changed (or removed)
  int8_t wall;     // -1 none, 0 left, 1 right (absorbing only)
  bool cfl;        // |floor(x)| >= nc
};

template <int KIND>
__device__ __forceinline__ void kick_drift(double &x, double &vx, double &vy,
                                           double &vz, int32_t cell,
                                           const pb_species &s,
                                           const double *__restrict__ e) {
  if (KIND == PB_KIND_KICK) {
    const double aj = __dmul_rn(s.kick_coef, __ldg(e + cell));
    const double aj1 = __dmul_rn(s.kick_coef, __ldg(e + cell + 1));
    const double daj = __dsub_rn(aj1, aj);
    const double atemp = __dadd_rn(aj, __dmul_rn(x, daj));
    const double v = __dadd_rn(vx, atemp);
    vx = v;
    x = __dadd_rn(x, __dmul_rn(s.fnstep, v));
  } else if (KIND == PB_KIND_BORIS) {
    // Boris (config 4, restated in oracle/picmc_oracle.c:boris_push):
    // half kick, rotation v' = v- + v- x t, v+ = v- + v' x s, half kick.
    const double aj = __dmul_rn(s.kick_coef, __ldg(e + cell));
    const double aj1 = __dmul_rn(s.kick_coef, __ldg(e + cell + 1));
    const double daj = __dsub_rn(aj1, aj);
    const double atemp = __dadd_rn(aj, __dmul_rn(x, daj));
    const double h = __dmul_rn(0.5, atemp);
    const double tx = s.boris_t[0], ty = s.boris_t[1], tz = s.boris_t[2];
    const double sx = s.boris_s[0], sy = s.boris_s[1], sz = s.boris_s[2];
    const double mx = __dadd_rn(vx, h), my = vy, mz = vz;
    const double px = __dadd_rn(mx, __dsub_rn(__dmul_rn(my, tz), __dmul_rn(mz, ty)));
    const double py = __dadd_rn(my, __dsub_rn(__dmul_rn(mz, tx), __dmul_rn(mx, tz)));
    const double pz = __dadd_rn(mz, __dsub_rn(__dmul_rn(mx, ty), __dmul_rn(my, tx)));
    const double qx = __dadd_rn(mx, __dsub_rn(__dmul_rn(py, sz), __dmul_rn(pz, sy)));
    const double qy = __dadd_rn(my, __dsub_rn(__dmul_rn(pz, sx), __dmul_rn(px, sz)));
    const double qz = __dadd_rn(mz, __dsub_rn(__dmul_rn(px, sy), __dmul_rn(py, sx)));
    vx = __dadd_rn(qx, h);
    vy = qy;
    vz = qz;
    x = __dadd_rn(x, __dmul_rn(s.fnstep, vx));
  } else {  // PB_KIND_DRIFT: no kick at all (keeps -0.0, mover.py:214-216)
    x = __dadd_rn(x, __dmul_rn(s.fnstep, vx));
  }
}

// Cell transfer (resort_collect, pkg/src/picmc/mover.py:136-163):
//   delta = floor(x); movers have delta != 0; CFL if |delta| >= nc;
//   dest = (src + delta) mod nc; new_x = x - delta;
//   carry: new_x >= 1.0 -> new_x -= 1.0, dest = (dest + 1) mod nc.
// Absorbing walls remove a mover whose unwrapped dest leaves [0, nc).
template <int BC>
__device__ __forceinline__ MoveOut transfer(double &x, int32_t cell,
                                            int64_t nc) {
  MoveOut o{cell, false, -1, false};
  const double d = floor(x);
  if (d != 0.0) {
    if (fabs(d) >= (double)nc) {
      o.cfl = true;
      return o;
    }
    int64_t dest = (int64_t)cell + (int64_t)d;
    double nx = __dsub_rn(x, d);
    if (nx >= 1.0) {
      nx = __dsub_rn(nx, 1.0);
      dest += 1;
    }
    x = nx;
    o.moved = true;
    if (BC == PB_BC_PERIODIC) {
      o.cell = (int32_t)floor_mod(dest, nc);
    } else {
      if (dest < 0) {
        o.wall = 0;
        o.cell = -1;
      } else if (dest >= nc) {
        o.wall = 1;
        o.cell = -1;
      } else {
        o.cell = (int32_t)dest;
      }
    }
  }
  return o;
}

// ---------------------------------------------------------------------------
// Deposit emission: warp segmented reduction of packed (count, R) words keyed
// by cell, then shared-memory window atomics or global atomics.
// ---------------------------------------------------------------------------
struct Window {
  uint64_t *sR;
  uint32_t *sC;
  int64_t base;
  uint64_t *gR;
  uint64_t *gC;

  __device__ __forceinline__ void emit(int32_t key, uint64_t w) const {
    const uint64_t r = w & kRMask;
    const uint32_t c = (uint32_t)(w >> kCountShift);
    const int64_t b = (int64_t)key - base;
    if (b >= 0 && b < kWin) {
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

template <int KIND, bool YP, int BC, bool PUSH, bool DEP>
__device__ __forceinline__ void process_chunk(const LaunchArgs &a, int isp,
                                              int64_t beg, int64_t end,
                                              const Window &win, Tally &t) {
  const pb_species &s = a.sp[isp];
  const int sid = a.id[isp];
  double *__restrict__ X = s.x;
  double *__restrict__ VX = s.vx;
  double *__restrict__ VY = s.vy;
  double *__restrict__ VZ = s.vz;
  double *__restrict__ YPp = s.yp;
  int32_t *__restrict__ CELL = s.cell;
  const int64_t nc = a.nc;
  const unsigned full = 0xffffffffu;
  constexpr bool kNeedV = (KIND == PB_KIND_KICK || KIND == PB_KIND_BORIS ||
                           KIND == PB_KIND_DRIFT);
  constexpr bool kNeedVyz = (KIND == PB_KIND_BORIS);
  // Charged kinds need the cell for the gather; drift species only for movers.
  constexpr bool kEagerCell = (KIND != PB_KIND_DRIFT) || DEP;

  for (int64_t tb = beg; tb < end; tb += kTile) {
#pragma unroll
    for (int p = 0; p < kPairsPerThread; ++p) {
      const int64_t i = tb + (int64_t)p * (2 * kThreads) + 2 * threadIdx.x;
      const bool v0 = i < end;
      const bool v1 = (i + 1) < end;
      double x0 = 0, x1 = 0, vx0 = 0, vx1 = 0, vy0 = 0, vy1 = 0, vz0 = 0,
             vz1 = 0, y0 = 0, y1 = 0;
      int32_t c0 = -1, c1 = -1;
      if (v1) {
        const double2 xx = __ldcs(reinterpret_cast<const double2 *>(X + i));
        x0 = xx.x;
        x1 = xx.y;
        if (PUSH && kNeedV) {
          const double2 vv = __ldcs(reinterpret_cast<const double2 *>(VX + i));
          vx0 = vv.x;
          vx1 = vv.y;
        }
        if (PUSH && (YP || kNeedVyz)) {
          const double2 vv = __ldcs(reinterpret_cast<const double2 *>(VY + i));
          vy0 = vv.x;
          vy1 = vv.y;
        }
        if (PUSH && kNeedVyz) {
          const double2 vv = __ldcs(reinterpret_cast<const double2 *>(VZ + i));
          vz0 = vv.x;
          vz1 = vv.y;
        }
        if (PUSH && YP) {
          const double2 vv = __ldcs(reinterpret_cast<const double2 *>(YPp + i));
          y0 = vv.x;
          y1 = vv.y;
        }
        if (kEagerCell) {
          const int2 cc = __ldcs(reinterpret_cast<const int2 *>(CELL + i));
          c0 = cc.x;
          c1 = cc.y;
        }
      } else if (v0) {
        x0 = X[i];
        if (PUSH && kNeedV) vx0 = VX[i];
        if (PUSH && (YP || kNeedVyz)) vy0 = VY[i];
        if (PUSH && kNeedVyz) vz0 = VZ[i];
        if (PUSH && YP) y0 = YPp[i];
        if (kEagerCell) c0 = CELL[i];
      }

      bool m0 = false, m1 = false, cfl0 = false, cfl1 = false;
      int8_t w0 = -1, w1 = -1;
      int32_t n0 = c0, n1 = c1;
      if (PUSH) {
        if (v0) {
          kick_drift<KIND>(x0, vx0, vy0, vz0, c0, s, a.e);
          if (YP) y0 = __dadd_rn(y0, __dmul_rn(s.fnstep, vy0));
          if (!kEagerCell && floor(x0) != 0.0) c0 = CELL[i];
          const MoveOut o = transfer<BC>(x0, c0, nc);
          n0 = o.cell;
          m0 = o.moved;
          w0 = o.wall;
          cfl0 = o.cfl;
        }
        if (v1) {
          kick_drift<KIND>(x1, vx1, vy1, vz1, c1, s, a.e);
          if (YP) y1 = __dadd_rn(y1, __dmul_rn(s.fnstep, vy1));
          if (!kEagerCell && floor(x1) != 0.0) c1 = CELL[i + 1];
          const MoveOut o = transfer<BC>(x1, c1, nc);
          n1 = o.cell;
          m1 = o.moved;
          w1 = o.wall;
          cfl1 = o.cfl;
        }
        // Stores.
        if (v1) {
          __stcs(reinterpret_cast<double2 *>(X + i), make_double2(x0, x1));
          if (KIND != PB_KIND_DRIFT)
            __stcs(reinterpret_cast<double2 *>(VX + i), make_double2(vx0, vx1));
          if (KIND == PB_KIND_BORIS) {
            __stcs(reinterpret_cast<double2 *>(VY + i), make_double2(vy0, vy1));
            __stcs(reinterpret_cast<double2 *>(VZ + i), make_double2(vz0, vz1));
          }
          if (YP) __stcs(reinterpret_cast<double2 *>(YPp + i), make_double2(y0, y1));
        } else if (v0) {
          X[i] = x0;
          if (KIND != PB_KIND_DRIFT) VX[i] = vx0;
          if (KIND == PB_KIND_BORIS) {
            VY[i] = vy0;
            VZ[i] = vz0;
          }
          if (YP) YPp[i] = y0;
        }
        if (m0) CELL[i] = n0;
        if (m1) CELL[i + 1] = n1;
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
              base = atomicAdd((unsigned long long *)&a.st->n_holes[sid],
                               (unsigned long long)tot);
            base = __shfl_sync(full, base, 0);
            const unsigned lt = (1u << lane) - 1u;
            if (r0) s.holes[base + __popc(b0 & lt)] = i;
            if (r1) s.holes[base + __popc(b0) + __popc(b1 & lt)] = i + 1;
          }
        }
        if (cfl0 || cfl1) {
          const uint64_t key =
              ((uint64_t)sid << 56) | (uint64_t)(cfl0 ? i : i + 1);
          atomicMin((unsigned long long *)&a.st->cfl_index,
                    (unsigned long long)key);
          atomicCAS(&a.st->code, PB_OK, PB_ERR_CFL);
          if (cfl0) n0 = -1;
          if (cfl1) n1 = -1;
        }
      }
      if (DEP) {
        deposit_pair(v0 ? n0 : -1, x0, v1 ? n1 : -1, x1, win);
      }
    }
  }
}

template <int KIND, bool YP, int BC, bool PUSH>
__device__ __forceinline__ void dispatch_dep(const LaunchArgs &a, int isp,
                                             int64_t beg, int64_t end,
                                             const Window &win, Tally &t,
                                             bool dep) {
  if (dep)
    process_chunk<KIND, YP, BC, PUSH, true>(a, isp, beg, end, win, t);
  else
    process_chunk<KIND, YP, BC, PUSH, false>(a, isp, beg, end, win, t);
}

template <int BC, bool PUSH>
__global__ void __launch_bounds__(kThreads)
    k_push_deposit(const __grid_constant__ LaunchArgs a) {
  __shared__ uint64_t sR[kWin];
  __shared__ uint32_t sC[kWin];
  __shared__ int sTally[3];

  // Which species does this block serve?
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
  if (threadIdx.x < 3) sTally[threadIdx.x] = 0;
  Window win;
  win.sR = sR;
  win.sC = sC;
  win.base = 0;
  win.gR = nullptr;
  win.gC = nullptr;
  if (dep) {
    win.gR = a.bins + (size_t)s.deposit * 2 * (size_t)a.nc;
    win.gC = win.gR + a.nc;
    win.base = (int64_t)s.cell[beg] - kMargin;
  }
  __syncthreads();

  Tally t;
  const bool yp = s.yp != nullptr;
  const int kind = PUSH ? s.kind : PB_KIND_INACTIVE;
  switch (kind) {
    case PB_KIND_KICK:
      if (yp) dispatch_dep<PB_KIND_KICK, true, BC, PUSH>(a, isp, beg, end, win, t, dep);
      else dispatch_dep<PB_KIND_KICK, false, BC, PUSH>(a, isp, beg, end, win, t, dep);
      break;
    case PB_KIND_BORIS:
      if (yp) dispatch_dep<PB_KIND_BORIS, true, BC, PUSH>(a, isp, beg, end, win, t, dep);
      else dispatch_dep<PB_KIND_BORIS, false, BC, PUSH>(a, isp, beg, end, win, t, dep);
      break;
    case PB_KIND_DRIFT:
      if (yp) dispatch_dep<PB_KIND_DRIFT, true, BC, PUSH>(a, isp, beg, end, win, t, dep);
      else dispatch_dep<PB_KIND_DRIFT, false, BC, PUSH>(a, isp, beg, end, win, t, dep);
      break;
    default:  // not pushed: deposit current positions only
      if (dep)
        process_chunk<PB_KIND_INACTIVE, false, BC, false, true>(a, isp, beg, end, win, t);
      break;
  }

  // Block reductions of the tallies and the shared-memory window flush.
  if (PUSH) {
    int mv = t.moved, al = t.absorbed[0], ar = t.absorbed[1];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      mv += __shfl_down_sync(0xffffffffu, mv, d);
      al += __shfl_down_sync(0xffffffffu, al, d);
      ar += __shfl_down_sync(0xffffffffu, ar, d);
    }
    if (lane_id() == 0) {
      if (mv) atomicAdd(&sTally[0], mv);
      if (al) atomicAdd(&sTally[1], al);
      if (ar) atomicAdd(&sTally[2], ar);
    }
  }
  __syncthreads();
  if (PUSH && threadIdx.x == 0) {
    if (sTally[0])
      atomicAdd((unsigned long long *)&a.st->moved[a.id[isp]], (unsigned long long)sTally[0]);
    if (sTally[1])
      atomicAdd((unsigned long long *)&a.st->absorbed[a.id[isp]][0], (unsigned long long)sTally[1]);
    if (sTally[2])
      atomicAdd((unsigned long long *)&a.st->absorbed[a.id[isp]][1], (unsigned long long)sTally[2]);
  }
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
// Host side.
// ---------------------------------------------------------------------------
static int g_blocks_per_sm[2][2] = {{0, 0}, {0, 0}};
static int g_sm_count = 0;

static int launch_cfg(int bc, bool push, int *grid) {
  if (g_sm_count == 0) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    e = cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  }
  int &bps = g_blocks_per_sm[bc][push ? 1 : 0];
  if (bps == 0) {
    const void *fn =
        bc == PB_BC_PERIODIC
            ? (push ? (const void *)k_push_deposit<PB_BC_PERIODIC, true>
                    : (const void *)k_push_deposit<PB_BC_PERIODIC, false>)
            : (push ? (const void *)k_push_deposit<PB_BC_ABSORBING, true>
                    : (const void *)k_push_deposit<PB_BC_ABSORBING, false>);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, kThreads, 0);
    if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (bps < 1) bps = 1;
  }
  *grid = g_sm_count * bps;
  return PB_OK;
}

// Approximate HBM bytes per particle, used only to balance blocks.
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

static int launch(const pb_species *sp, int nsp, const double *e, int64_t nc,
                  int bc, bool push, uint64_t *bins, pb_status *st,
                  cudaStream_t stream) {
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
  a.nsp = 0;
  a.push = push ? 1 : 0;
  a.e = e;
  a.nc = nc;
  a.bins = bins;
  a.st = st;
  double w[PB_MAX_SPECIES];
  double wsum = 0.0;
  // Only species with work take part; map back to their caller index.
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
    if (((uintptr_t)s.x | (uintptr_t)s.vx | (uintptr_t)s.vy | (uintptr_t)s.vz |
         (uintptr_t)s.yp) & 15u || ((uintptr_t)s.cell & 7u)) {
      set_error("species %d: arrays must be 16-byte aligned", k);
      return PB_ERR_INVALID;
    }
    a.id[a.nsp] = k;
    a.sp[a.nsp] = s;
    if (!moves) a.sp[a.nsp].kind = PB_KIND_INACTIVE;
    w[a.nsp] = (double)s.n * bytes_per_particle(a.sp[a.nsp], push);
    wsum += w[a.nsp];
    a.nsp++;
  }
  if (a.nsp == 0) return PB_OK;
  int grid = 0;
  int rc = launch_cfg(bc, push, &grid);
  if (rc) return rc;
  // Blocks per species proportional to bytes, at least one, at most tiles.
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
  const LaunchArgs &b = a;
  if (bc == PB_BC_PERIODIC) {
    if (push) k_push_deposit<PB_BC_PERIODIC, true><<<start, kThreads, 0, stream>>>(b);
    else k_push_deposit<PB_BC_PERIODIC, false><<<start, kThreads, 0, stream>>>(b);
  } else {
    if (push) k_push_deposit<PB_BC_ABSORBING, true><<<start, kThreads, 0, stream>>>(b);
    else k_push_deposit<PB_BC_ABSORBING, false><<<start, kThreads, 0, stream>>>(b);
  }
  PB_CHECK_LAUNCH("k_push_deposit");
  return PB_OK;
}

}  // namespace pb

extern "C" int pb_push_deposit(const pb_species *sp, int nsp,
                               const double *e_nodes, int64_t nc,
                               int particle_bc, uint64_t *bins,
                               pb_status *status, void *stream) {
  return pb::launch(sp, nsp, e_nodes, nc, particle_bc, true, bins, status,
                    (cudaStream_t)stream);
}

extern "C" int pb_deposit_only(const pb_species *sp, int nsp, int64_t nc,
                               uint64_t *bins, pb_status *status,
                               void *stream) {
  if (!bins) {
    pb::set_error("bins pointer is NULL");
    return PB_ERR_INVALID;
  }
  return pb::launch(sp, nsp, nullptr, nc, PB_BC_PERIODIC, false, bins, status,
                    (cudaStream_t)stream);
}
