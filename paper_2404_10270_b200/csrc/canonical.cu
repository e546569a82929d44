// Canonical slot order mode and Monte Carlo collisions.
//
// The production engine (push_deposit.cu) keeps particles in any order and
// deposits with order-independent fixed-point sums.  This file reproduces
// the reference's exact per-cell slot order instead, which is what makes its
// slot-indexed collision streams (pkg/src/picmc/collisions.py:190-219) and
// its sequential per-cell deposit (pkg/src/picmc/backends/_kernels.pyx:14-34)
// bitwise reproducible on the GPU.
//
// Layout: per species a flat SoA in cell-major slot order -- exactly the
// reference CellSortedStore's live slots concatenated over cells
// (pkg/src/picmc/core.py:100-181) -- plus per-cell offs[nc+1] / counts[nc]
// (int64, the reference's own dtype).
//
// One canonical step per species (after the optional collision pass):
//   rank   canonical pre-move position: survivors of cell j in slot order,
//          then the cell's newborns in event order (commit_pending appends,
//          collisions.py:286-289);
//   push   the reference kick/drift + resort_collect transfer (mover.cuh);
//          key = (dest, moved, rank)
//   sort   CUB radix sort of the keys: per destination cell the survivors
//          keep their slot order, then incomers by (src_cell, src_slot) --
//          resort_collect + commit_incomers (pkg/src/picmc/mover.py:167-195);
//   gather every field into the ping-pong buffers, rebuild counts/offs.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "mover.cuh"
#include "rng.cuh"

namespace pb {

static inline size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

static int bits_for(uint64_t v) {  // smallest b with v < 2^b
  int b = 1;
  while (b < 63 && (v >> b) != 0) ++b;
  return b;
}

constexpr uint64_t kDeadKey = ~0ull;

// ---------------------------------------------------------------------------
// Collisions (pkg/src/picmc/collisions.py).  One warp per cell.
// ---------------------------------------------------------------------------
constexpr double kGuard = 0.1;  // collisions.py:44
constexpr int kMaxGuardLevels = 30;

struct CollideArgs {
  pb_species e, nt, ion;
  const int64_t *e_offs, *e_counts, *n_offs;
  int64_t *n_counts;
  int64_t *nb_per_cell;
  int32_t *nb_k;
  int64_t nb_cap;
  int64_t nc;
  pb_collide_params p;
  unsigned long long *ctr;
};

// _probabilities (collisions.py:188-192): p = -expm1(-(n*R)*dt).
__device__ __forceinline__ double coll_prob(double nden, double rate, double dt) {
  return -expm1(__dmul_rn(-__dmul_rn(nden, rate), dt));
}

// _unit_vector (collisions.py:97-108): rejection on the unit disc, sqrt only.
__device__ __forceinline__ void unit_vector(uint64_t key, double &ux, double &uy, double &uz) {
  uint64_t t = 0;
  double u, v, s;
  while (true) {
    u = __dsub_rn(__dmul_rn(2.0, uniform(key, 2 * t)), 1.0);
    v = __dsub_rn(__dmul_rn(2.0, uniform(key, 2 * t + 1)), 1.0);
    s = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
    if (s < 1.0) break;
    ++t;
  }
  const double f = __dmul_rn(2.0, __dsqrt_rn(__dsub_rn(1.0, s)));
  ux = __dmul_rn(u, f);
  uy = __dmul_rn(v, f);
  uz = __dsub_rn(1.0, __dmul_rn(2.0, s));
}

__device__ __forceinline__ double speed_of(double vx, double vy, double vz) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy)), __dmul_rn(vz, vz)));
}

__global__ void __launch_bounds__(256) k_collide(const __grid_constant__ CollideArgs a) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const pb_collide_params &P = a.p;
  unsigned long long n_el = 0, n_ex = 0, n_io = 0, n_sup = 0, n_ovf = 0;
  for (int64_t j = w0; j < a.nc; j += nw) {
    const int64_t ne = a.e_counts[j];
    int64_t nn = a.n_counts[j];
    int64_t kev = 0;  // newborn pairs of this cell, in event order
    if (ne > 0) {
      const uint64_t ckey = derive(P.step_key, (uint64_t)(j + P.global_offset));
      const int64_t eb = a.e_offs[j], nb = a.n_offs[j];
      // collide_block (collisions.py:222-283): single pass below the guard,
      // else 2^m substeps with thresholds refrozen from live counts.
      double nd = __dmul_rn((double)nn, P.w_over_dx);
      double pe = coll_prob(nd, P.rate_elastic, P.dt);
      double px = coll_prob(nd, P.rate_excitation, P.dt);
      double pi = coll_prob(nd, P.rate_ionization, P.dt);
      int64_t nsub = 1;
      double dts = P.dt;
      if (!(__dadd_rn(__dadd_rn(pe, px), pi) < kGuard)) {
        int m = 0;
        while (true) {
          ++m;
          dts = __ddiv_rn(P.dt, (double)(1ull << m));
          const double q = __dadd_rn(__dadd_rn(coll_prob(nd, P.rate_elastic, dts),
                                               coll_prob(nd, P.rate_excitation, dts)),
                                     coll_prob(nd, P.rate_ionization, dts));
          if (q < kGuard || m >= kMaxGuardLevels) break;
        }
        if (m >= kMaxGuardLevels) ++n_ovf;
        nsub = (int64_t)1 << m;
      }
      for (int64_t s = 0; s < nsub; ++s) {
        if (nsub > 1) {
          nd = __dmul_rn((double)nn, P.w_over_dx);
          pe = coll_prob(nd, P.rate_elastic, dts);
          px = coll_prob(nd, P.rate_excitation, dts);
          pi = coll_prob(nd, P.rate_ionization, dts);
        }
        // _select_and_apply (collisions.py:195-219)
        const uint64_t sub = derive(ckey, (uint64_t)s);
        const uint64_t sel = derive(sub, 0), evb = derive(sub, 1);
        const double t1 = pe, t2 = __dadd_rn(pe, px), t3 = __dadd_rn(t2, pi);
        for (int64_t c0 = 0; c0 < ne; c0 += 32) {
          const int64_t slot = c0 + lane;
          int kind = 0;
          if (slot < ne) {
            const double u = uniform(sel, (uint64_t)slot);
            if (u < t3) kind = u < t1 ? 1 : (u < t2 ? 2 : 3);
          }
          const int64_t i = eb + slot;
          if (kind == 1 || kind == 2) {  // _apply_event elastic / excitation (:126-152)
            const uint64_t ev = derive(evb, (uint64_t)slot);
            const double speed = speed_of(a.e.vx[i], a.e.vy[i], a.e.vz[i]);
            double ns = speed;
            if (kind == 2) {
              const double vsi = __dmul_rn(speed, P.dx_over_dt);
              double ke = __dmul_rn(__dmul_rn(__dmul_rn(0.5, P.mass_e), vsi), vsi);
              const double d = __dsub_rn(ke, P.threshold_j);
              ke = (0.0 > d) ? 0.0 : d;  // Python max(d, 0.0)
              ns = __ddiv_rn(__dsqrt_rn(__ddiv_rn(__dmul_rn(2.0, ke), P.mass_e)), P.dx_over_dt);
            }
            double ux, uy, uz;
            unit_vector(derive(ev, 1), ux, uy, uz);
            a.e.vx[i] = __dmul_rn(ns, ux);
            a.e.vy[i] = __dmul_rn(ns, uy);
            a.e.vz[i] = __dmul_rn(ns, uz);
            if (kind == 1) ++n_el; else ++n_ex;
          }
          // Ionizations in slot order: each consumes a live neutral of the
          // cell (swap_remove, core.py:205-218), so they are serialised.
          unsigned im = __ballot_sync(full, kind == 3);
          while (im) {
            const int src = __ffs(im) - 1;
            im &= im - 1;
            if (lane == src) {
              if (nn == 0) {
                ++n_sup;
              } else {
                const uint64_t ev = derive(evb, (uint64_t)slot);
                int64_t pick = (int64_t)__dmul_rn(uniform(derive(ev, 0), 0), (double)nn);
                if (pick >= nn) pick = nn - 1;
                const int64_t ip = nb + pick, il = nb + nn - 1;
                const double qx = a.nt.x[ip], qvx = a.nt.vx[ip], qvy = a.nt.vy[ip], qvz = a.nt.vz[ip];
                const double qyp = a.nt.yp ? a.nt.yp[ip] : 0.0;
                a.nt.x[ip] = a.nt.x[il];
                a.nt.vx[ip] = a.nt.vx[il];
                a.nt.vy[ip] = a.nt.vy[il];
                a.nt.vz[ip] = a.nt.vz[il];
                if (a.nt.yp) a.nt.yp[ip] = a.nt.yp[il];
                a.nt.cell[il] = -1;  // vacated tail slot: dropped by the resort
                nn -= 1;
                const double speed = speed_of(a.e.vx[i], a.e.vy[i], a.e.vz[i]);
                const double vsi = __dmul_rn(speed, P.dx_over_dt);
                const double keh = __dmul_rn(__dmul_rn(__dmul_rn(0.25, P.mass_e), vsi), vsi);
                const double sh = __ddiv_rn(__dsqrt_rn(__ddiv_rn(__dmul_rn(2.0, keh), P.mass_e)), P.dx_over_dt);
                double ux, uy, uz, ex, ey, ez;
                unit_vector(derive(ev, 1), ux, uy, uz);
                unit_vector(derive(ev, 2), ex, ey, ez);
                a.e.vx[i] = __dmul_rn(sh, ux);
                a.e.vy[i] = __dmul_rn(sh, uy);
                a.e.vz[i] = __dmul_rn(sh, uz);
                const unsigned long long t = atomicAdd(&a.ctr[4], 1ull);
                if ((int64_t)t < a.nb_cap) {
                  const int64_t ki = a.ion.n + (int64_t)t, ke = a.e.n + (int64_t)t;
                  a.ion.x[ki] = qx;
                  a.ion.vx[ki] = qvx;
                  a.ion.vy[ki] = qvy;
                  a.ion.vz[ki] = qvz;
                  if (a.ion.yp) a.ion.yp[ki] = qyp;
                  a.ion.cell[ki] = (int32_t)j;
                  a.e.x[ke] = a.e.x[i];
                  a.e.vx[ke] = __dmul_rn(sh, ex);
                  a.e.vy[ke] = __dmul_rn(sh, ey);
                  a.e.vz[ke] = __dmul_rn(sh, ez);
                  if (a.e.yp) a.e.yp[ke] = a.e.yp[i];
                  a.e.cell[ke] = (int32_t)j;
                  a.nb_k[t] = (int32_t)kev;
                } else {
                  ++n_ovf;
                }
                ++kev;
                ++n_io;
              }
            }
            __syncwarp();  // the next event may read slots this one rewrote
            nn = __shfl_sync(full, nn, src);
            kev = __shfl_sync(full, kev, src);
          }
        }
      }
    }
    if (lane == 0) {
      a.n_counts[j] = nn;
      a.nb_per_cell[j] = kev;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    n_el += __shfl_down_sync(full, n_el, d);
    n_ex += __shfl_down_sync(full, n_ex, d);
    n_io += __shfl_down_sync(full, n_io, d);
    n_sup += __shfl_down_sync(full, n_sup, d);
    n_ovf += __shfl_down_sync(full, n_ovf, d);
  }
  if (lane == 0) {
    if (n_el) atomicAdd(&a.ctr[0], n_el);
    if (n_ex) atomicAdd(&a.ctr[1], n_ex);
    if (n_io) atomicAdd(&a.ctr[2], n_io);
    if (n_sup) atomicAdd(&a.ctr[3], n_sup);
    if (n_ovf) atomicAdd(&a.ctr[5], n_ovf);
  }
}

// ---------------------------------------------------------------------------
// Canonical resort.
// ---------------------------------------------------------------------------
__global__ void k_sum_counts(const int64_t *__restrict__ a, const int64_t *__restrict__ b,
                             int64_t *__restrict__ out, int64_t nc) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nc;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = a[j] + (b ? b[j] : 0);
}

struct CanonPushArgs {
  pb_species s;
  int64_t n_old, n_tot;
  int64_t rank_offset;  // global canonical position of this rank's first particle
  const int64_t *offs, *cnt_after, *offp;
  const int32_t *nb_k;
  const double *e;
  int64_t nc;
  int sid, rank_bits;
  pb_status *st;
  uint64_t *keys;
  uint32_t *vals;
  // scatter resort: classify the keys in the same pass (scat_classify_warp), or null
  uint32_t *stay_by_rank;
  int64_t *cnt_stay, *cnt_in;
  uint64_t *mkeys;
  uint32_t *midx;
  unsigned long long *mcount;
};

// the scatter resort's classification of one warp's keys: stayers flagged by rank and
// counted per cell, movers appended (see k_scat_stay)
__device__ __forceinline__ void scat_classify_warp(uint64_t key, int64_t i, int rank_bits,
                                                   uint32_t *stay_by_rank, int64_t *cnt_stay,
                                                   int64_t *cnt_in, uint64_t *mkeys, uint32_t *midx,
                                                   unsigned long long *mcount) {
  const unsigned lane = threadIdx.x & 31;
  const bool live = key != kDeadKey;
  const int64_t dest = live ? (int64_t)((key >> rank_bits) >> 1) : -1;
  const bool mv = live && ((key >> rank_bits) & 1ull);
  const bool stay = live && !mv;
  if (stay) stay_by_rank[key & ((1ull << rank_bits) - 1)] = 1u;
  const unsigned grp = __match_any_sync(0xffffffffu, stay ? dest : -1);
  if (stay && lane == (unsigned)(__ffs(grp) - 1))
    atomicAdd((unsigned long long *)&cnt_stay[dest], (unsigned long long)__popc(grp));
  const unsigned mb = __ballot_sync(0xffffffffu, mv);
  if (mb) {
    const unsigned leader = (unsigned)(__ffs(mb) - 1);
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(mcount, (unsigned long long)__popc(mb));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (mv) {
      unsigned lt;
      asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
      const unsigned long long t = base + __popc(mb & lt);
      mkeys[t] = key;
      midx[t] = (uint32_t)i;
      atomicAdd((unsigned long long *)&cnt_in[dest], 1ull);
    }
  }
}

template <int KIND, int BC>
__device__ __forceinline__ uint64_t canon_push_one(const CanonPushArgs &a, int64_t i, int &moved,
                                                   int &abs_l, int &abs_r) {
  const pb_species &s = a.s;
  a.vals[i] = (uint32_t)i;
  const int32_t c = s.cell[i];
  if (c < 0) return kDeadKey;
  {
    const int64_t rank = a.rank_offset + (i < a.n_old ? a.offp[c] + (i - a.offs[c])
                                                      : a.offp[c] + a.cnt_after[c] + a.nb_k[i - a.n_old]);
    int32_t dest = c;
    bool mv = false;
    if (KIND != PB_KIND_INACTIVE) {
      double x = s.x[i], vx = s.vx[i], vy = s.vy[i], vz = s.vz[i];
      kick_drift<KIND>(x, vx, vy, vz, c, s, a.e);
      if (s.yp) s.yp[i] = __dadd_rn(s.yp[i], __dmul_rn(s.fnstep, vy));
      const MoveOut o = transfer<BC>(x, c, a.nc);
      s.x[i] = x;
      if (KIND != PB_KIND_DRIFT) s.vx[i] = vx;
      if (is_boris(KIND)) {
        s.vy[i] = vy;
        s.vz[i] = vz;
      }
      if (o.cfl) {
        const uint64_t key = ((uint64_t)a.sid << 56) | (uint64_t)i;
        atomicMin((unsigned long long *)&a.st->cfl_index, (unsigned long long)key);
        atomicCAS(&a.st->code, PB_OK, PB_ERR_CFL);
      } else if (o.moved) {
        ++moved;
        mv = true;
        dest = o.cell;
        if (BC == PB_BC_ABSORBING && o.wall >= 0) {
          if (o.wall == 0) ++abs_l; else ++abs_r;
          return kDeadKey;
        }
      }
    }
    return ((((uint64_t)dest << 1) | (mv ? 1u : 0u)) << a.rank_bits) | (uint64_t)rank;
  }
}

template <int KIND, int BC>
__global__ void __launch_bounds__(256) k_canon_push(const __grid_constant__ CanonPushArgs a) {
  int moved = 0, abs_l = 0, abs_r = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-aligned grid stride: every lane reaches the classification collectives
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < a.n_tot; b += stride) {
    const int64_t i = b + threadIdx.x;
    uint64_t key = kDeadKey;
    if (i < a.n_tot) {
      key = canon_push_one<KIND, BC>(a, i, moved, abs_l, abs_r);
      a.keys[i] = key;
    }
    if (a.stay_by_rank)
      scat_classify_warp(key, i, a.rank_bits, a.stay_by_rank, a.cnt_stay, a.cnt_in, a.mkeys, a.midx,
                         a.mcount);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    moved += __shfl_down_sync(0xffffffffu, moved, d);
    abs_l += __shfl_down_sync(0xffffffffu, abs_l, d);
    abs_r += __shfl_down_sync(0xffffffffu, abs_r, d);
  }
  if ((threadIdx.x & 31) == 0) {
    if (moved) atomicAdd((unsigned long long *)&a.st->moved[a.sid], (unsigned long long)moved);
    if (abs_l) atomicAdd((unsigned long long *)&a.st->absorbed[a.sid][0], (unsigned long long)abs_l);
    if (abs_r) atomicAdd((unsigned long long *)&a.st->absorbed[a.sid][1], (unsigned long long)abs_r);
  }
}

struct GatherArgs {
  const double *src[5];
  double *dst[5];
  int nf;
};

// Gather every field in sorted order; cell from the key; count live
// particles per destination cell.
__global__ void k_canon_gather(GatherArgs g, const uint32_t *__restrict__ perm,
                               const uint64_t *__restrict__ keys, int64_t n, int rank_bits,
                               int32_t *__restrict__ cell_out, int64_t *__restrict__ counts) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[k];
    if (key == kDeadKey) continue;  // dead keys sort last
    const uint32_t p = perm[k];
#pragma unroll
    for (int f = 0; f < 5; ++f)
      if (f < g.nf) g.dst[f][k] = __ldg(g.src[f] + p);
    const int32_t c = (int32_t)((key >> rank_bits) >> 1);
    cell_out[k] = c;
    atomicAdd((unsigned long long *)&counts[c], 1ull);
  }
}

// counts of a cell-sorted cell array (layout build at load time); flags
// unsorted input.
__global__ void k_cell_hist(const int32_t *__restrict__ cell, int64_t n, int64_t nc,
                            int64_t *__restrict__ counts, int *__restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = cell[i];
    if (c < 0 || c >= nc || (i > 0 && cell[i - 1] > c)) {
      atomicExch(bad, 1);
      continue;
    }
    atomicAdd((unsigned long long *)&counts[c], 1ull);
  }
}

static size_t scan_temp_bytes(int64_t nc) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int64_t *)nullptr, (int64_t *)nullptr,
                                (int)(nc + 1));
  return t;
}

static size_t sort_temp_bytes(int64_t n) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (int)(n > 0 ? n : 1), 0, 64);
  return t;
}

// offs[0..nc] = exclusive scan of counts[0..nc-1] (offs[nc] = total).
// `tmp` holds nc+1 int64 followed by the CUB temp storage.
static int offsets_from_counts(const int64_t *counts, int64_t *offs, int64_t nc, char *tmp,
                               cudaStream_t st) {
  int64_t *ext = (int64_t *)tmp;
  char *cub_tmp = tmp + a256((size_t)(nc + 1) * 8);
  cudaError_t e = cudaMemcpyAsync(ext, counts, (size_t)nc * 8, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync");
  e = cudaMemsetAsync(ext + nc, 0, 8, st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMemsetAsync");
  size_t tb = scan_temp_bytes(nc);
  e = cub::DeviceScan::ExclusiveSum(cub_tmp, tb, ext, offs, (int)(nc + 1), st);
  if (e != cudaSuccess) return cuda_status(e, "DeviceScan::ExclusiveSum");
  return PB_OK;
}

static int launch_canon_push(const pb_species *src, const pb_canon *cv, const double *e_nodes,
                             int64_t nc, int particle_bc, int species_id, pb_status *status,
                             int64_t rank_offset, int rank_bits, const int64_t *offp,
                             uint64_t *keys, uint32_t *vals, cudaStream_t st,
                             const CanonPushArgs *cls = nullptr) {
  CanonPushArgs a;
  memset(&a, 0, sizeof(a));
  if (cls) {  // the scatter resort's classification outputs
    a.stay_by_rank = cls->stay_by_rank;
    a.cnt_stay = cls->cnt_stay;
    a.cnt_in = cls->cnt_in;
    a.mkeys = cls->mkeys;
    a.midx = cls->midx;
    a.mcount = cls->mcount;
  }
  a.s = *src;
  a.n_old = cv->n_old;
  a.n_tot = cv->n_old + cv->n_tail;
  a.rank_offset = rank_offset;
  a.offs = cv->offs;
  a.cnt_after = cv->counts;
  a.offp = offp;
  a.nb_k = cv->newborn_k;
  a.e = e_nodes;
  a.nc = nc;
  a.sid = species_id;
  a.rank_bits = rank_bits;
  a.st = status;
  a.keys = keys;
  a.vals = vals;
  int64_t blocks = (a.n_tot + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  const bool abs = particle_bc == PB_BC_ABSORBING;
#define PB_CANON(KIND)                                                              \
  (abs ? k_canon_push<KIND, PB_BC_ABSORBING><<<(unsigned)blocks, 256, 0, st>>>(a) \
       : k_canon_push<KIND, PB_BC_PERIODIC><<<(unsigned)blocks, 256, 0, st>>>(a))
  switch (src->kind) {
    case PB_KIND_INACTIVE: PB_CANON(PB_KIND_INACTIVE); break;
    case PB_KIND_DRIFT: PB_CANON(PB_KIND_DRIFT); break;
    case PB_KIND_KICK: PB_CANON(PB_KIND_KICK); break;
    case PB_KIND_BORIS:
      if (src->b_nodes) PB_CANON(kKindBorisB);
      else PB_CANON(PB_KIND_BORIS);
      break;
    default:
      set_error("canonical push: unknown kind %d", src->kind);
      return PB_ERR_INVALID;
  }
#undef PB_CANON
  PB_CHECK_LAUNCH("k_canon_push");
  return PB_OK;
}

static size_t offsets_tmp_bytes(int64_t nc) {
  return a256((size_t)(nc + 1) * 8) + a256(scan_temp_bytes(nc));
}

// ---- canonical resort as a scatter (no full key sort) ----------------------
// The canonical order is (dest cell, moved, rank): within every cell first
// the particles that stayed, in their pre-move rank order, then the
// incomers in rank order.  The stayers' relative order is unchanged, so
// their new slot is new_off[cell] + (stayers with a smaller rank in the cell)
// = new_off[c] + G[rank] - G[offp[c]] with G the exclusive prefix count of
// stayers over the pre-move ranks; only the movers (~0.6% of electrons per
// step) are sorted by key (the push classifies its keys as it writes them:
// scat_classify_warp).  Same final order as sorting every key.
struct ScatArgs {
  const double *src[5];
  double *dst[5];
  int nf;
  int rank_bits;
  const uint64_t *keys;
  const uint32_t *G;
  const int64_t *offp, *new_off, *cnt_stay, *in_off;
  const uint64_t *mkeys_s;
  const uint32_t *midx_s;
  int32_t *cell_out;
};

__global__ void k_scat_stay(const __grid_constant__ ScatArgs a, int64_t n) {
  const uint64_t rmask = (1ull << a.rank_bits) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = a.keys[i];
    if (key == kDeadKey || ((key >> a.rank_bits) & 1ull)) continue;
    const int64_t c = (int64_t)((key >> a.rank_bits) >> 1);
    const uint64_t rank = key & rmask;
    const int64_t pos = a.new_off[c] + (int64_t)a.G[rank] - (int64_t)a.G[a.offp[c]];
#pragma unroll
    for (int f = 0; f < 5; ++f)
      if (f < a.nf) a.dst[f][pos] = __ldg(a.src[f] + i);
    a.cell_out[pos] = (int32_t)c;
  }
}

__global__ void k_scat_movers(const __grid_constant__ ScatArgs a, int64_t m) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = a.mkeys_s[t];
    const int64_t d = (int64_t)((key >> a.rank_bits) >> 1);
    const int64_t pos = a.new_off[d] + a.cnt_stay[d] + (t - a.in_off[d]);
    const uint32_t i = a.midx_s[t];
#pragma unroll
    for (int f = 0; f < 5; ++f)
      if (f < a.nf) a.dst[f][pos] = __ldg(a.src[f] + i);
    a.cell_out[pos] = (int32_t)d;
  }
}

__global__ void k_add_counts(const int64_t *__restrict__ a, const int64_t *__restrict__ b,
                             int64_t *__restrict__ out, int64_t nc) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nc;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = a[j] + b[j];
}

// Stores with at least this many particles take the scatter resort; smaller
// ones keep the full key sort (the scatter path's host read of the mover
// count costs more than sorting ~1M keys).  pb_set_canonical_scatter_min
// moves it (tests exercise both paths; INT64_MAX = key sort only).
static int64_t g_scatter_min = (int64_t)1 << 20;

static size_t scan_u32_bytes(int64_t n) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                (int)(n + 1));
  return t;
}

static size_t scatter_extra_bytes(int64_t n, int64_t nc) {
  return 2 * a256((size_t)(n + 1) * 4) + a256((size_t)n * 8) + 3 * a256((size_t)(nc + 1) * 8) +
         a256(8) + a256(scan_u32_bytes(n));
}

}  // namespace pb

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" size_t pb_layout_scratch_bytes(int64_t nc) {
  return pb::offsets_tmp_bytes(nc) + 256;
}

extern "C" int pb_cell_layout(const int32_t *cell, int64_t n, int64_t nc, int64_t *offs,
                              int64_t *counts, void *scratch, size_t scratch_bytes,
                              void *stream) {
  if (nc < 1 || n < 0 || !offs || !counts || (n > 0 && !cell) ||
      scratch_bytes < pb_layout_scratch_bytes(nc) || !scratch) {
    pb::set_error("pb_cell_layout: bad arguments");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int *bad = (int *)scratch;
  char *tmp = (char *)scratch + 256;
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)nc * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0, sizeof(int), st);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaMemsetAsync");
  if (n > 0) {
    pb::k_cell_hist<<<148 * 4, 256, 0, st>>>(cell, n, nc, counts, bad);
    PB_CHECK_LAUNCH("k_cell_hist");
  }
  int rc = pb::offsets_from_counts(counts, offs, nc, tmp, st);
  if (rc) return rc;
  int h_bad = 0;
  e = cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return pb::cuda_status(e, "pb_cell_layout sync");
  if (h_bad) {
    pb::set_error("pb_cell_layout: particles are not in cell-major order");
    return PB_ERR_CONTRACT;
  }
  return PB_OK;
}

extern "C" int pb_collide(const pb_species *e, const pb_species *neutral, const pb_species *ion,
                          const int64_t *e_offs, const int64_t *e_counts, const int64_t *n_offs,
                          int64_t *n_counts, int64_t nc, const pb_collide_params *params,
                          int64_t *newborn_per_cell, int32_t *newborn_k, int64_t newborn_cap,
                          uint64_t *counters, void *stream) {
  if (!e || !neutral || !ion || !e_offs || !e_counts || !n_offs || !n_counts || !params ||
      !newborn_per_cell || !counters || nc < 1 || newborn_cap < 0 ||
      (newborn_cap > 0 && !newborn_k)) {
    pb::set_error("pb_collide: bad arguments");
    return PB_ERR_INVALID;
  }
  if (!neutral->cell || !e->cell || !ion->cell) {
    pb::set_error("pb_collide: species without cell arrays");
    return PB_ERR_INVALID;
  }
  pb::CollideArgs a;
  a.e = *e;
  a.nt = *neutral;
  a.ion = *ion;
  a.e_offs = e_offs;
  a.e_counts = e_counts;
  a.n_offs = n_offs;
  a.n_counts = n_counts;
  a.nb_per_cell = newborn_per_cell;
  a.nb_k = newborn_k;
  a.nb_cap = newborn_cap;
  a.nc = nc;
  a.p = *params;
  a.ctr = (unsigned long long *)counters;
  cudaError_t ze = cudaMemsetAsync(counters, 0, 6 * sizeof(uint64_t), (cudaStream_t)stream);
  if (ze != cudaSuccess) return pb::cuda_status(ze, "cudaMemsetAsync");
  const int threads = 256;
  int64_t blocks = (nc + 7) / 8;
  if (blocks > 148 * 64) blocks = 148 * 64;
  pb::k_collide<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(a);
  PB_CHECK_LAUNCH("k_collide");
  return PB_OK;
}

extern "C" size_t pb_canonical_scratch_bytes(int64_t n_cap, int64_t nc) {
  if (n_cap < 1) n_cap = 1;
  return 2 * pb::a256((size_t)n_cap * 8) + 2 * pb::a256((size_t)n_cap * 4) +
         pb::a256((size_t)(nc + 1) * 8) + pb::a256((size_t)nc * 8) +
         pb::a256(pb::sort_temp_bytes(n_cap)) + pb::offsets_tmp_bytes(nc) +
         pb::scatter_extra_bytes(n_cap, nc);
}

extern "C" int pb_canonical_resort(const pb_species *src, const pb_species *dst,
                                   const pb_canon *cv, const double *e_nodes, int64_t nc,
                                   int particle_bc, int species_id, pb_status *status,
                                   void *scratch, size_t scratch_bytes, void *stream) {
  if (!src || !dst || !cv || !status || nc < 1 || nc > 0x3fffffffLL ||
      species_id < 0 || species_id >= PB_MAX_SPECIES) {
    pb::set_error("pb_canonical_resort: bad arguments");
    return PB_ERR_INVALID;
  }
  const int64_t n_tot = cv->n_old + cv->n_tail;
  if (cv->n_old < 0 || cv->n_tail < 0 || n_tot > 0x7fffffffLL || !cv->offs || !cv->counts ||
      (cv->n_tail > 0 && (!cv->newborn_per_cell || !cv->newborn_k))) {
    pb::set_error("pb_canonical_resort: bad layout (n_old=%lld n_tail=%lld)",
                  (long long)cv->n_old, (long long)cv->n_tail);
    return PB_ERR_INVALID;
  }
  if ((src->kind == PB_KIND_KICK || src->kind == PB_KIND_BORIS) && !e_nodes) {
    pb::set_error("pb_canonical_resort: charged species needs e_nodes");
    return PB_ERR_INVALID;
  }
  if (!scratch || scratch_bytes < pb_canonical_scratch_bytes(n_tot, nc)) {
    pb::set_error("pb_canonical_resort: scratch too small");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t err;
  if (n_tot == 0) {
    err = cudaMemsetAsync(cv->counts, 0, (size_t)nc * 8, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(cv->offs, 0, (size_t)(nc + 1) * 8, st);
    return err == cudaSuccess ? PB_OK : pb::cuda_status(err, "cudaMemsetAsync");
  }
  char *p = (char *)scratch;
  uint64_t *keys = (uint64_t *)p;
  p += pb::a256((size_t)n_tot * 8);
  uint64_t *keys_s = (uint64_t *)p;
  p += pb::a256((size_t)n_tot * 8);
  uint32_t *vals = (uint32_t *)p;
  p += pb::a256((size_t)n_tot * 4);
  uint32_t *perm = (uint32_t *)p;
  p += pb::a256((size_t)n_tot * 4);
  int64_t *offp = (int64_t *)p;
  p += pb::a256((size_t)(nc + 1) * 8);
  int64_t *pre = (int64_t *)p;
  p += pb::a256((size_t)nc * 8);
  char *sort_tmp = p;
  p += pb::a256(pb::sort_temp_bytes(n_tot));
  char *scan_tmp = p;

  // Canonical pre-move offsets: survivors + newborns per cell.
  pb::k_sum_counts<<<148, 256, 0, st>>>(cv->counts, cv->n_tail ? cv->newborn_per_cell : nullptr,
                                        pre, nc);
  PB_CHECK_LAUNCH("k_sum_counts");
  int rc = pb::offsets_from_counts(pre, offp, nc, scan_tmp, st);
  if (rc) return rc;

  const int rank_bits = pb::bits_for((uint64_t)n_tot);
  const int key_bits = rank_bits + pb::bits_for((uint64_t)(2 * nc));
  if (key_bits > 63) {
    pb::set_error("pb_canonical_resort: key needs %d bits", key_bits);
    return PB_ERR_INVALID;
  }
  pb::GatherArgs g;
  int nf = 0;
  g.src[nf] = src->x; g.dst[nf++] = dst->x;
  g.src[nf] = src->vx; g.dst[nf++] = dst->vx;
  g.src[nf] = src->vy; g.dst[nf++] = dst->vy;
  g.src[nf] = src->vz; g.dst[nf++] = dst->vz;
  if (src->yp && dst->yp) {
    g.src[nf] = src->yp;
    g.dst[nf++] = dst->yp;
  }
  g.nf = nf;
  if (n_tot < pb::g_scatter_min) {
    rc = pb::launch_canon_push(src, cv, e_nodes, nc, particle_bc, species_id, status, 0, rank_bits,
                               offp, keys, vals, st);
    if (rc) return rc;
  } else {
    // scatter path (see k_scat_stay): extra scratch after the sort path's
    char *q = scan_tmp + pb::offsets_tmp_bytes(nc);
    uint32_t *stay = (uint32_t *)q;
    q += pb::a256((size_t)(n_tot + 1) * 4);
    uint32_t *G = (uint32_t *)q;
    q += pb::a256((size_t)(n_tot + 1) * 4);
    uint64_t *mkeys_s = (uint64_t *)q;
    q += pb::a256((size_t)n_tot * 8);
    int64_t *cnt_stay = (int64_t *)q;
    q += pb::a256((size_t)(nc + 1) * 8);
    int64_t *cnt_in = (int64_t *)q;
    q += pb::a256((size_t)(nc + 1) * 8);
    int64_t *in_off = (int64_t *)q;
    q += pb::a256((size_t)(nc + 1) * 8);
    unsigned long long *mcount = (unsigned long long *)q;
    q += pb::a256(8);
    char *u32_tmp = q;
    const int64_t R = n_tot;  // pre-move ranks lie in [0, offp[nc]) <= n_tot
    err = cudaMemsetAsync(stay, 0, (size_t)(R + 1) * 4, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(cnt_stay, 0, (size_t)(nc + 1) * 8, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(cnt_in, 0, (size_t)(nc + 1) * 8, st);
    if (err == cudaSuccess) err = cudaMemsetAsync(mcount, 0, 8, st);
    if (err != cudaSuccess) return pb::cuda_status(err, "cudaMemsetAsync");
    // the push classifies its keys as it writes them
    pb::CanonPushArgs cls;
    memset(&cls, 0, sizeof(cls));
    cls.stay_by_rank = stay;
    cls.cnt_stay = cnt_stay;
    cls.cnt_in = cnt_in;
    cls.mkeys = keys_s;
    cls.midx = perm;
    cls.mcount = mcount;
    rc = pb::launch_canon_push(src, cv, e_nodes, nc, particle_bc, species_id, status, 0, rank_bits,
                               offp, keys, vals, st, &cls);
    if (rc) return rc;
    int64_t blocks = (n_tot + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    size_t tb = pb::scan_u32_bytes(R);
    err = cub::DeviceScan::ExclusiveSum(u32_tmp, tb, stay, G, (int)(R + 1), st);
    if (err != cudaSuccess) return pb::cuda_status(err, "DeviceScan (stayers)");
    pb::k_add_counts<<<148, 256, 0, st>>>(cnt_stay, cnt_in, cv->counts, nc);
    PB_CHECK_LAUNCH("k_add_counts");
    rc = pb::offsets_from_counts(cv->counts, cv->offs, nc, scan_tmp, st);
    if (rc) return rc;
    rc = pb::offsets_from_counts(cnt_in, in_off, nc, scan_tmp, st);
    if (rc) return rc;
    unsigned long long m = 0;
    err = cudaMemcpyAsync(&m, mcount, 8, cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return pb::cuda_status(err, "mover count");
    if (m > 0) {
      size_t sb = pb::sort_temp_bytes((int64_t)m);
      err = cub::DeviceRadixSort::SortPairs(sort_tmp, sb, keys_s, mkeys_s, perm, vals, (int)m, 0,
                                            key_bits, st);
      if (err != cudaSuccess) return pb::cuda_status(err, "DeviceRadixSort::SortPairs (movers)");
    }
    pb::ScatArgs sa;
    for (int f = 0; f < 5; ++f) {
      sa.src[f] = f < nf ? g.src[f] : nullptr;
      sa.dst[f] = f < nf ? g.dst[f] : nullptr;
    }
    sa.nf = nf;
    sa.rank_bits = rank_bits;
    sa.keys = keys;
    sa.G = G;
    sa.offp = offp;
    sa.new_off = cv->offs;
    sa.cnt_stay = cnt_stay;
    sa.in_off = in_off;
    sa.mkeys_s = mkeys_s;
    sa.midx_s = vals;
    sa.cell_out = dst->cell;
    pb::k_scat_stay<<<(unsigned)blocks, 256, 0, st>>>(sa, n_tot);
    PB_CHECK_LAUNCH("k_scat_stay");
    if (m > 0) {
      int64_t mb = ((int64_t)m + 255) / 256;
      if (mb > 148 * 16) mb = 148 * 16;
      pb::k_scat_movers<<<(unsigned)mb, 256, 0, st>>>(sa, (int64_t)m);
      PB_CHECK_LAUNCH("k_scat_movers");
    }
    return PB_OK;
  }
  size_t tb = pb::sort_temp_bytes(n_tot);
  err = cub::DeviceRadixSort::SortPairs(sort_tmp, tb, keys, keys_s, vals, perm, (int)n_tot, 0,
                                        key_bits, st);
  if (err != cudaSuccess) return pb::cuda_status(err, "DeviceRadixSort::SortPairs");
  // Dead keys have every bit set, so they also sort last inside key_bits.
  err = cudaMemsetAsync(cv->counts, 0, (size_t)nc * 8, st);
  if (err != cudaSuccess) return pb::cuda_status(err, "cudaMemsetAsync");
  int64_t blocks = (n_tot + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  pb::k_canon_gather<<<(unsigned)blocks, 256, 0, st>>>(g, perm, keys_s, n_tot, rank_bits,
                                                       dst->cell, cv->counts);
  PB_CHECK_LAUNCH("k_canon_gather");
  return pb::offsets_from_counts(cv->counts, cv->offs, nc, scan_tmp, st);
}

// All species of a step in one call (one host round trip instead of one per
// species): pb_canonical_resort for each, then the new live counts
// (offs[nc] of every species) copied to the host array n_new; synchronises
// the stream.
extern "C" int pb_canonical_step(const pb_species *src, const pb_species *dst, const pb_canon *cv,
                                 int nsp, const double *e_nodes, int64_t nc, int particle_bc,
                                 pb_status *status, void *scratch, size_t scratch_bytes,
                                 int64_t *n_new, void *stream) {
  if (nsp < 0 || nsp > PB_MAX_SPECIES || (nsp > 0 && (!src || !dst || !cv || !n_new))) {
    pb::set_error("pb_canonical_step: bad arguments");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  for (int k = 0; k < nsp; ++k) {
    const int rc = pb_canonical_resort(&src[k], &dst[k], &cv[k], e_nodes, nc, particle_bc, k,
                                       status, scratch, scratch_bytes, stream);
    if (rc) return rc;
  }
  for (int k = 0; k < nsp; ++k) {
    const cudaError_t e = cudaMemcpyAsync(&n_new[k], cv[k].offs + nc, sizeof(int64_t),
                                          cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return pb::cuda_status(e, "cudaMemcpyAsync");
  }
  const cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? PB_OK : pb::cuda_status(e, "cudaStreamSynchronize");
}

// Multi-rank canonical step, first half: push + transfer every particle of
// the species in place and write its key (dest cell, moved, global canonical
// rank = rank_offset + local rank) to keys[0, n_old + n_tail) -- all ones for
// vacated / absorbed slots.  The caller exchanges emigrants between ranks and
// orders the union by key (the same order pb_canonical_resort produces).
extern "C" int pb_canonical_keys(const pb_species *src, const pb_canon *cv, const double *e_nodes,
                                 int64_t nc, int particle_bc, int species_id, pb_status *status,
                                 int64_t rank_offset, int rank_bits, int64_t *keys,
                                 void *scratch, size_t scratch_bytes, void *stream) {
  if (!src || !cv || !status || !keys || nc < 1 || species_id < 0 || species_id >= PB_MAX_SPECIES ||
      rank_bits < 1 || rank_bits + pb::bits_for((uint64_t)(2 * nc)) > 63) {
    pb::set_error("pb_canonical_keys: bad arguments");
    return PB_ERR_INVALID;
  }
  const int64_t n_tot = cv->n_old + cv->n_tail;
  if (n_tot == 0) return PB_OK;
  if (!scratch || scratch_bytes < pb_canonical_scratch_bytes(n_tot, nc)) {
    pb::set_error("pb_canonical_keys: scratch too small");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char *p = (char *)scratch;
  p += 2 * pb::a256((size_t)n_tot * 8);
  uint32_t *vals = (uint32_t *)p;
  p += 2 * pb::a256((size_t)n_tot * 4);
  int64_t *offp = (int64_t *)p;
  p += pb::a256((size_t)(nc + 1) * 8);
  int64_t *pre = (int64_t *)p;
  p += pb::a256((size_t)nc * 8);
  p += pb::a256(pb::sort_temp_bytes(n_tot));
  char *scan_tmp = p;
  pb::k_sum_counts<<<148, 256, 0, st>>>(cv->counts, cv->n_tail ? cv->newborn_per_cell : nullptr,
                                        pre, nc);
  PB_CHECK_LAUNCH("k_sum_counts");
  int rc = pb::offsets_from_counts(pre, offp, nc, scan_tmp, st);
  if (rc) return rc;
  return pb::launch_canon_push(src, cv, e_nodes, nc, particle_bc, species_id, status, rank_offset,
                               rank_bits, offp, (uint64_t *)keys, vals, st);
}

// Weighted partials + stitch from per-species fp64 partials (the bitwise
// sequential deposit of pb_deposit_partials): fields.py:64-92, :115-117.
namespace pb {
struct RawCoef {
  double c[PB_MAX_SPECIES];
};
__device__ __forceinline__ void raw_partials(const double *__restrict__ raw, const RawCoef &ca,
                                             int ndep, int64_t nc, int64_t j, double &l,
                                             double &r) {
  double a = 0.0, b = 0.0;
  for (int s = 0; s < ndep; ++s) {
    a = __dadd_rn(a, __dmul_rn(ca.c[s], raw[(size_t)s * 2 * nc + j]));
    b = __dadd_rn(b, __dmul_rn(ca.c[s], raw[(size_t)s * 2 * nc + nc + j]));
  }
  l = a;
  r = b;
}
__global__ void k_rho_raw(const double *__restrict__ raw, RawCoef ca, int ndep, int64_t nc,
                          int field_bc, double *__restrict__ left, double *__restrict__ right,
                          double *__restrict__ rho) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g > nc) return;
  double lg = 0.0, rg = 0.0, lp = 0.0, rp = 0.0;
  if (g < nc) {
    raw_partials(raw, ca, ndep, nc, g, lg, rg);
    if (left) left[g] = lg;
    if (right) right[g] = rg;
  }
  if (g > 0) raw_partials(raw, ca, ndep, nc, g - 1, lp, rp);
  double v;
  if (g > 0 && g < nc) {
    v = __dadd_rn(rp, lg);
  } else if (field_bc == PB_FIELD_PERIODIC) {
    double l0, r0, ll, rl;
    raw_partials(raw, ca, ndep, nc, 0, l0, r0);
    raw_partials(raw, ca, ndep, nc, nc - 1, ll, rl);
    v = __dadd_rn(rl, l0);
  } else if (g == 0) {
    v = __dmul_rn(lg, 2.0);
  } else {
    v = __dmul_rn(rp, 2.0);
  }
  rho[g] = v;
}
}  // namespace pb

extern "C" int pb_rho_from_partials(const double *raw, const double *coef, int ndep, int64_t nc,
                                    int field_bc, double *left, double *right, double *rho,
                                    void *stream) {
  if (ndep < 0 || ndep > PB_MAX_SPECIES || nc < 1 || !rho || (ndep > 0 && (!raw || !coef)) ||
      (field_bc != PB_FIELD_PERIODIC && field_bc != PB_FIELD_DIRICHLET)) {
    pb::set_error("pb_rho_from_partials: bad arguments");
    return PB_ERR_INVALID;
  }
  pb::RawCoef ca;
  memset(&ca, 0, sizeof(ca));
  for (int s = 0; s < ndep; ++s) ca.c[s] = coef[s];
  const int64_t blocks = (nc + 1 + 255) / 256;
  pb::k_rho_raw<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(raw, ca, ndep, nc, field_bc,
                                                                     left, right, rho);
  PB_CHECK_LAUNCH("k_rho_raw");
  return PB_OK;
}

extern "C" int pb_set_canonical_scatter_min(int64_t n) {
  if (n < 0) {
    pb::set_error("pb_set_canonical_scatter_min: n=%lld < 0", (long long)n);
    return PB_ERR_INVALID;
  }
  pb::g_scatter_min = n;
  return PB_OK;
}
