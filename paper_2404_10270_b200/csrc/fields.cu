// Replicated field pipeline: 1-2-1 smoothing, Poisson solve, E = -grad phi.
//
// The grid is tiny next to the particle arrays (nc+1 doubles), so every GPU
// holds a replica and solves it locally after the density allreduce.  The
// stencils reproduce the reference's NumPy expression order exactly
// (pkg/src/picmc/fields.py:121-135, :205-218).  The Poisson solve offers the
// reference's direct elimination (fields.py:138-202), restated operation for
// operation -- including NumPy's pairwise summation inside np.mean -- on one
// thread, so a given rho yields a bitwise-identical phi.
#include "common.cuh"
#include "density.cuh"

#include <cstring>

namespace pb {

// ---- stencils ---------------------------------------------------------------
// core = 0.25*roll(core,1) + 0.5*core + 0.25*roll(core,-1); out[nc] = out[0]
__device__ __forceinline__ void smooth_node(const double *__restrict__ in, double *__restrict__ out,
                                            int64_t nc, int64_t j) {
  const int64_t jj = j == nc ? 0 : j;
  const double a = in[jj == 0 ? nc - 1 : jj - 1];
  const double b = in[jj];
  const double c = in[jj == nc - 1 ? 0 : jj + 1];
  out[j] = __dadd_rn(__dadd_rn(__dmul_rn(0.25, a), __dmul_rn(0.5, b)), __dmul_rn(0.25, c));
}

__global__ void k_smooth_pass(const double *__restrict__ in,
                              double *__restrict__ out, int64_t nc) {
  pdl_enter();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > nc) return;
  smooth_node(in, out, nc, j);
}

__device__ __forceinline__ void efield_node(const double *__restrict__ phi, double *__restrict__ e,
                                            int64_t nc, double two_dx, int field_bc, int64_t j) {
  if (field_bc == PB_FIELD_PERIODIC) {
    const int64_t jj = j == nc ? 0 : j;  // e[nc] = e[0]
    const double l = phi[jj == 0 ? nc - 1 : jj - 1];
    const double r = phi[jj == nc - 1 ? 0 : jj + 1];
    e[j] = __ddiv_rn(__dsub_rn(l, r), two_dx);
    return;
  }
  if (j == 0) {
    const double t = __dadd_rn(__dsub_rn(__dmul_rn(3.0, phi[0]), __dmul_rn(4.0, phi[1])), phi[2]);
    e[0] = __ddiv_rn(t, two_dx);
  } else if (j == nc) {
    const double t = __dadd_rn(__dsub_rn(__dmul_rn(3.0, phi[nc]), __dmul_rn(4.0, phi[nc - 1])),
                               phi[nc - 2]);
    e[nc] = __ddiv_rn(-t, two_dx);
  } else {
    e[j] = __ddiv_rn(__dsub_rn(phi[j - 1], phi[j + 1]), two_dx);
  }
}

__global__ void k_efield(const double *__restrict__ phi, double *__restrict__ e,
                         int64_t nc, double two_dx, int field_bc) {
  pdl_enter();
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > nc) return;
  efield_node(phi, e, nc, two_dx, field_bc, j);
}

// ---- NumPy-exact reductions -------------------------------------------------
// numpy pairwise_sum for float64 (blocks of 8 accumulators, PW_BLOCKSIZE 128).
__device__ double pairwise_sum(const double *a, int64_t n) {
  // Iterative restatement of the recursion: an explicit stack of ranges.
  struct R { int64_t lo, n; int state; double left; };
  R stk[64];
  int sp = 0;
  double ret = 0.0;
  stk[sp++] = {0, n, 0, 0.0};
  while (sp) {
    R &f = stk[sp - 1];
    if (f.n < 8) {
      double res = -0.0;  // numpy starts from the reduction identity (-0.0)
      for (int64_t i = 0; i < f.n; ++i) res = __dadd_rn(res, a[f.lo + i]);
      ret = res;
      --sp;
    } else if (f.n <= 128) {
      double r[8];
      for (int k = 0; k < 8; ++k) r[k] = a[f.lo + k];
      int64_t i;
      for (i = 8; i < f.n - (f.n % 8); i += 8)
        for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], a[f.lo + i + k]);
      double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                             __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < f.n; ++i) res = __dadd_rn(res, a[f.lo + i]);
      ret = res;
      --sp;
    } else {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      if (f.state == 0) {
        f.state = 1;
        stk[sp++] = {f.lo, n2, 0, 0.0};
      } else if (f.state == 1) {
        f.left = ret;
        f.state = 2;
        stk[sp++] = {f.lo + n2, f.n - n2, 0, 0.0};
      } else {
        ret = __dadd_rn(f.left, ret);
        --sp;
      }
    }
  }
  return ret;
}

// np.add.reduce over a contiguous float64 array is one pairwise_sum over
// all n elements (checked against NumPy 2.3 for n = 3 .. 1e5).
__device__ double np_sum(const double *a, int64_t n) {
  if (n == 0) return 0.0;
  return pairwise_sum(a, n);
}

// _thomas_unit (fields.py:138-153) on rhs[0..n) -> x[0..n); diag/y scratch.
__device__ void thomas_unit(const double *rhs, double *x, double *diag,
                            double *y, int64_t n) {
  diag[0] = -2.0;
  y[0] = rhs[0];
  for (int64_t i = 1; i < n; ++i) {
    const double m = __ddiv_rn(1.0, diag[i - 1]);
    diag[i] = __dsub_rn(-2.0, m);
    y[i] = __dsub_rn(rhs[i], __dmul_rn(m, y[i - 1]));
  }
  x[n - 1] = __ddiv_rn(y[n - 1], diag[n - 1]);
  for (int64_t i = n - 2; i >= 0; --i)
    x[i] = __ddiv_rn(__dsub_rn(y[i], x[i + 1]), diag[i]);
}

// solve_poisson (fields.py:156-202), one thread.
__global__ void k_poisson_exact(const double *__restrict__ rho, double *phi,
                                int64_t nc, double scale, int field_bc,
                                double phi_left, double phi_right,
                                double *scratch) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double *rhs = scratch;
  double *diag = scratch + (nc + 1);
  double *y = scratch + 2 * (nc + 1);
  if (field_bc == PB_FIELD_PERIODIC) {
    const double mean = __ddiv_rn(np_sum(rho, nc), (double)nc);
    for (int64_t j = 0; j < nc; ++j)
      rhs[j] = __dmul_rn(-__dsub_rn(rho[j], mean), scale);
    phi[0] = 0.0;
    thomas_unit(rhs + 1, phi + 1, diag, y, nc - 1);
    phi[nc] = phi[0];
    const double shift = __ddiv_rn(np_sum(phi, nc), (double)nc);
    for (int64_t j = 0; j <= nc; ++j) phi[j] = __dsub_rn(phi[j], shift);
  } else {
    for (int64_t j = 1; j < nc; ++j) rhs[j - 1] = __dmul_rn(-rho[j], scale);
    rhs[0] = __dsub_rn(rhs[0], phi_left);
    rhs[nc - 2] = __dsub_rn(rhs[nc - 2], phi_right);
    phi[0] = phi_left;
    phi[nc] = phi_right;
    thomas_unit(rhs, phi + 1, diag, y, nc - 1);
  }
}

// ---- parallel Poisson (scan form) ---------------------------------------------
// The (1,-2,1) elimination has closed-form pivots d_i = -(i+2)/(i+1), so the
// forward sweep y_i = rhs_i - y_{i-1}/d_{i-1} becomes z_i = z_{i-1} + (i+1) rhs_i
// with y_i = z_i/(i+1), and the back substitution x_i = (y_i - x_{i+1})/d_i
// becomes w_i = w_{i+1} - y_i/(i+2) with x_i = (i+1) w_i: two prefix sums.
// Sums run in double-double (TwoSum) so the result matches the serial
// elimination to ~1e-15 relative; one block of 1024 threads, contiguous
// per-thread segments, shared-memory scan of the segment totals.
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  const double s = __dadd_rn(a.hi, b.hi);
  const double bb = __dsub_rn(s, a.hi);
  const double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
  const double e = __dadd_rn(err, __dadd_rn(a.lo, b.lo));
  const double hi = __dadd_rn(s, e);
  return {hi, __dsub_rn(e, __dsub_rn(hi, s))};
}
__device__ __forceinline__ DD dd_of(double v) { return {v, 0.0}; }

// ---- multi-block scan solve ------------------------------------------------
// Closed-form pivots d_k = -(k+2)/(k+1) turn the two Thomas sweeps into
//   z_k = sum_{i<=k} (i+1) rhs_i,  y_k = z_k/(k+1)          (forward)
//   w_k = sum_{i>=k} -y_i/(i+2),   x_k = (k+1) w_k          (backward)
// Both are prefix sums, done with double-double accumulation over a grid of
// 512-element tiles (256 threads x 2; the phases are latency-bound, so more,
// smaller blocks win: config 3 step -3% against 2048-element tiles, 1 per
// thread no better): per-tile DD partials, then every block adds the
// partials before it (deterministic order) and scans its own tile.
#ifndef PB_MB_PER
#define PB_MB_PER 2
#endif
constexpr int kMbThreads = 256;
constexpr int kMbPer = PB_MB_PER;
constexpr int kMbTile = kMbThreads * kMbPer;

__device__ __forceinline__ DD dd_shfl_up(DD v, int d) {
  return {__shfl_up_sync(0xffffffffu, v.hi, d), __shfl_up_sync(0xffffffffu, v.lo, d)};
}
__device__ __forceinline__ DD dd_shfl_down(DD v, int d) {
  return {__shfl_down_sync(0xffffffffu, v.hi, d), __shfl_down_sync(0xffffffffu, v.lo, d)};
}

constexpr int kMbWarps = kMbThreads / 32;

// Block sum (every thread gets it): a shuffle tree in each warp, then the
// warp sums in warp order.  A fixed tree, so every block computing the same
// sum gets the same bits.
__device__ DD mb_block_reduce(DD v, DD *sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const DD o = dd_shfl_down(v, d);
    if (lane + d < 32) v = dd_add(v, o);
  }
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  DD r = sm[0];
#pragma unroll
  for (int w = 1; w < kMbWarps; ++w) r = dd_add(r, sm[w]);
  __syncthreads();
  return r;
}

// Exclusive scan over threads in order t (rev = false) or NT-1-t (rev = true):
// a shuffle scan in each warp (logical lane order), the warp totals
// scanned in logical warp order through shared memory.
__device__ DD mb_block_excl(DD v, DD *sm, bool rev) {
  const int t = rev ? kMbThreads - 1 - (int)threadIdx.x : (int)threadIdx.x;  // logical position
  const int lane = t & 31, warp = t >> 5;
  DD inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const DD o = rev ? dd_shfl_down(inc, d) : dd_shfl_up(inc, d);  // logical lane - d
    if (lane >= d) inc = dd_add(o, inc);
  }
  DD lex = rev ? dd_shfl_down(inc, 1) : dd_shfl_up(inc, 1);
  if (lane == 0) lex = dd_of(0.0);
  if (lane == 31) sm[warp] = inc;
  __syncthreads();
  DD wex = dd_of(0.0);
  for (int w = 0; w < warp; ++w) wex = dd_add(wex, sm[w]);
  __syncthreads();
  return dd_add(wex, lex);
}

// Sum of part[lo, hi) in index order (each block computes the same value).
__device__ DD mb_sum_parts(const DD *part, int64_t lo, int64_t hi, DD *sm) {
  DD acc = dd_of(0.0);
  for (int64_t i = lo + threadIdx.x; i < hi; i += kMbThreads) acc = dd_add(acc, part[i]);
  return mb_block_reduce(acc, sm);
}

struct PoissonArgs {
  const double *rho;
  double *phi;
  double *y;
  DD *p0, *p1, *p2, *p3;  // per-tile partials: rho, forward, backward, phi
  int64_t nc, n;
  int nt;                 // tiles over the n unknowns
  int ntc;                // tiles over the nc nodes
  double scale, phi_left, phi_right;
  int field_bc;
};

__device__ __forceinline__ double mb_mean(const PoissonArgs &a, DD *sm) {
  if (a.field_bc != PB_FIELD_PERIODIC) return 0.0;
  const DD s = mb_sum_parts(a.p0, 0, a.ntc, sm);
  return __ddiv_rn(__dadd_rn(s.hi, s.lo), (double)a.nc);
}

__device__ __forceinline__ double mb_rhs(const PoissonArgs &a, int64_t k, double mean) {
  if (a.field_bc == PB_FIELD_PERIODIC) return __dmul_rn(-__dsub_rn(a.rho[k + 1], mean), a.scale);
  double r = __dmul_rn(-a.rho[k + 1], a.scale);
  if (k == 0) r = __dsub_rn(r, a.phi_left);
  if (k == a.n - 1) r = __dsub_rn(r, a.phi_right);
  return r;
}

// ---- scan phases, one tile each ----------------------------------------------
// tile partial sums of src[0, len) -> part[tile]
__device__ void mb_tile_sum(const double *__restrict__ src, int64_t len, DD *part, int64_t tile,
                            DD *sm) {
  const int64_t base = tile * kMbTile + (int64_t)threadIdx.x * kMbPer;
  DD acc = dd_of(0.0);
  for (int j = 0; j < kMbPer; ++j)
    if (base + j < len) acc = dd_add(acc, dd_of(src[base + j]));
  const DD r = mb_block_reduce(acc, sm);
  if (threadIdx.x == 0) part[tile] = r;
}

__device__ void mb_fwd_part(const PoissonArgs &a, int64_t tile, DD *sm) {
  const double mean = mb_mean(a, sm);
  const int64_t base = tile * kMbTile + (int64_t)threadIdx.x * kMbPer;
  DD acc = dd_of(0.0);
  for (int j = 0; j < kMbPer; ++j) {
    const int64_t k = base + j;
    if (k < a.n) acc = dd_add(acc, dd_of(__dmul_rn((double)(k + 1), mb_rhs(a, k, mean))));
  }
  const DD r = mb_block_reduce(acc, sm);
  if (threadIdx.x == 0) a.p1[tile] = r;
}

__device__ void mb_fwd_scan(const PoissonArgs &a, int64_t tile, DD *sm) {
  const double mean = mb_mean(a, sm);
  const DD before = mb_sum_parts(a.p1, 0, tile, sm);
  const int64_t base = tile * kMbTile + (int64_t)threadIdx.x * kMbPer;
  double v[kMbPer];
  DD loc = dd_of(0.0);
  for (int j = 0; j < kMbPer; ++j) {
    const int64_t k = base + j;
    v[j] = k < a.n ? __dmul_rn((double)(k + 1), mb_rhs(a, k, mean)) : 0.0;
    loc = dd_add(loc, dd_of(v[j]));
  }
  DD off = dd_add(before, mb_block_excl(loc, sm, false));
  DD bsum = dd_of(0.0);
  for (int j = 0; j < kMbPer; ++j) {
    const int64_t k = base + j;
    if (k >= a.n) break;
    off = dd_add(off, dd_of(v[j]));
    const double y = __ddiv_rn(__dadd_rn(off.hi, off.lo), (double)(k + 1));
    a.y[k] = y;
    bsum = dd_add(bsum, dd_of(-__ddiv_rn(y, (double)(k + 2))));
  }
  const DD r = mb_block_reduce(bsum, sm);
  if (threadIdx.x == 0) a.p2[tile] = r;
}

__device__ void mb_bwd_scan(const PoissonArgs &a, int64_t tile, DD *sm) {
  const DD after = mb_sum_parts(a.p2, tile + 1, a.nt, sm);
  const int64_t base = tile * kMbTile + (int64_t)threadIdx.x * kMbPer;
  double u[kMbPer];
  DD loc = dd_of(0.0);
  for (int j = kMbPer - 1; j >= 0; --j) {
    const int64_t k = base + j;
    u[j] = k < a.n ? -__ddiv_rn(a.y[k], (double)(k + 2)) : 0.0;
    loc = dd_add(loc, dd_of(u[j]));
  }
  DD off = dd_add(after, mb_block_excl(loc, sm, true));
  for (int j = kMbPer - 1; j >= 0; --j) {
    const int64_t k = base + j;
    if (k >= a.n) continue;
    off = dd_add(off, dd_of(u[j]));
    a.phi[k + 1] = __dmul_rn((double)(k + 1), __dadd_rn(off.hi, off.lo));
  }
  if (tile == 0 && threadIdx.x == 0) {
    if (a.field_bc == PB_FIELD_PERIODIC) {
      a.phi[0] = 0.0;
    } else {
      a.phi[0] = a.phi_left;
      a.phi[a.nc] = a.phi_right;
    }
  }
}

// periodic: phi[0..nc) -= mean(phi[:nc]) over nodes j = first, first+stride, ...
__device__ void mb_shift(const PoissonArgs &a, int64_t first, int64_t stride, DD *sm) {
  const DD s = mb_sum_parts(a.p3, 0, a.ntc, sm);
  const double shift = __ddiv_rn(__dadd_rn(s.hi, s.lo), (double)a.nc);
  for (int64_t j = first; j < a.nc; j += stride) a.phi[j] = __dsub_rn(a.phi[j], shift);
}

__global__ void __launch_bounds__(kMbThreads) k_mb_tile_sum(const double *__restrict__ src,
                                                            int64_t len, DD *part) {
  pdl_enter();
  __shared__ DD sm[kMbThreads];
  mb_tile_sum(src, len, part, blockIdx.x, sm);
}

__global__ void __launch_bounds__(kMbThreads) k_mb_fwd_part(const PoissonArgs a) {
  pdl_enter();
  __shared__ DD sm[kMbThreads];
  mb_fwd_part(a, blockIdx.x, sm);
}

__global__ void __launch_bounds__(kMbThreads) k_mb_fwd_scan(const PoissonArgs a) {
  pdl_enter();
  __shared__ DD sm[kMbThreads];
  mb_fwd_scan(a, blockIdx.x, sm);
}

__global__ void __launch_bounds__(kMbThreads) k_mb_bwd_scan(const PoissonArgs a) {
  pdl_enter();
  __shared__ DD sm[kMbThreads];
  mb_bwd_scan(a, blockIdx.x, sm);
}

__global__ void __launch_bounds__(kMbThreads) k_mb_shift(const PoissonArgs a) {
  pdl_enter();
  __shared__ DD sm[kMbThreads];
  mb_shift(a, (int64_t)blockIdx.x * kMbThreads + threadIdx.x, (int64_t)gridDim.x * kMbThreads, sm);
}

__global__ void k_mb_wrap(double *phi, int64_t nc) {
  pdl_enter();
  phi[nc] = phi[0];
}


// E from phi, then zero bin sets whose density has been taken (the serial
// field-solve cycle reads the bins with the one-kernel epilogue, which does
// not clear them -- neighbouring nodes read the same cells -- and clears
// them here, one launch later, before the push deposits again).
__global__ void k_efield_clear(const double *__restrict__ phi, double *__restrict__ e, int64_t nc,
                               double two_dx, int field_bc, uint64_t *__restrict__ clr_a,
                               uint64_t *__restrict__ clr_b, int64_t nwords) {
  pdl_enter();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g <= nc) efield_node(phi, e, nc, two_dx, field_bc, g);
  for (int64_t w = g; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    if (clr_a) clr_a[w] = 0;
    if (clr_b) clr_b[w] = 0;
  }
}

static unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

static PoissonArgs poisson_args(const double *rho, double *phi, int64_t nc, double dx, double eps0,
                                int field_bc, double phi_left, double phi_right, void *scratch) {
  PoissonArgs a;
  a.rho = rho;
  a.phi = phi;
  a.nc = nc;
  a.n = nc - 1;
  a.nt = (int)((a.n + kMbTile - 1) / kMbTile);
  a.ntc = (int)((nc + kMbTile - 1) / kMbTile);
  a.scale = (dx * dx) / eps0;
  a.phi_left = phi_left;
  a.phi_right = phi_right;
  a.field_bc = field_bc;
  a.y = (double *)scratch;
  const size_t off = ((size_t)(nc + 1) * sizeof(double) + 255) & ~(size_t)255;
  DD *parts = (DD *)((char *)scratch + off);
  const int ptile = a.ntc + 1;
  a.p0 = parts;
  a.p1 = parts + ptile;
  a.p2 = parts + 2 * ptile;
  a.p3 = parts + 3 * ptile;
  return a;
}

// The density epilogue with one smoothing pass folded in (pb_field_cycle,
// passes == 1): thread g forms rho at nodes g-1, g, g+1 from the bins
// itself (the same weighted partials k_rho_epilogue forms, so the same
// bits) and smooths them -- one launch instead of k_rho_epilogue +
// k_smooth_pass, bitwise the same left / right / rho / rho_s.
struct RhoSmoothArgs {
  const uint64_t *bins;
  CoefArgs ca;
  int ndep, field_bc;
  int64_t nc;
  double *left, *right, *rho, *rho_s;
  pb_status *st;
};

// core value rho[c] of node c in [0, nc) (the array the smoothing wraps over)
__device__ __forceinline__ double rs_core(const RhoSmoothArgs &a, int64_t c, double lc, double rcm1) {
  return (a.field_bc != PB_FIELD_PERIODIC && c == 0) ? __dmul_rn(lc, 2.0) : __dadd_rn(rcm1, lc);
}

__global__ void k_rho_smooth(const __grid_constant__ RhoSmoothArgs a) {
  pdl_enter();
  const int64_t nc = a.nc;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g > nc) return;
  const int64_t jj = g == nc ? 0 : g;
  const int64_t jm = jj == 0 ? nc - 1 : jj - 1, jp = jj == nc - 1 ? 0 : jj + 1;
  const int64_t jmm = jm == 0 ? nc - 1 : jm - 1;
  double l_m, r_m, l_0, r_0, l_p, r_p, l_mm, r_mm;
  weighted_partials(a.bins, a.ca.c, a.ndep, nc, jj, l_0, r_0, g < nc ? a.st : nullptr);
  weighted_partials(a.bins, a.ca.c, a.ndep, nc, jm, l_m, r_m, nullptr);
  weighted_partials(a.bins, a.ca.c, a.ndep, nc, jp, l_p, r_p, nullptr);
  weighted_partials(a.bins, a.ca.c, a.ndep, nc, jmm, l_mm, r_mm, nullptr);
  (void)r_p;
  const double c0 = rs_core(a, jj, l_0, r_m);
  const double cm = rs_core(a, jm, l_m, r_mm);
  const double cp = rs_core(a, jp, l_p, r_0);
  if (g < nc) {
    if (a.left) a.left[g] = l_0;
    if (a.right) a.right[g] = r_0;
    a.rho[g] = c0;
  } else {
    a.rho[nc] = a.field_bc == PB_FIELD_PERIODIC ? c0 : __dmul_rn(r_m, 2.0);  // rho[0] / 2 R[nc-1]
  }
  a.rho_s[g] = __dadd_rn(__dadd_rn(__dmul_rn(0.25, cm), __dmul_rn(0.5, c0)), __dmul_rn(0.25, cp));
}

}  // namespace pb

extern "C" size_t pb_field_scratch_bytes(int64_t nc) {
  // smoothing ping-pong + the scan solve's y and DD tile partials
  const size_t tiles = (size_t)((nc + 1 + pb::kMbTile - 1) / pb::kMbTile) + 1;
  return 4 * (size_t)(nc + 1) * sizeof(double) + 4 * tiles * sizeof(pb::DD) + 512;
}

extern "C" int pb_smooth_density(const double *rho, double *out, int64_t nc,
                                 int passes, void *scratch, void *stream) {
  if (nc < 2 || passes < 0 || !rho || !out || (passes > 1 && !scratch)) {
    pb::set_error("pb_smooth_density: bad arguments");
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (passes == 0) {
    // smooth_density(rho, 0) returns a copy with out[nc] = out[0]
    cudaError_t e = cudaMemcpyAsync(out, rho, (size_t)nc * sizeof(double),
                                    cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return pb::cuda_status(e, "cudaMemcpyAsync");
    e = cudaMemcpyAsync(out + nc, rho, sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return pb::cuda_status(e, "cudaMemcpyAsync");
    return PB_OK;
  }
  // Ping-pong so the last pass lands in `out`.
  double *tmp = (double *)scratch;
  const double *src = rho;
  for (int p = 0; p < passes; ++p) {
    double *dst = ((passes - 1 - p) % 2 == 0) ? out : tmp;
    cudaError_t e = pb::launch_pdl(pb::k_smooth_pass, dim3(pb::blocks_for(nc + 1, 256)), dim3(256), 0,
                                   st, src, dst, nc);
    if (e != cudaSuccess) return pb::cuda_status(e, "k_smooth_pass");
    src = dst;
  }
  return PB_OK;
}

extern "C" int pb_solve_poisson(const double *rho, double *phi, int64_t nc,
                                double dx, double eps0, int field_bc,
                                double phi_left, double phi_right,
                                void *scratch, void *stream) {
  if (nc < 3) {
    pb::set_error("poisson solve needs nc >= 3, got %lld", (long long)nc);
    return PB_ERR_INVALID;
  }
  if (!rho || !phi || !scratch) {
    pb::set_error("pb_solve_poisson: NULL argument");
    return PB_ERR_INVALID;
  }
  if (field_bc != PB_FIELD_PERIODIC && field_bc != PB_FIELD_DIRICHLET) {
    pb::set_error("unknown boundary condition %d", field_bc);
    return PB_ERR_INVALID;
  }
  const double scale = (dx * dx) / eps0;  // grid.dx_m * grid.dx_m / eps0
  pb::k_poisson_exact<<<1, 32, 0, (cudaStream_t)stream>>>(
      rho, phi, nc, scale, field_bc, phi_left, phi_right, (double *)scratch);
  PB_CHECK_LAUNCH("k_poisson_exact");
  return PB_OK;
}

extern "C" int pb_solve_poisson_scan(const double *rho, double *phi, int64_t nc, double dx,
                                     double eps0, int field_bc, double phi_left,
                                     double phi_right, void *scratch, void *stream) {
  if (nc < 3) {
    pb::set_error("poisson solve needs nc >= 3, got %lld", (long long)nc);
    return PB_ERR_INVALID;
  }
  if (!rho || !phi || !scratch) {
    pb::set_error("pb_solve_poisson_scan: NULL argument");
    return PB_ERR_INVALID;
  }
  if (field_bc != PB_FIELD_PERIODIC && field_bc != PB_FIELD_DIRICHLET) {
    pb::set_error("unknown boundary condition %d", field_bc);
    return PB_ERR_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  pb::PoissonArgs a = pb::poisson_args(rho, phi, nc, dx, eps0, field_bc, phi_left, phi_right, scratch);
  const dim3 tb(pb::kMbThreads);
  cudaError_t e = cudaSuccess;
  if (field_bc == PB_FIELD_PERIODIC && e == cudaSuccess)
    e = pb::launch_pdl(pb::k_mb_tile_sum, dim3(a.ntc), tb, 0, st, rho, nc, a.p0);
  if (e == cudaSuccess) e = pb::launch_pdl(pb::k_mb_fwd_part, dim3(a.nt), tb, 0, st, a);
  if (e == cudaSuccess) e = pb::launch_pdl(pb::k_mb_fwd_scan, dim3(a.nt), tb, 0, st, a);
  if (e == cudaSuccess) e = pb::launch_pdl(pb::k_mb_bwd_scan, dim3(a.nt), tb, 0, st, a);
  if (field_bc == PB_FIELD_PERIODIC) {
    if (e == cudaSuccess)
      e = pb::launch_pdl(pb::k_mb_tile_sum, dim3(a.ntc), tb, 0, st, (const double *)phi, nc, a.p3);
    if (e == cudaSuccess) e = pb::launch_pdl(pb::k_mb_shift, dim3(a.ntc), tb, 0, st, a);
    if (e == cudaSuccess) e = pb::launch_pdl(pb::k_mb_wrap, dim3(1), dim3(1), 0, st, phi, nc);
  }
  if (e != cudaSuccess) return pb::cuda_status(e, "poisson scan");
  PB_CHECK_LAUNCH("poisson scan");
  return PB_OK;
}

extern "C" int pb_compute_efield(const double *phi, double *e, int64_t nc,
                                 double dx, int field_bc, void *stream) {
  if (nc < 3 || !phi || !e) {
    pb::set_error("pb_compute_efield: bad arguments");
    return PB_ERR_INVALID;
  }
  cudaError_t err = pb::launch_pdl(pb::k_efield, dim3(pb::blocks_for(nc + 1, 256)), dim3(256), 0,
                                   (cudaStream_t)stream, phi, e, nc, 2.0 * dx, field_bc);
  if (err != cudaSuccess) return pb::cuda_status(err, "k_efield");
  return PB_OK;
}

extern "C" int pb_compute_efield_clear(const double *phi, double *e, int64_t nc, double dx,
                                       int field_bc, uint64_t *clr_a, uint64_t *clr_b,
                                       int64_t nwords, void *stream) {
  if (nc < 3 || !phi || !e || nwords < 0) {
    pb::set_error("pb_compute_efield_clear: bad arguments");
    return PB_ERR_INVALID;
  }
  cudaError_t err = pb::launch_pdl(pb::k_efield_clear, dim3(pb::blocks_for(nc + 1, 256)), dim3(256), 0,
                                   (cudaStream_t)stream, phi, e, nc, 2.0 * dx, field_bc, clr_a, clr_b,
                                   nwords);
  if (err != cudaSuccess) return pb::cuda_status(err, "k_efield_clear");
  return PB_OK;
}


extern "C" int pb_field_cycle(const uint64_t *bins, const double *coef, int ndep, int64_t nc,
                              int field_bc, int passes, double dx, double eps0, double phi_left,
                              double phi_right, double *left, double *right, double *rho,
                              double *rho_s, double *phi, double *e, uint64_t *clr_a,
                              uint64_t *clr_b, int64_t nwords, pb_status *status, void *scratch,
                              void *stream) {
  if (nc < 3 || ndep < 0 || ndep > PB_MAX_SPECIES || (ndep > 0 && (!bins || !coef)) || !rho ||
      !rho_s || !phi || !e || !scratch || nwords < 0) {
    pb::set_error("pb_field_cycle: bad arguments (nc=%lld ndep=%d)", (long long)nc, ndep);
    return PB_ERR_INVALID;
  }
  if (passes < 0) {
    pb::set_error("pb_field_cycle: %d smoothing passes", passes);
    return PB_ERR_INVALID;
  }
  if (field_bc != PB_FIELD_PERIODIC && field_bc != PB_FIELD_DIRICHLET) {
    pb::set_error("unknown boundary condition %d", field_bc);
    return PB_ERR_INVALID;
  }
  int rc = PB_OK;
  if (passes == 1) {
    pb::RhoSmoothArgs a;
    memset(&a, 0, sizeof(a));
    a.bins = bins;
    for (int s = 0; s < ndep; ++s) a.ca.c[s] = coef[s];
    a.ndep = ndep;
    a.field_bc = field_bc;
    a.nc = nc;
    a.left = left;
    a.right = right;
    a.rho = rho;
    a.rho_s = rho_s;
    a.st = status;
    cudaError_t err = pb::launch_pdl(pb::k_rho_smooth, dim3(pb::blocks_for(nc + 1, 256)), dim3(256), 0,
                                     (cudaStream_t)stream, a);
    if (err != cudaSuccess) return pb::cuda_status(err, "k_rho_smooth");
  } else {
    rc = pb_rho_epilogue(bins, coef, ndep, nc, field_bc, left, right, rho, status, stream);
    if (!rc) rc = pb_smooth_density(rho, rho_s, nc, passes, scratch, stream);
  }
  if (!rc) rc = pb_solve_poisson_scan(rho_s, phi, nc, dx, eps0, field_bc, phi_left, phi_right, scratch, stream);
  if (!rc) rc = pb_compute_efield_clear(phi, e, nc, dx, field_bc, clr_a, clr_b, (clr_a || clr_b) ? nwords : 0, stream);
  return rc;
}
