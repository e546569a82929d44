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
#include "compact.cuh"
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

// E at node j from phi(i) (a getter: the phi array, or the fused cycle's
// shifted L2 reads)
template <typename Phi>
__device__ __forceinline__ void efield_node_g(const Phi &phi, double *__restrict__ e, int64_t nc,
                                              double two_dx, int field_bc, int64_t j) {
  if (field_bc == PB_FIELD_PERIODIC) {
    const int64_t jj = j == nc ? 0 : j;  // e[nc] = e[0]
    const double l = phi(jj == 0 ? nc - 1 : jj - 1);
    const double r = phi(jj == nc - 1 ? 0 : jj + 1);
    e[j] = __ddiv_rn(__dsub_rn(l, r), two_dx);
    return;
  }
  if (j == 0) {
    const double t = __dadd_rn(__dsub_rn(__dmul_rn(3.0, phi(0)), __dmul_rn(4.0, phi(1))), phi(2));
    e[0] = __ddiv_rn(t, two_dx);
  } else if (j == nc) {
    const double t = __dadd_rn(__dsub_rn(__dmul_rn(3.0, phi(nc)), __dmul_rn(4.0, phi(nc - 1))),
                               phi(nc - 2));
    e[nc] = __ddiv_rn(-t, two_dx);
  } else {
    e[j] = __ddiv_rn(__dsub_rn(phi(j - 1), phi(j + 1)), two_dx);
  }
}

__device__ __forceinline__ void efield_node(const double *__restrict__ phi, double *__restrict__ e,
                                            int64_t nc, double two_dx, int field_bc, int64_t j) {
  efield_node_g([phi](int64_t i) { return phi[i]; }, e, nc, two_dx, field_bc, j);
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

// ---- parallel Poisson: closed form + one prefix scan -------------------------
// The (1,-2,1) system with zero ends, -2 x_k + x_{k-1} + x_{k+1} = r_k for
// k in [0, n), has the Green's function form (telescoping the closed-form
// Thomas pivots d_k = -(k+2)/(k+1) through both sweeps)
//
//   x_k = -[ Z_k + (k+1) (S_tot - S_k) - (k+1) Z_tot / (n+1) ]
//   S_k = sum_{j<=k} r_j,   Z_k = sum_{j<=k} (j+1) r_j
//
// so the whole solve is ONE prefix scan of (S, Z) plus the totals.  The
// periodic variant (fields.py:179-190: mean-subtracted rhs, phi[0] = 0, then a
// shift to zero mean) is linear in the mean: r_j = a_j + scale*mean with
// a_j = -rho[j+1]*scale, the mean part has the closed form
// x_k = -(k+1)(n-k)/2 * scale*mean, and sum_k x_k needs one more tile sum,
// M = sum_j (j+1)(2n-j)/2 a_j (sum_k Z_k and sum_k (k+1) S_k regrouped):
//
//   sum_k x_k = -(M - Z_tot n/2) - scale*mean * n(n+1)(n+2)/12
//
// Plain fp64 tree sums: ~1e-14 max|phi| from a long-double elimination at
// 1e5 unknowns (noise, smooth and sheath-shaped rho), so within the bars the
// tests hold it to against the reference's serial solve (1e-12 max|phi| on
// its golden fields).  Tiles of 512 unknowns (256 threads x 2): each tile
// scans itself and publishes its aggregates; every consumer forms the same
// exclusive tile prefixes with the same tree.  A tile's last unknown takes
// the NEXT tile's prefix (not its own running sum) and its first unknown is
// prefix + (0 + term), exactly how the neighbours derive them as halo values
// (k = base-1, base+512): the fused kernel's E from its local phi equals E
// from the phi array, bit for bit.
constexpr int kMbThreads = 256;
constexpr int kMbPer = 2;
constexpr int kMbTile = kMbThreads * kMbPer;  // unknowns per tile
constexpr int kMbWarps = kMbThreads / 32;

// per-tile aggregates: S = sum r, Z = sum (k+1) r, M = sum (k+1)(2n-k)/2 r and
// R = sum rho over the tile's nodes (the periodic mean; M and R periodic only)
struct Agg {
  double s, z, m, r;
};
__device__ __forceinline__ Agg agg_zero() { return {0.0, 0.0, 0.0, 0.0}; }
__device__ __forceinline__ Agg agg_add(const Agg &a, const Agg &b, bool per) {
  if (!per) return {__dadd_rn(a.s, b.s), __dadd_rn(a.z, b.z), a.m, a.r};
  return {__dadd_rn(a.s, b.s), __dadd_rn(a.z, b.z), __dadd_rn(a.m, b.m), __dadd_rn(a.r, b.r)};
}
__device__ __forceinline__ Agg agg_shfl_up(const Agg &v, int d, bool per) {
  const unsigned f = 0xffffffffu;
  if (!per) return {__shfl_up_sync(f, v.s, d), __shfl_up_sync(f, v.z, d), v.m, v.r};
  return {__shfl_up_sync(f, v.s, d), __shfl_up_sync(f, v.z, d), __shfl_up_sync(f, v.m, d),
          __shfl_up_sync(f, v.r, d)};
}
// another CTA's aggregate: through L2 (never a stale L1 line)
__device__ __forceinline__ Agg agg_ldcg(const Agg *p, bool per) {
  const double *d = reinterpret_cast<const double *>(p);
  Agg a = {__ldcg(d), __ldcg(d + 1), 0.0, 0.0};
  if (per) {
    a.m = __ldcg(d + 2);
    a.r = __ldcg(d + 3);
  }
  return a;
}

// Exclusive scan over threads in index order (thread 0 gets +0.0) and the
// block total (warp totals summed in warp order): a fixed tree, so every CTA
// scanning the same values agrees bit for bit.
__device__ Agg block_excl(Agg v, Agg *sm, bool per, Agg &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Agg inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Agg o = agg_shfl_up(inc, d, per);
    if (lane >= d) inc = agg_add(o, inc, per);
  }
  Agg lex = agg_shfl_up(inc, 1, per);
  if (lane == 0) lex = agg_zero();
  if (lane == 31) sm[warp] = inc;
  __syncthreads();
  Agg wex = agg_zero(), tot = sm[0];
  for (int w = 0; w < warp; ++w) wex = agg_add(wex, sm[w], per);
#pragma unroll
  for (int w = 1; w < kMbWarps; ++w) tot = agg_add(tot, sm[w], per);
  __syncthreads();
  total = tot;
  return warp == 0 ? lex : agg_add(wex, lex, per);
}

struct ScanArgs {
  int64_t nc, n;  // n = nc - 1 unknowns: phi[1 .. nc-1]
  int G;          // tiles of kMbTile unknowns
  int field_bc;
  double scale, phi_left, phi_right;
  Agg *agg;  // [G] tile aggregates
  Agg *pre;  // [G + 1] exclusive tile prefixes (multi-kernel path)
};

// r_k without the periodic mean (fields.py:182-184, :193-197)
__device__ __forceinline__ double rhs_term(const ScanArgs &a, int64_t k, double rho_k1) {
  double r = __dmul_rn(-rho_k1, a.scale);
  if (a.field_bc != PB_FIELD_PERIODIC) {
    if (k == 0) r = __dsub_rn(r, a.phi_left);
    if (k == a.n - 1) r = __dsub_rn(r, a.phi_right);
  }
  return r;
}

// Tile t's local scan: thread i holds unknowns k = base + 2i + j; s[j] / z[j]
// run through its element j, ex is the exclusive scan of the thread totals,
// tot the tile's aggregates.  rs(j) = rho_s at node j.
struct TileLocal {
  Agg ex, tot;
  double s[kMbPer], z[kMbPer];
};
template <typename Rs>
__device__ void tile_local(const ScanArgs &a, int t, const Rs &rs, Agg *sm, TileLocal &L) {
  const bool per = a.field_bc == PB_FIELD_PERIODIC;
  const int64_t base = (int64_t)t * kMbTile;
  const int64_t kend = base + kMbTile < a.n ? base + kMbTile : a.n;
  const int64_t k0 = base + 2 * threadIdx.x;
  const double two_n = 2.0 * (double)a.n;
  Agg acc = agg_zero();
  if (per && t == 0 && threadIdx.x == 0) acc.r = rs(0);  // node 0 of the mean
#pragma unroll
  for (int j = 0; j < kMbPer; ++j) {
    const int64_t k = k0 + j;
    if (k < kend) {
      const double rho = rs(k + 1);
      const double r = rhs_term(a, k, rho);
      acc.s = __dadd_rn(acc.s, r);
      acc.z = __dadd_rn(acc.z, __dmul_rn((double)(k + 1), r));
      if (per) {
        const double w = __dmul_rn(0.5, __dmul_rn((double)(k + 1), __dsub_rn(two_n, (double)k)));
        acc.m = __dadd_rn(acc.m, __dmul_rn(w, r));
        acc.r = __dadd_rn(acc.r, rho);
      }
    }
    L.s[j] = acc.s;
    L.z[j] = acc.z;
  }
  L.ex = block_excl(acc, sm, per, L.tot);
}

// Exclusive tile prefixes: thread i sums tiles [i c, i c + c) in order, a
// block scan, and pre[q] is formed by the one thread min(q / c, 255) as its
// scan value plus its tiles before q, in order.  The fused cycle's CTAs (the
// q they need) and k_scan_prefixes (every q) run the same operations.
__device__ __forceinline__ int prefix_owner(int q, int c) {
  return q / c < kMbThreads ? q / c : kMbThreads - 1;
}
__device__ __forceinline__ Agg block_tile_excl(const Agg *agg, int G, int c, Agg *sm, bool per) {
  const int i0 = threadIdx.x * c;
  Agg loc = agg_zero(), tot;
  for (int q = 0; q < c; ++q)
    if (i0 + q < G) loc = agg_add(loc, agg_ldcg(&agg[i0 + q], per), per);
  return block_excl(loc, sm, per, tot);
}
__device__ __forceinline__ Agg owner_prefix(const Agg *agg, int q, int c, const Agg &ex, bool per) {
  Agg p = ex;
  for (int r = threadIdx.x * c; r < q; ++r) p = agg_add(p, agg_ldcg(&agg[r], per), per);
  return p;
}

// Constants every tile derives identically from the totals.
struct SolveConst {
  double zt_n1;  // Z_tot / (n+1)
  double sm;     // periodic: scale * mean
  double shift;  // periodic: mean of phi[0, nc) before the shift
};
__device__ __forceinline__ SolveConst solve_const(const ScanArgs &a, const Agg &tot) {
  SolveConst c;
  const double n = (double)a.n;
  c.zt_n1 = __ddiv_rn(tot.z, n + 1.0);
  c.sm = 0.0;
  c.shift = 0.0;
  if (a.field_bc == PB_FIELD_PERIODIC) {
    c.sm = __dmul_rn(__ddiv_rn(tot.r, (double)a.nc), a.scale);
    const double g1 = __ddiv_rn(__dmul_rn(__dmul_rn(0.5, __dmul_rn(n, n + 1.0)), n + 2.0), 6.0);
    const double gx = -__dsub_rn(tot.m, __dmul_rn(tot.z, __dmul_rn(0.5, n)));
    c.shift = __ddiv_rn(__dsub_rn(gx, __dmul_rn(c.sm, g1)), (double)a.nc);
  }
  return c;
}

// phi at unknown k from Z_k, S_k (periodic: shifted)
__device__ __forceinline__ double solve_phi(const ScanArgs &a, const SolveConst &c, const Agg &tot, int64_t k,
                                            double z, double s) {
  const double k1 = (double)(k + 1);
  double x = -__dadd_rn(z, __dmul_rn(__dsub_rn(__dsub_rn(tot.s, s), c.zt_n1), k1));
  if (a.field_bc == PB_FIELD_PERIODIC) {
    x = __dsub_rn(x, __dmul_rn(c.sm, __dmul_rn(0.5, __dmul_rn(k1, (double)(a.n - k)))));
    x = __dsub_rn(x, c.shift);
  }
  return x;
}
// phi[0] and phi[nc]
__device__ __forceinline__ double phi_wall0(const ScanArgs &a, const SolveConst &c) {
  return a.field_bc == PB_FIELD_PERIODIC ? -c.shift : a.phi_left;
}
__device__ __forceinline__ double phi_wallnc(const ScanArgs &a, const SolveConst &c) {
  return a.field_bc == PB_FIELD_PERIODIC ? -c.shift : a.phi_right;
}

// Tile t's unknowns -> px[i] = phi at node base + i, i in [0, kMbTile + 2):
// own nodes [base+1, kend+1), the halo nodes base and base+513 (or the wall /
// wrap node nc).  pre = {pre[t], pre[t+1], pre[min(t+2, G)], pre[G]}.
template <typename Rs>
__device__ void tile_solve(const ScanArgs &a, int t, const Rs &rs, const TileLocal &L, const Agg *pre,
                           const SolveConst &c, double *px) {
  const Agg &tot = pre[3];
  const int64_t base = (int64_t)t * kMbTile;
  const int64_t kend = base + kMbTile < a.n ? base + kMbTile : a.n;
  const int64_t k0 = base + 2 * threadIdx.x;
#pragma unroll
  for (int j = 0; j < kMbPer; ++j) {
    const int64_t k = k0 + j;
    if (k >= kend) break;
    double z, s;
    if (k == kend - 1) {  // the tile's last unknown: the next tile's prefix
      z = pre[1].z;
      s = pre[1].s;
    } else {
      z = __dadd_rn(pre[0].z, __dadd_rn(L.ex.z, L.z[j]));
      s = __dadd_rn(pre[0].s, __dadd_rn(L.ex.s, L.s[j]));
    }
    px[k - base + 1] = solve_phi(a, c, tot, k, z, s);
  }
  if (threadIdx.x == 0) {
    // left halo: node base = unknown base-1, the last of tile t-1
    px[0] = t == 0 ? phi_wall0(a, c) : solve_phi(a, c, tot, base - 1, pre[0].z, pre[0].s);
    // right halo: node base+513 = unknown base+512, the first of tile t+1
    const int64_t k = base + kMbTile;
    if (k < a.n) {
      double z, s;
      if (k == a.n - 1) {  // also that tile's last
        z = pre[2].z;
        s = pre[2].s;
      } else {  // that tile's thread 0: pre + (0 + term)
        const double rk = rhs_term(a, k, rs(k + 1));
        z = __dadd_rn(pre[1].z, __dadd_rn(0.0, __dmul_rn((double)(k + 1), rk)));
        s = __dadd_rn(pre[1].s, __dadd_rn(0.0, rk));
      }
      px[kMbTile + 1] = solve_phi(a, c, tot, k, z, s);
    } else {
      px[a.nc - base] = phi_wallnc(a, c);  // the last tile: node nc
    }
  }
  __syncthreads();
}

// phi at node i seen from tile t's window (+ the wall / wrap nodes)
struct PhiWin {
  const double *px;
  int64_t base, nc;
  double phi0, phinc, phi_last;  // phi[0], phi[nc], phi[nc-1] (periodic E[0])
  __device__ __forceinline__ double operator()(int64_t i) const {
    if (i == 0) return phi0;
    if (i == nc) return phinc;
    const int64_t o = i - base;
    if (o >= 0 && o < kMbTile + 2) return px[o];
    return phi_last;
  }
};

// ---- multi-kernel solve (pb_solve_poisson_scan; large grids) -----------------
__global__ void __launch_bounds__(kMbThreads) k_scan_aggregate(const ScanArgs a, const double *__restrict__ rho_s) {
  pdl_enter();
  __shared__ Agg sm[kMbWarps];
  TileLocal L;
  tile_local(a, blockIdx.x, [rho_s](int64_t j) { return rho_s[j]; }, sm, L);
  if (threadIdx.x == 0) a.agg[blockIdx.x] = L.tot;
}

// one CTA: pre[0 .. G] (thread min(q / c, 255) forms pre[q], as in the fused cycle)
__global__ void __launch_bounds__(kMbThreads) k_scan_prefixes(const ScanArgs a) {
  pdl_enter();
  __shared__ Agg sm[kMbWarps];
  const bool per = a.field_bc == PB_FIELD_PERIODIC;
  const int G = a.G, c = (G + kMbThreads - 1) / kMbThreads, i0 = threadIdx.x * c;
  Agg p = block_tile_excl(a.agg, G, c, sm, per);
  for (int q = i0; q <= i0 + c && q <= G; ++q) {
    if (prefix_owner(q, c) == (int)threadIdx.x) a.pre[q] = p;
    if (q < G && q < i0 + c) p = agg_add(p, agg_ldcg(&a.agg[q], per), per);
  }
}

__global__ void __launch_bounds__(kMbThreads) k_scan_solve(const ScanArgs a, const double *__restrict__ rho_s,
                                                           double *__restrict__ phi) {
  pdl_enter();
  __shared__ Agg sm[kMbWarps];
  __shared__ double px[kMbTile + 2];
  const int t = blockIdx.x;
  const auto rs = [rho_s](int64_t j) { return rho_s[j]; };
  TileLocal L;
  tile_local(a, t, rs, sm, L);
  Agg pre[4];
  pre[0] = a.pre[t];
  pre[1] = a.pre[t + 1];
  pre[2] = a.pre[t + 2 <= a.G ? t + 2 : a.G];
  pre[3] = a.pre[a.G];
  const SolveConst c = solve_const(a, pre[3]);
  tile_solve(a, t, rs, L, pre, c, px);
  const int64_t base = (int64_t)t * kMbTile;
  const int64_t kend = base + kMbTile < a.n ? base + kMbTile : a.n;
  for (int64_t i = threadIdx.x; i < kend - base; i += kMbThreads) phi[base + 1 + i] = px[1 + i];
  if (threadIdx.x == 0) {
    if (t == 0) phi[0] = phi_wall0(a, c);
    if (t == a.G - 1) phi[a.nc] = phi_wallnc(a, c);
  }
}

// ---- the field step: density epilogue + smoothing + solve + E ---------------
// k_field_fused runs the whole replicated field step in ONE launch: CTA t
// forms rho and `passes` 1-2-1 smoothing passes on a halo'd shared-memory
// window of the bins (the cells its tile's nodes read, so no neighbour
// exchange), writes its tile aggregates and arrives on a counter, waits for
// every tile's arrival (the only grid-wide wait), forms the tile prefixes
// itself, solves its tile and writes phi and E, then zeroes the bins it was
// handed.  The arrival and exit counters return to zero at the end of every
// launch: the scratch is zeroed once, and the launch is graph-replayable.
// Every CTA must be
// co-resident: pb_field_cycle checks the occupancy and otherwise runs the
// same code as separate kernels (bitwise the same results).
constexpr int kFfMaxPasses = 4;
constexpr int kFfWin = kMbTile + 2 + 2 * kFfMaxPasses;  // core nodes [base - P, base + 514 + P)
constexpr int kFfCellIters = (kFfWin + 1 + kMbThreads - 1) / kMbThreads;

struct FieldArgs {
  ScanArgs sa;
  const uint64_t *bins;
  CoefArgs ca;
  int ndep, passes;
  double *left, *right, *rho, *rho_s, *phi, *e;
  uint64_t *sync;   // [0] arrivals, [1] exits (both back to 0 after every launch)
                    // (+ the PB_FF_TRACE words)
  uint64_t *clr_a, *clr_b;
  int64_t nwords;
  double two_dx;
  pb_status *st;
  // absorbing walls: the previous step's holes are filled by cpt.nsp extra
  // blocks of the same launch (blockIdx >= G), independent of the field work
  CompactArgs cpt;
};

struct Window {
  double l[kFfWin + 1], r[kFfWin + 1];  // weighted partials of cell base - P - 1 + p
  double c[2][kFfWin];                  // rho core, then the smoothing passes
};

// rho (+ smoothing) of tile t's window; writes the owned left / right / rho /
// rho_s; returns sw with sw[i] = rho_s at node base + i, i in [0, 514).
__device__ __forceinline__ const double *window_rho(const FieldArgs &a, const ScanArgs &sa, int t, Window &w) {
  const int64_t nc = sa.nc;
  const int P = a.passes;
  const bool periodic = sa.field_bc == PB_FIELD_PERIODIC;
  const int64_t base = (int64_t)t * kMbTile;
  const int64_t kend = base + kMbTile < sa.n ? base + kMbTile : sa.n;
  const int W = kMbTile + 2 + 2 * P;
  const bool wrap = nc <= W;  // a window wrapping more than once (tiny grids): true modulo
  // the tile owns cells (and nodes) [base+1, kend+1), tile 0 also cell 0:
  // each cell's overflow is flagged once
  int64_t cell[kFfCellIters];
  bool on[kFfCellIters], mine[kFfCellIters];
  double lacc[kFfCellIters], racc[kFfCellIters];
#pragma unroll
  for (int i = 0; i < kFfCellIters; ++i) {
    const int p = threadIdx.x + i * kMbThreads;
    const int64_t g = base - P - 1 + p;
    on[i] = p <= W;
    mine[i] = on[i] && ((g >= base + 1 && g < kend + 1) || (t == 0 && g == 0));
    cell[i] = wrap ? floor_mod(g, nc) : (g < 0 ? g + nc : (g >= nc ? g - nc : g));
    lacc[i] = racc[i] = 0.0;
  }
  uint64_t cmax = 0;
  for (int s = 0; s < a.ndep; ++s) {  // species order (fields.py:64-77); loads batched per species
    const uint64_t *B = a.bins + (size_t)s * 2 * nc;
    uint64_t R[kFfCellIters], C[kFfCellIters];
#pragma unroll
    for (int i = 0; i < kFfCellIters; ++i) {
      R[i] = on[i] ? B[cell[i]] : 0;
      C[i] = on[i] ? B[nc + cell[i]] : 0;
    }
    const double cf = a.ca.c[s];
#pragma unroll
    for (int i = 0; i < kFfCellIters; ++i) {
      if (mine[i] && C[i] > cmax) cmax = C[i];
      const uint64_t L = (C[i] << kFracBits) - R[i];
      lacc[i] = __dadd_rn(lacc[i], __dmul_rn(cf, __dmul_rn(__ull2double_rn(L), kFracInv)));
      racc[i] = __dadd_rn(racc[i], __dmul_rn(cf, __dmul_rn(__ull2double_rn(R[i]), kFracInv)));
    }
  }
  if (cmax >= kMaxCellCount) flag_overflow(a.st, cmax);
#pragma unroll
  for (int i = 0; i < kFfCellIters; ++i) {
    if (on[i]) {
      const int p = threadIdx.x + i * kMbThreads;
      w.l[p] = lacc[i];
      w.r[p] = racc[i];
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < W; q += kMbThreads) {  // rho core: rs_core of fields.py:85-91, :115-117
    const int64_t g = base - P + q;
    const int64_t core = wrap ? floor_mod(g, nc) : (g < 0 ? g + nc : (g >= nc ? g - nc : g));
    w.c[0][q] = (!periodic && core == 0) ? __dmul_rn(w.l[q + 1], 2.0) : __dadd_rn(w.r[q], w.l[q + 1]);
  }
  __syncthreads();
  int cur = 0;
  for (int pass = 1; pass <= P; ++pass) {  // the valid window shrinks by a node a side (fields.py:131)
    const double *in = w.c[cur];
    double *out = w.c[cur ^ 1];
    for (int q = pass + threadIdx.x; q < W - pass; q += kMbThreads)
      out[q] = __dadd_rn(__dadd_rn(__dmul_rn(0.25, in[q - 1]), __dmul_rn(0.5, in[q])),
                         __dmul_rn(0.25, in[q + 1]));
    cur ^= 1;
    __syncthreads();
  }
  const double *sw = w.c[cur] + P;
  const double *lw = w.l + P + 1, *rw = w.r + P + 1;  // partials of cell base + i, i in [-1, 514)
  for (int64_t i = 1 + threadIdx.x; i < kend - base + 1; i += kMbThreads) {
    const int64_t j = base + i;  // an interior node / cell
    if (a.left) a.left[j] = lw[i];
    if (a.right) a.right[j] = rw[i];
    a.rho[j] = __dadd_rn(rw[i - 1], lw[i]);
    a.rho_s[j] = sw[i];
  }
  if (threadIdx.x == 0) {
    if (t == 0) {
      if (a.left) a.left[0] = lw[0];
      if (a.right) a.right[0] = rw[0];
      a.rho[0] = periodic ? __dadd_rn(rw[-1], lw[0]) : __dmul_rn(lw[0], 2.0);
      a.rho_s[0] = sw[0];
    }
    if (kend == sa.n) {  // node nc == core node 0
      const int64_t i = nc - base;
      a.rho[nc] = periodic ? __dadd_rn(rw[i - 1], lw[i]) : __dmul_rn(rw[i - 1], 2.0);
      a.rho_s[nc] = sw[i];
    }
  }
  return sw;
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// PB_FF_TRACE builds record %globaltimer at the phase boundaries per CTA
// (scripts/field_fused_trace.py), nothing otherwise
#ifdef PB_FF_TRACE
#define FF_MARK(k)                                                   \
  do {                                                               \
    if (threadIdx.x == 0) {                                          \
      uint64_t ns, ck;                                               \
      uint32_t sm;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));         \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(ck));             \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));                \
      a.sync[2 + (size_t)blockIdx.x * 16 + (k)] = ns;                \
      a.sync[2 + (size_t)blockIdx.x * 16 + 8 + (k)] =                \
          (k) == 0 ? (uint64_t)sm : ck;                              \
    }                                                                \
  } while (0)
__device__ unsigned long long g_flog[512][2];  // per launch: CTA 0 start (past the wait), CTA 0 end
__device__ unsigned long long g_flog_n;
#define FF_LOG(k)                                                              \
  do {                                                                         \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                                 \
      uint64_t ns;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));                   \
      if ((k) == 0) {                                                          \
        g_flog[g_flog_n % 512][0] = ns;                                        \
      } else {                                                                 \
        g_flog[g_flog_n % 512][1] = ns;                                        \
        g_flog_n++;                                                            \
      }                                                                        \
    }                                                                          \
  } while (0)
#else
#define FF_MARK(k) \
  do {             \
  } while (0)
#define FF_LOG(k) \
  do {            \
  } while (0)
#endif

#ifndef PB_FF_LATE_TRIGGER
#define PB_FF_LATE_TRIGGER 1
#endif
// PER: the boundary condition as a compile-time constant (one instantiation
// each): the kernel runs once per step, cold in the instruction cache after
// the mover, so the code it does not need stays out of its path.
template <bool PER>
__global__ void __launch_bounds__(kMbThreads) k_field_fused(const __grid_constant__ FieldArgs a) {
#if PB_FF_LATE_TRIGGER
  pdl_wait();  // the dependent (the mover) is released after the solve, below
#else
  pdl_enter();
#endif
  __shared__ union {
    Window win;
    CompactSmem<kMbThreads> cpt;
  } su;
  Window &win = su.win;
  __shared__ Agg sm_agg[kMbWarps];
  __shared__ Agg s_pre[4];
  __shared__ double px[kMbTile + 2];
  ScanArgs sa = a.sa;
  sa.field_bc = PER ? PB_FIELD_PERIODIC : PB_FIELD_DIRICHLET;  // folded at compile time
  const int t = blockIdx.x, G = sa.G;
  if (t >= G) {  // a compaction block: the previous step's holes of one species
    compact_species<kMbThreads>(a.cpt, t - G, su.cpt);
    __syncthreads();
    if (threadIdx.x == 0 &&
        atomicAdd((unsigned long long *)&a.sync[1], 1ull) == (unsigned long long)(G + a.cpt.nsp - 1)) {
      a.sync[0] = 0;
      a.sync[1] = 0;
    }
    return;
  }
  FF_MARK(0);
  FF_LOG(0);
  const int64_t nc = sa.nc, base = (int64_t)t * kMbTile;
  const int64_t kend = base + kMbTile < sa.n ? base + kMbTile : sa.n;
  const bool periodic = sa.field_bc == PB_FIELD_PERIODIC;

  const double *sw = window_rho(a, sa, t, win);  // (synchronises the CTA)
  FF_MARK(1);
  auto rs = [sw, base](int64_t j) { return sw[j - base]; };
  TileLocal L;
  tile_local(sa, t, rs, sm_agg, L);  // the tile's own scan, before any wait
  FF_MARK(2);
  // the one grid-wide wait: arrive (the barrier inside tile_local has ordered
  // the CTA's bin reads and writes before thread 0's release; release is
  // cumulative), then poll the arrival count with relaxed loads and take the
  // acquire once it is complete
  if (threadIdx.x == 0) {
    sa.agg[t] = L.tot;
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&a.sync[0]) : "memory");
    while (ld_relaxed_u64(&a.sync[0]) < (uint64_t)G) {
    }
    (void)ld_acquire_u64(&a.sync[0]);
  }
  __syncthreads();
  FF_MARK(3);
  // every CTA has read its bins (it arrived after reading them), so the bins
  // are cleared here: the stores drain while the prefix, solve and E phases
  // wait on L2 round trips, instead of after E on the way to the mover
  if (a.nwords > 0) {
    for (int64_t w = (int64_t)t * kMbThreads + threadIdx.x; w < a.nwords; w += (int64_t)G * kMbThreads) {
      if (a.clr_a) a.clr_a[w] = 0;
      if (a.clr_b) a.clr_b[w] = 0;
    }
  }

  Agg pre[4];
  {  // the tile prefixes this tile needs, formed by their owner threads
    const int c = (G + kMbThreads - 1) / kMbThreads;
    const Agg ex = block_tile_excl(sa.agg, G, c, sm_agg, periodic);
    const int want[4] = {t, t + 1, t + 2 <= G ? t + 2 : G, G};
#pragma unroll
    for (int w = 0; w < 4; ++w)
      if (prefix_owner(want[w], c) == (int)threadIdx.x) s_pre[w] = owner_prefix(sa.agg, want[w], c, ex, periodic);
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 4; ++w) pre[w] = s_pre[w];
  }
  const SolveConst c = solve_const(sa, pre[3]);
  FF_MARK(4);
  tile_solve(sa, t, rs, L, pre, c, px);
  FF_MARK(5);

  PhiWin pw{px, base, nc, phi_wall0(sa, c), phi_wallnc(sa, c), 0.0};
  if (t == 0 && periodic && G > 1)  // E[0] wraps to node nc-1: the last unknown
    pw.phi_last = solve_phi(sa, c, pre[3], sa.n - 1, pre[3].z, pre[3].s);
  for (int64_t i = 1 + threadIdx.x; i < kend - base + 1; i += kMbThreads) {
    const int64_t j = base + i;
    a.phi[j] = px[i];
    efield_node_g(pw, a.e, nc, a.two_dx, sa.field_bc, j);
  }
  if (threadIdx.x == 0) {
    if (t == 0) {
      a.phi[0] = pw.phi0;
      efield_node_g(pw, a.e, nc, a.two_dx, sa.field_bc, 0);
      if (periodic) {
        a.phi[nc] = pw.phinc;
        efield_node_g(pw, a.e, nc, a.two_dx, sa.field_bc, nc);
      }
    }
    if (t == G - 1 && !periodic) {
      a.phi[nc] = pw.phinc;
      efield_node_g(pw, a.e, nc, a.two_dx, sa.field_bc, nc);
    }
  }
  FF_MARK(6);
#if PB_FF_LATE_TRIGGER
  pdl_trigger();
#endif

  // the last CTA out (every CTA is past its wait) re-arms the counters
  __syncthreads();
  FF_MARK(7);
  FF_LOG(7);
  if (threadIdx.x == 0 &&
      atomicAdd((unsigned long long *)&a.sync[1], 1ull) == (unsigned long long)(G + a.cpt.nsp - 1)) {
    a.sync[0] = 0;
    a.sync[1] = 0;
  }
}

// The same phases as separate kernels (grids too large to be co-resident):
// window + aggregates here, then k_scan_prefixes, k_scan_solve and E.
__global__ void __launch_bounds__(kMbThreads) k_field_window(const __grid_constant__ FieldArgs a) {
  pdl_enter();
  __shared__ Window win;
  __shared__ Agg sm_agg[kMbWarps];
  const int t = blockIdx.x;
  const int64_t base = (int64_t)t * kMbTile;
  const double *sw = window_rho(a, a.sa, t, win);
  TileLocal L;
  tile_local(a.sa, t, [sw, base](int64_t j) { return sw[j - base]; }, sm_agg, L);
  if (threadIdx.x == 0) a.sa.agg[t] = L.tot;
}

// scratch: [exact solve rhs / diag / y, or the smoothing ping-pong: 3 (nc+1)
// doubles] [tile aggregates G] [tile prefixes G+1] [arrivals, exits]
// (+ PB_FF_TRACE words)
struct FieldScratch {
  size_t agg_off, pre_off, flag_off, bytes;
  int G;
};
static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }
static FieldScratch field_scratch_layout(int64_t nc) {
  FieldScratch f;
  f.G = (int)((nc - 1 + kMbTile - 1) / kMbTile);
  if (f.G < 1) f.G = 1;
  f.agg_off = align256(3 * (size_t)(nc + 1) * sizeof(double));
  f.pre_off = f.agg_off + align256((size_t)f.G * sizeof(Agg));
  f.flag_off = f.pre_off + align256((size_t)(f.G + 1) * sizeof(Agg));
  f.bytes = f.flag_off + 2 * sizeof(uint64_t);
#ifdef PB_FF_TRACE
  f.bytes += 16 * (size_t)f.G * sizeof(uint64_t);
#endif
  return f;
}

// Placement of k_field_fused: its blocks are latency chains, so they should
// sit one (or as few as possible) per SM -- launched early behind the mover
// (PDL), they would otherwise pile up on the first SMs the mover frees (up to
// four per SM measured, the field step 9.4 -> 11.9 us).  Dynamic shared
// memory pads each block so at most k = ceil(grid / SMs) fit on an SM.
// Returns the padding (bytes) for `grid` blocks, or -1 when the grid cannot
// be co-resident at all.
static int field_fused_pad(int grid, bool periodic) {
  static int sms = -1, static_smem[2] = {0, 0}, per_sm_smem = 0, max_optin = 0;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    for (int p = 0; p < 2; ++p) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, p ? (const void *)k_field_fused<true> : (const void *)k_field_fused<false>);
      static_smem[p] = (int)fa.sharedSizeBytes;
      cudaFuncSetAttribute(p ? (const void *)k_field_fused<true> : (const void *)k_field_fused<false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin - (int)fa.sharedSizeBytes);
    }
  }
  const int k = (grid + sms - 1) / sms;  // blocks per SM wanted
  const int reserve = 1024;              // per-block system shared memory
  // the per-block footprint must exceed per_sm / (k + 1)
  int pad = per_sm_smem / (k + 1) + 1 - reserve - static_smem[periodic ? 1 : 0];
  if (pad < 0) pad = 0;
  if (pad > max_optin - static_smem[periodic ? 1 : 0]) pad = max_optin - static_smem[periodic ? 1 : 0];
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per, periodic ? k_field_fused<true> : k_field_fused<false>, kMbThreads, pad);
  return (int64_t)per * sms >= grid ? pad : -1;
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

}  // namespace pb

extern "C" size_t pb_field_scratch_bytes(int64_t nc) {
  // smoothing ping-pong, tile aggregates / prefixes of the scan solve, and the
  // fused cycle's flag words (zeroed once by the caller)
  return pb::field_scratch_layout(nc).bytes;
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

// closed-form scan solve as three kernels: tile aggregates, the tile
// prefixes (one CTA), the tile solves
static int scan_solve(const double *rho_s, double *phi, const pb::ScanArgs &sa, cudaStream_t st,
                      bool aggregates) {
  const dim3 tb(pb::kMbThreads);
  cudaError_t e = cudaSuccess;
  if (aggregates) e = pb::launch_pdl(pb::k_scan_aggregate, dim3(sa.G), tb, 0, st, sa, rho_s);
  if (e == cudaSuccess) e = pb::launch_pdl(pb::k_scan_prefixes, dim3(1), tb, 0, st, sa);
  if (e == cudaSuccess) e = pb::launch_pdl(pb::k_scan_solve, dim3(sa.G), tb, 0, st, sa, rho_s, phi);
  if (e != cudaSuccess) return pb::cuda_status(e, "poisson scan");
  PB_CHECK_LAUNCH("poisson scan");
  return PB_OK;
}

static pb::ScanArgs host_scan_args(int64_t nc, double dx, double eps0, int field_bc, double phi_left,
                                   double phi_right, void *scratch) {
  const pb::FieldScratch fl = pb::field_scratch_layout(nc);
  pb::ScanArgs sa;
  sa.nc = nc;
  sa.n = nc - 1;
  sa.G = fl.G;
  sa.field_bc = field_bc;
  sa.scale = (dx * dx) / eps0;  // grid.dx_m * grid.dx_m / eps0
  sa.phi_left = phi_left;
  sa.phi_right = phi_right;
  sa.agg = (pb::Agg *)((char *)scratch + fl.agg_off);
  sa.pre = (pb::Agg *)((char *)scratch + fl.pre_off);
  return sa;
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
  const pb::ScanArgs sa = host_scan_args(nc, dx, eps0, field_bc, phi_left, phi_right, scratch);
  return scan_solve(rho, phi, sa, (cudaStream_t)stream, true);
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
                              const pb_species *compact_sp, int compact_nsp, void *compact_scratch,
                              size_t compact_scratch_bytes, void *stream) {
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
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nw = (clr_a || clr_b) ? nwords : 0;
  pb::CompactArgs cpt;
  memset(&cpt, 0, sizeof(cpt));
  if (compact_nsp > 0) {
    if (!status) {
      pb::set_error("pb_field_cycle: compaction needs the status");
      return PB_ERR_INVALID;
    }
    const int rc = pb::compact_args(compact_sp, compact_nsp, status, compact_scratch, compact_scratch_bytes, cpt);
    if (rc) return rc;
  }
  if (passes <= pb::kFfMaxPasses) {
    const pb::FieldScratch fl = pb::field_scratch_layout(nc);
    pb::FieldArgs a;
    memset(&a, 0, sizeof(a));
    a.sa = host_scan_args(nc, dx, eps0, field_bc, phi_left, phi_right, scratch);
    a.bins = bins;
    for (int s = 0; s < ndep; ++s) a.ca.c[s] = coef[s];
    a.ndep = ndep;
    a.passes = passes;
    a.left = left;
    a.right = right;
    a.rho = rho;
    a.rho_s = rho_s;
    a.phi = phi;
    a.e = e;
    a.sync = (uint64_t *)((char *)scratch + fl.flag_off);
    a.clr_a = clr_a;
    a.clr_b = clr_b;
    a.nwords = nw;
    a.two_dx = 2.0 * dx;
    a.st = status;
    a.cpt = cpt;
    const int pad = pb::field_fused_pad(fl.G + cpt.nsp, field_bc == PB_FIELD_PERIODIC);
    if (pad >= 0) {  // one launch, every block co-resident, spread over the SMs
      cudaError_t err =
          pb::launch_pdl(field_bc == PB_FIELD_PERIODIC ? pb::k_field_fused<true> : pb::k_field_fused<false>,
                         dim3(fl.G + cpt.nsp), dim3(pb::kMbThreads), (size_t)pad, st, a);
      if (err != cudaSuccess) return pb::cuda_status(err, "k_field_fused");
      return PB_OK;
    }
    a.cpt.nsp = 0;  // the kernels below take no compaction blocks
    // too many tiles to be co-resident: the same phases as kernels
    cudaError_t err = pb::launch_pdl(pb::k_field_window, dim3(fl.G), dim3(pb::kMbThreads), 0, st, a);
    if (err != cudaSuccess) return pb::cuda_status(err, "k_field_window");
    int rc = scan_solve(rho_s, phi, a.sa, st, false);
    if (!rc) rc = pb_compute_efield_clear(phi, e, nc, dx, field_bc, clr_a, clr_b, nw, stream);
    if (!rc && cpt.nsp > 0)
      rc = pb_compact(compact_sp, compact_nsp, status, compact_scratch, compact_scratch_bytes, stream);
    return rc;
  }
  int rc = pb_rho_epilogue(bins, coef, ndep, nc, field_bc, left, right, rho, status, stream);
  if (!rc) rc = pb_smooth_density(rho, rho_s, nc, passes, scratch, stream);
  if (!rc) rc = pb_solve_poisson_scan(rho_s, phi, nc, dx, eps0, field_bc, phi_left, phi_right, scratch, stream);
  if (!rc) rc = pb_compute_efield_clear(phi, e, nc, dx, field_bc, clr_a, clr_b, nw, stream);
  if (!rc && cpt.nsp > 0)
    rc = pb_compact(compact_sp, compact_nsp, status, compact_scratch, compact_scratch_bytes, stream);
  return rc;
}

#ifdef PB_FF_TRACE
// debug: the field-step launch log (CTA 0 past its wait, CTA 0 end) and its count
extern "C" int pb_debug_field_log(unsigned long long *out, unsigned long long *count) {
  if (cudaMemcpyFromSymbol(out, pb::g_flog, sizeof(pb::g_flog)) != cudaSuccess) return PB_ERR_CUDA;
  return cudaMemcpyFromSymbol(count, pb::g_flog_n, sizeof(unsigned long long)) == cudaSuccess ? PB_OK
                                                                                            : PB_ERR_CUDA;
}
#endif
