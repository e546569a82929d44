/*
 * picmc_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA kernels:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, never the product path.  Build: oracle/Makefile (gcc -O3
 * -ffp-contract=off, the reference's own flags, pkg/setup.py:12).
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * golden vectors produced by the reference itself (tests/golden/, made by
 * tests/golden/make_golden.py from /root/reference) and, when present,
 * against the reference's compiled kernels built from its own sources into
 * oracle/_ref/ (oracle/Makefile `ref` target).
 *
 * Two layouts are restated:
 *   packed -- the reference CellSortedStore segments (offs/counts), for the
 *             kernel-signature shims;
 *   flat   -- one record per particle with its cell index, which is the
 *             device engine layout; shown equivalent to the reference's
 *             fused_move + resort in tests.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ---- packed layout: the three reference kernels ------------------------- */

/* fused_move, pkg/src/picmc/backends/_kernels.pyx:60-102 */
void or_fused_move(const double *accel, double *x, double *vx, const double *vy,
                   double *yp, const int64_t *offs, const int64_t *counts,
                   int64_t nc, double fnstep) {
  for (int64_t j = 0; j < nc; ++j) {
    const int64_t b = offs[j];
    double aj = 0.0, daj = 0.0;
    if (accel) {
      aj = accel[j];
      daj = accel[j + 1] - aj;
    }
    for (int64_t i = 0; i < counts[j]; ++i) {
      double v = vx[b + i];
      if (accel) {
        const double atemp = aj + x[b + i] * daj;
        v = v + atemp;
        vx[b + i] = v;
      }
      x[b + i] = x[b + i] + fnstep * v;
    }
  }
  if (yp)
    for (int64_t j = 0; j < nc; ++j)
      for (int64_t i = 0; i < counts[j]; ++i)
        yp[offs[j] + i] = yp[offs[j] + i] + fnstep * vy[offs[j] + i];
}

/* deposit_partials, _kernels.pyx:14-34 (sequential slot order per cell) */
void or_deposit_partials(const double *x, const int64_t *offs,
                         const int64_t *counts, int64_t nc, double *left,
                         double *right) {
  for (int64_t j = 0; j < nc; ++j) {
    double sl = 0.0, sr = 0.0;
    for (int64_t i = 0; i < counts[j]; ++i) {
      const double xv = x[offs[j] + i];
      sl = sl + (1.0 - xv);
      sr = sr + xv;
    }
    left[j] = sl;
    right[j] = sr;
  }
}

/* gather, _kernels.pyx:37-57 */
void or_gather(const double *nodes, const double *x, const int64_t *offs,
               const int64_t *counts, int64_t nc, double *out) {
  int64_t k = 0;
  for (int64_t j = 0; j < nc; ++j) {
    const double aj = nodes[j], daj = nodes[j + 1] - nodes[j];
    for (int64_t i = 0; i < counts[j]; ++i) out[k++] = aj + x[offs[j] + i] * daj;
  }
}

/* fused_move_aos, _kernels.pyx:128-152 (fused_move_table is nc = 1) */
void or_fused_move_aos(double *tab, int64_t ncols, const int64_t *starts,
                       const int64_t *counts, int64_t nc, const double *accel,
                       double fnstep, int has_yp) {
  for (int64_t j = 0; j < nc; ++j) {
    double aj = 0.0, daj = 0.0;
    if (accel) {
      aj = accel[j];
      daj = accel[j + 1] - aj;
    }
    for (int64_t i = starts[j]; i < starts[j] + counts[j]; ++i) {
      double *r = tab + i * ncols;
      double v = r[1];
      if (accel) {
        const double atemp = aj + r[0] * daj;
        v = r[1] + atemp;
        r[1] = v;
      }
      r[0] = r[0] + fnstep * v;
      if (has_yp) r[4] = r[4] + fnstep * r[2];
    }
  }
}

/* ---- flat layout: one mover step ----------------------------------------- */

enum { OR_DRIFT = 1, OR_KICK = 2, OR_BORIS = 3 };
enum { OR_PERIODIC = 0, OR_ABSORBING = 1 };

/* Boris extension (config 4; no reference behaviour -- restated here and in
 * DESIGN.md): half kick with the gathered acceleration, rotation
 * v' = v- + v- x t, v+ = v- + v' x s, half kick, then the reference drift. */
static void boris(double *vx, double *vy, double *vz, double atemp,
                  const double *t, const double *s) {
  const double h = 0.5 * atemp;
  const double mx = *vx + h, my = *vy, mz = *vz;
  const double px = mx + (my * t[2] - mz * t[1]);
  const double py = my + (mz * t[0] - mx * t[2]);
  const double pz = mz + (mx * t[1] - my * t[0]);
  const double qx = mx + (py * s[2] - pz * s[1]);
  const double qy = my + (pz * s[0] - px * s[2]);
  const double qz = mz + (px * s[1] - py * s[0]);
  *vx = qx + h;
  *vy = qy;
  *vz = qz;
}

/* Spatially varying B (pb_species.b_nodes, include/picmc_b200.h): nodes
 * hold (Bx, By, Bz, pad) in tesla; t = the one-sided linear gather of f*B
 * (f = q dt / (2 m)) in the accel_nodes form (pkg/src/picmc/mover.py:221,
 * _kernels.pyx:83-86), s = t * (2 / (1 + |t|^2)) in the host's
 * boris_coefficients op order.  Each operation rounds separately. */
static void boris_t_gather(const double *bnodes, double f, int32_t c, double x, double *t,
                           double *s) {
  const double *b0 = bnodes + 4 * (int64_t)c, *b1 = b0 + 4;
  for (int k = 0; k < 3; ++k) {
    const double t0 = f * b0[k];
    const double t1 = f * b1[k];
    t[k] = t0 + x * (t1 - t0);
  }
  const double t2 = t[0] * t[0] + t[1] * t[1] + t[2] * t[2];
  const double g = 2.0 / (1.0 + t2);
  for (int k = 0; k < 3; ++k) s[k] = t[k] * g;
}

static int64_t pymod(int64_t a, int64_t m) {
  int64_t r = a % m;
  return r < 0 ? r + m : r;
}

/*
 * Push every particle (arithmetic of _kernels.pyx:81-101, aj = coef*E[j] as
 * accel_nodes_for_species, pkg/src/picmc/mover.py:221), then the cell
 * transfer of resort_collect (pkg/src/picmc/mover.py:136-163):
 *   delta = floor(x); if delta != 0: CFL if |delta| >= nc;
 *   dest = (cell + delta) mod nc; x -= delta; if x >= 1: x -= 1, dest += 1.
 * Absorbing walls (config 3 extension): a mover whose unwrapped dest leaves
 * [0, nc) is removed (removed[i] = 1 left / 2 right) and not wrapped.
 * Returns the number of movers; *cfl_index = first violator or -1.  As in
 * the reference the CFL check precedes every transfer of the species, so on
 * a violation no particle is transferred.
 */
int64_t or_step_flat(int kind, int bc, double fnstep, double kick_coef,
                     const double *bt, const double *bs, const double *e,
                     int64_t nc, int64_t n, double *x, double *vx, double *vy,
                     double *vz, double *yp, int32_t *cell, uint8_t *removed,
                     int64_t *cfl_index, const double *bnodes, double bf) {
  for (int64_t i = 0; i < n; ++i) {
    const int32_t c = cell[i];
    if (kind == OR_KICK || kind == OR_BORIS) {
      const double aj = kick_coef * e[c];
      const double aj1 = kick_coef * e[c + 1];
      const double atemp = aj + x[i] * (aj1 - aj);
      if (kind == OR_KICK) {
        const double v = vx[i] + atemp;
        vx[i] = v;
      } else {
        double tg[3], sg[3];
        if (bnodes) boris_t_gather(bnodes, bf, c, x[i], tg, sg);
        boris(&vx[i], &vy[i], &vz[i], atemp, bnodes ? tg : bt, bnodes ? sg : bs);
      }
    }
    if (kind != 0) x[i] = x[i] + fnstep * vx[i];
    if (kind != 0 && yp) yp[i] = yp[i] + fnstep * vy[i];
  }
  *cfl_index = -1;
  for (int64_t i = 0; i < n; ++i) {
    const double d = floor(x[i]);
    if (d != 0.0 && fabs(d) >= (double)nc) {
      *cfl_index = i;
      return -1;
    }
  }
  int64_t moved = 0;
  for (int64_t i = 0; i < n; ++i) {
    removed[i] = 0;
    const double d = floor(x[i]);
    if (d == 0.0) continue;
    ++moved;
    int64_t dest = (int64_t)cell[i] + (int64_t)d;
    double nx = x[i] - d;
    if (nx >= 1.0) {
      nx -= 1.0;
      dest += 1;
    }
    x[i] = nx;
    if (bc == OR_PERIODIC) {
      cell[i] = (int32_t)pymod(dest, nc);
    } else if (dest < 0) {
      removed[i] = 1;
    } else if (dest >= nc) {
      removed[i] = 2;
    } else {
      cell[i] = (int32_t)dest;
    }
  }
  return moved;
}

/* Sequential fp64 deposit in array order per cell (the reference's
 * accumulation, _kernels.pyx:24-33, when array order is slot order). */
void or_deposit_seq(const double *x, const int32_t *cell,
                    const uint8_t *removed, int64_t n, int64_t nc,
                    double *left, double *right) {
  for (int64_t j = 0; j < nc; ++j) left[j] = right[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (removed && removed[i]) continue;
    left[cell[i]] = left[cell[i]] + (1.0 - x[i]);
    right[cell[i]] = right[cell[i]] + x[i];
  }
}

/* The device's fixed-point deposit: R += round(x * 2^48), C += 1. */
void or_deposit_fixed(const double *x, const int32_t *cell,
                      const uint8_t *removed, int64_t n, int64_t nc,
                      uint64_t *R, uint64_t *C) {
  for (int64_t i = 0; i < n; ++i) {
    if (removed && removed[i]) continue;
    R[cell[i]] += (uint64_t)llrint(x[i] * 281474976710656.0);
    C[cell[i]] += 1;
  }
}

/* Weighted partials (pkg/src/picmc/fields.py:64-77) from raw per-species
 * L/R, then stitch (fields.py:81-92, :115-117).  raw is [nsp][2][nc]. */
void or_rho(const double *raw, const double *coef, int nsp, int64_t nc,
            int periodic, double *left, double *right, double *rho) {
  for (int64_t j = 0; j < nc; ++j) {
    double l = 0.0, r = 0.0;
    for (int s = 0; s < nsp; ++s) {
      l = l + coef[s] * raw[(size_t)s * 2 * nc + j];
      r = r + coef[s] * raw[(size_t)s * 2 * nc + nc + j];
    }
    left[j] = l;
    right[j] = r;
  }
  for (int64_t g = 1; g < nc; ++g) rho[g] = right[g - 1] + left[g];
  if (periodic) {
    rho[0] = right[nc - 1] + left[0];
    rho[nc] = rho[0];
  } else {
    rho[0] = left[0] * 2.0;
    rho[nc] = right[nc - 1] * 2.0;
  }
}

/* ---- collisions (pkg/src/picmc/collisions.py, rng.py) -------------------- */

static uint64_t or_mix64(uint64_t z) { /* rng.py:56-61 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t or_derive(uint64_t key, uint64_t n) { /* rng.py:72-77 */
  return or_mix64(key + (n + 1) * 0x9E3779B97F4A7C15ull);
}
static double or_uniform(uint64_t key, uint64_t c) { /* rng.py:96-98 */
  return (double)(or_derive(key, c) >> 11) * 0x1p-53;
}
static double or_prob(double nden, double rate, double dt) { /* collisions.py:188-192 */
  return -expm1(-(nden * rate) * dt);
}
static void or_unit_vector(uint64_t key, double *ux, double *uy, double *uz) {
  /* collisions.py:97-108 */
  uint64_t t = 0;
  double u, v, s;
  for (;;) {
    u = 2.0 * or_uniform(key, 2 * t) - 1.0;
    v = 2.0 * or_uniform(key, 2 * t + 1) - 1.0;
    s = u * u + v * v;
    if (s < 1.0) break;
    ++t;
  }
  const double f = 2.0 * sqrt(1.0 - s);
  *ux = u * f;
  *uy = v * f;
  *uz = 1.0 - 2.0 * s;
}

/*
 * collision_phase (collisions.py:310-351, collide_block :222-283,
 * _select_and_apply :195-219, _apply_event :111-185) on the canonical flat
 * layout: species arrays in cell-major slot order addressed by offs/counts.
 * Electron velocities are updated in place; each ionization swap_removes a
 * neutral (core.py:205-218): n_counts shrinks and the vacated tail slot gets
 * n_cell = -1.  Newborn pairs are written in ascending cell / event order:
 * nb_cell[k], nb_ion[k*5 .. +5] = (x, vx, vy, vz, yp), nb_e likewise.
 * prm = {w_over_dx, dt, rate_el, rate_ex, rate_io, threshold_j, mass_e,
 * dx_over_dt}.  Returns the number of pairs, -1 on overflow of nb_cap.
 */
int64_t or_collide(uint64_t step_key, int64_t global_offset, int64_t nc, const double *prm,
                   double *evx, double *evy, double *evz, const double *ex, const double *eyp,
                   const int64_t *e_offs, const int64_t *e_counts, double *nx, double *nvx,
                   double *nvy, double *nvz, double *nyp, const int64_t *n_offs,
                   int64_t *n_counts, int32_t *n_cell, int64_t *nb_cell, double *nb_ion,
                   double *nb_e, int64_t nb_cap, int64_t *tally) {
  const double w = prm[0], dt = prm[1], rel = prm[2], rex = prm[3], rio = prm[4];
  const double thr = prm[5], me = prm[6], dxdt = prm[7];
  int64_t nb = 0;
  for (int64_t j = 0; j < nc; ++j) {
    const int64_t ne = e_counts[j];
    if (ne == 0) continue;
    const uint64_t ckey = or_derive(step_key, (uint64_t)(j + global_offset));
    double nd = (double)n_counts[j] * w;
    double pe = or_prob(nd, rel, dt), px = or_prob(nd, rex, dt), pi = or_prob(nd, rio, dt);
    int64_t nsub = 1;
    double dts = dt;
    if (!(pe + px + pi < 0.1)) {
      int m = 0;
      for (;;) {
        ++m;
        dts = dt / (double)(1ull << m);
        if (or_prob(nd, rel, dts) + or_prob(nd, rex, dts) + or_prob(nd, rio, dts) < 0.1) break;
      }
      nsub = (int64_t)1 << m;
    }
    for (int64_t s = 0; s < nsub; ++s) {
      if (nsub > 1) {
        nd = (double)n_counts[j] * w;
        pe = or_prob(nd, rel, dts);
        px = or_prob(nd, rex, dts);
        pi = or_prob(nd, rio, dts);
      }
      const uint64_t sub = or_derive(ckey, (uint64_t)s);
      const uint64_t sel = or_derive(sub, 0), evb = or_derive(sub, 1);
      const double t1 = pe, t2 = pe + px, t3 = t2 + pi;
      for (int64_t slot = 0; slot < ne; ++slot) {
        const double u = or_uniform(sel, (uint64_t)slot);
        if (!(u < t3)) continue;
        const int kind = u < t1 ? 1 : (u < t2 ? 2 : 3);
        const uint64_t ev = or_derive(evb, (uint64_t)slot);
        const int64_t i = e_offs[j] + slot;
        const double speed = sqrt(evx[i] * evx[i] + evy[i] * evy[i] + evz[i] * evz[i]);
        double ux, uy, uz;
        if (kind == 1 || kind == 2) {
          double ns = speed;
          if (kind == 2) {
            const double vsi = speed * dxdt;
            double ke = 0.5 * me * vsi * vsi;
            const double d = ke - thr;
            ke = (0.0 > d) ? 0.0 : d;
            ns = sqrt(2.0 * ke / me) / dxdt;
            tally[1]++;
          } else {
            tally[0]++;
          }
          or_unit_vector(or_derive(ev, 1), &ux, &uy, &uz);
          evx[i] = ns * ux;
          evy[i] = ns * uy;
          evz[i] = ns * uz;
          continue;
        }
        const int64_t nn = n_counts[j];
        if (nn == 0) {
          tally[3]++;
          continue;
        }
        int64_t pick = (int64_t)(or_uniform(or_derive(ev, 0), 0) * (double)nn);
        if (pick >= nn) pick = nn - 1;
        const int64_t ip = n_offs[j] + pick, il = n_offs[j] + nn - 1;
        const double rx = nx[ip], rvx = nvx[ip], rvy = nvy[ip], rvz = nvz[ip];
        const double ryp = nyp ? nyp[ip] : 0.0;
        nx[ip] = nx[il];
        nvx[ip] = nvx[il];
        nvy[ip] = nvy[il];
        nvz[ip] = nvz[il];
        if (nyp) nyp[ip] = nyp[il];
        n_cell[il] = -1;
        n_counts[j] = nn - 1;
        const double vsi = speed * dxdt;
        const double keh = 0.25 * me * vsi * vsi;
        const double sh = sqrt(2.0 * keh / me) / dxdt;
        double qx, qy, qz;
        or_unit_vector(or_derive(ev, 1), &ux, &uy, &uz);
        evx[i] = sh * ux;
        evy[i] = sh * uy;
        evz[i] = sh * uz;
        or_unit_vector(or_derive(ev, 2), &qx, &qy, &qz);
        if (nb >= nb_cap) return -1;
        nb_cell[nb] = j;
        double *r = nb_ion + 5 * nb;
        r[0] = rx; r[1] = rvx; r[2] = rvy; r[3] = rvz; r[4] = ryp;
        r = nb_e + 5 * nb;
        r[0] = ex[i]; r[1] = sh * qx; r[2] = sh * qy; r[3] = sh * qz;
        r[4] = eyp ? eyp[i] : 0.0;
        ++nb;
        tally[2]++;
      }
    }
  }
  return nb;
}

/* push + transfer of one particle array in place, recording per-particle
 * moved flags (delta != 0) for the canonical commit order; same arithmetic as
 * or_step_flat.  Returns the CFL violator index or -1. */
int64_t or_step_moved(int kind, int bc, double fnstep, double kick_coef, const double *bt,
                      const double *bs, const double *e, int64_t nc, int64_t n, double *x,
                      double *vx, double *vy, double *vz, double *yp, int32_t *cell,
                      uint8_t *removed, uint8_t *moved, const double *bnodes, double bf) {
  for (int64_t i = 0; i < n; ++i) moved[i] = 0;
  if (kind == 0) {
    for (int64_t i = 0; i < n; ++i) removed[i] = 0;
    return -1;
  }
  for (int64_t i = 0; i < n; ++i) {
    const int32_t c = cell[i];
    if (kind == OR_KICK || kind == OR_BORIS) {
      const double aj = kick_coef * e[c];
      const double aj1 = kick_coef * e[c + 1];
      const double atemp = aj + x[i] * (aj1 - aj);
      if (kind == OR_KICK) {
        vx[i] = vx[i] + atemp;
      } else {
        double tg[3], sg[3];
        if (bnodes) boris_t_gather(bnodes, bf, c, x[i], tg, sg);
        boris(&vx[i], &vy[i], &vz[i], atemp, bnodes ? tg : bt, bnodes ? sg : bs);
      }
    }
    x[i] = x[i] + fnstep * vx[i];
    if (yp) yp[i] = yp[i] + fnstep * vy[i];
  }
  for (int64_t i = 0; i < n; ++i) {
    const double d = floor(x[i]);
    if (d != 0.0 && fabs(d) >= (double)nc) return i;
  }
  for (int64_t i = 0; i < n; ++i) {
    removed[i] = 0;
    const double d = floor(x[i]);
    if (d == 0.0) continue;
    moved[i] = 1;
    int64_t dest = (int64_t)cell[i] + (int64_t)d;
    double nxv = x[i] - d;
    if (nxv >= 1.0) {
      nxv -= 1.0;
      dest += 1;
    }
    x[i] = nxv;
    if (bc == OR_PERIODIC) {
      cell[i] = (int32_t)pymod(dest, nc);
    } else if (dest < 0) {
      removed[i] = 1;
    } else if (dest >= nc) {
      removed[i] = 2;
    } else {
      cell[i] = (int32_t)dest;
    }
  }
  return -1;
}
