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
                     int64_t *cfl_index) {
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
        boris(&vx[i], &vy[i], &vz[i], atemp, bt, bs);
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
