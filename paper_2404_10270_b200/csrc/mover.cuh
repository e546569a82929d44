// Per-particle mover arithmetic shared by the production mover
// (push_deposit.cu) and the canonical-order mover (canonical.cu): the
// reference kick/drift (pkg/src/picmc/backends/_kernels.pyx:81-101), the
// Boris extension and the resort_collect cell transfer
// (pkg/src/picmc/mover.py:136-163), all with explicit _rn intrinsics.
#pragma once

#include "common.cuh"

namespace pb {

// ---------------------------------------------------------------------------
// Per-particle mover arithmetic.  Returns the new state in place.
// ---------------------------------------------------------------------------
struct MoveOut {
  int32_t cell;
  bool moved;      // cell changed (or removed)
  int8_t wall;     // -1 none, 0 left, 1 right (absorbing only)
  bool cfl;        // |floor(x)| >= nc
};

// Device-internal kind: PB_KIND_BORIS with a B node profile (b_nodes set).
// A separate instantiation, so the uniform-B Boris path keeps its registers.
constexpr int kKindBorisB = 4;
__host__ __device__ constexpr bool is_boris(int k) { return k == PB_KIND_BORIS || k == kKindBorisB; }

// Spatially varying B (pb_species.b_nodes): one 32-byte read-only load per
// node (bx, by, bz, pad; L2-resident), the one-sided linear gather of
// f*B in the same form as accel_nodes (pkg/src/picmc/mover.py:221), then
// s = t * (2 / (1 + |t|^2)) -- one division per particle; the host's
// boris_coefficients op order (engine.py), so a constant profile reproduces
// the uniform path.
__device__ __forceinline__ void ldg_node4(const double *p, double &a, double &b, double &c) {
  double d;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

__device__ __forceinline__ double node_gather(double f, double b0, double b1, double x) {
  const double t0 = __dmul_rn(f, b0);
  const double t1 = __dmul_rn(f, b1);
  return __dadd_rn(t0, __dmul_rn(x, __dsub_rn(t1, t0)));
}

__device__ __forceinline__ void boris_t_gather(const pb_species &s, int32_t cell, double x,
                                               double &tx, double &ty, double &tz, double &sx,
                                               double &sy, double &sz) {
  double b0x, b0y, b0z, b1x, b1y, b1z;
  ldg_node4(s.b_nodes + 4 * (int64_t)cell, b0x, b0y, b0z);
  ldg_node4(s.b_nodes + 4 * (int64_t)cell + 4, b1x, b1y, b1z);
  const double f = s.boris_f;
  tx = node_gather(f, b0x, b1x, x);
  ty = node_gather(f, b0y, b1y, x);
  tz = node_gather(f, b0z, b1z, x);
  const double t2 = __dadd_rn(__dadd_rn(__dmul_rn(tx, tx), __dmul_rn(ty, ty)), __dmul_rn(tz, tz));
  const double g = __ddiv_rn(2.0, __dadd_rn(1.0, t2));
  sx = __dmul_rn(tx, g);
  sy = __dmul_rn(ty, g);
  sz = __dmul_rn(tz, g);
}

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
  } else if (is_boris(KIND)) {
    // Boris (config 4, restated in oracle/picmc_oracle.c:boris_push):
    // half kick, rotation v' = v- + v- x t, v+ = v- + v' x s, half kick.
    const double aj = __dmul_rn(s.kick_coef, __ldg(e + cell));
    const double aj1 = __dmul_rn(s.kick_coef, __ldg(e + cell + 1));
    const double daj = __dsub_rn(aj1, aj);
    const double atemp = __dadd_rn(aj, __dmul_rn(x, daj));
    const double h = __dmul_rn(0.5, atemp);
    double tx = s.boris_t[0], ty = s.boris_t[1], tz = s.boris_t[2];
    double sx = s.boris_s[0], sy = s.boris_s[1], sz = s.boris_s[2];
    if (KIND == kKindBorisB) boris_t_gather(s, cell, x, tx, ty, tz, sx, sy, sz);
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

}  // namespace pb
