// Library plumbing: error text, version, device queries, and the density
// epilogue (weighted partials + stitch) that turns fixed-point bins into rho.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "density.cuh"

namespace pb {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// Programmatic dependent launch for the per-step chain (measured, DESIGN.md
// 3.1c); compile with -DPB_PDL=0 for the A/B without it.
#ifndef PB_PDL
#define PB_PDL 1
#endif
bool pdl_enabled() { return PB_PDL != 0; }

int cuda_status(cudaError_t err, const char *what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(err), cudaGetErrorName(err));
  return PB_ERR_CUDA;
}

__global__ void k_rho_epilogue(const uint64_t *__restrict__ bins, CoefArgs ca,
                               int ndep, int64_t nc, int field_bc,
                               double *__restrict__ left,
                               double *__restrict__ right,
                               double *__restrict__ rho,
                               uint64_t *__restrict__ clear,
                               pb_status *st) {
  pdl_enter();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g > nc) return;
  // Step fusion: zero the other (ping-pong) bin set for the coming mover
  // launch.
  if (clear && g < nc)
    for (int s = 0; s < ndep; ++s) {
      clear[(size_t)s * 2 * nc + g] = 0;
      clear[(size_t)s * 2 * nc + nc + g] = 0;
    }
  double lg = 0.0, rg = 0.0, lp = 0.0, rp = 0.0;
  if (g < nc) {
    weighted_partials(bins, ca.c, ndep, nc, g, lg, rg, st);
    if (left) left[g] = lg;
    if (right) right[g] = rg;
  }
  if (g > 0) weighted_partials(bins, ca.c, ndep, nc, g - 1, lp, rp, nullptr);
  double v;
  if (g > 0 && g < nc) {
    v = __dadd_rn(rp, lg);  // rho[g] = R[g-1] + L[g] (fields.py:85)
  } else if (field_bc == PB_FIELD_PERIODIC) {
    double l0, r0, ll, rl;  // rho[0] = rho[nc] = R[nc-1] + L[0]
    weighted_partials(bins, ca.c, ndep, nc, 0, l0, r0, nullptr);
    weighted_partials(bins, ca.c, ndep, nc, nc - 1, ll, rl, nullptr);
    v = __dadd_rn(rl, l0);
  } else if (g == 0) {
    v = __dmul_rn(lg, 2.0);  // walls own half a cell (fields.py:115-117)
  } else {
    v = __dmul_rn(rp, 2.0);
  }
  rho[g] = v;
}

// Engine form, split in two so the bins can be cleared as they are read:
// k_partials_clear has one thread per cell touching only its own bins, so it
// zeroes them after reading (the ping-pong invariant: a bin set is zero again
// once its density has been taken), then k_stitch builds rho from left/right.
// Neither touches the set the concurrent mover deposits into, so in CUDA-graph
// replay the epilogue runs on a side stream overlapped with the next push.
__global__ void k_partials_clear(uint64_t *__restrict__ bins, CoefArgs ca, int ndep, int64_t nc,
                                 double *__restrict__ left, double *__restrict__ right,
                                 uint64_t *__restrict__ clear, pb_status *st) {
  pdl_enter();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nc) return;
  double l, r;
  weighted_partials(bins, ca.c, ndep, nc, g, l, r, st);
  left[g] = l;
  right[g] = r;
  for (int s = 0; s < ndep; ++s) {
    bins[(size_t)s * 2 * nc + g] = 0;
    bins[(size_t)s * 2 * nc + nc + g] = 0;
    if (clear) {
      clear[(size_t)s * 2 * nc + g] = 0;
      clear[(size_t)s * 2 * nc + nc + g] = 0;
    }
  }
}

// wall = 2.0: deposit_charge's doubled wall nodes (fields.py:115-117);
// wall = 1.0: plain stitch_rho (fields.py:89-91, x*1.0 == x exactly).
__global__ void k_stitch(const double *__restrict__ left, const double *__restrict__ right,
                         int64_t nc, int field_bc, double *__restrict__ rho, double wall) {
  pdl_enter();
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g > nc) return;
  double v;
  if (g > 0 && g < nc) {
    v = __dadd_rn(right[g - 1], left[g]);  // fields.py:85
  } else if (field_bc == PB_FIELD_PERIODIC) {
    v = __dadd_rn(right[nc - 1], left[0]);
  } else if (g == 0) {
    v = __dmul_rn(left[0], wall);
  } else {
    v = __dmul_rn(right[nc - 1], wall);
  }
  rho[g] = v;
}

}  // namespace pb

extern "C" int pb_abi_version(void) { return PB_ABI_VERSION; }

extern "C" size_t pb_status_bytes(void) { return sizeof(pb_status); }

extern "C" const char *pb_last_error(void) { return pb::g_err; }

extern "C" int pb_device_sm_count(int *out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaGetDevice");
  e = cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return pb::cuda_status(e, "cudaDeviceGetAttribute");
  return PB_OK;
}

static int rho_epilogue(const uint64_t *bins, const double *coef, int ndep, int64_t nc,
                        int field_bc, double *left, double *right, double *rho,
                        uint64_t *clear, pb_status *status, void *stream) {
  if (ndep < 0 || ndep > PB_MAX_SPECIES) {
    pb::set_error("ndep=%d outside [0, %d]", ndep, PB_MAX_SPECIES);
    return PB_ERR_INVALID;
  }
  if (nc < 2 || !rho || (ndep > 0 && (!bins || !coef))) {
    pb::set_error("pb_rho_epilogue: bad arguments (nc=%lld)", (long long)nc);
    return PB_ERR_INVALID;
  }
  if (field_bc != PB_FIELD_PERIODIC && field_bc != PB_FIELD_DIRICHLET) {
    pb::set_error("unknown field boundary %d", field_bc);
    return PB_ERR_INVALID;
  }
  pb::CoefArgs ca;  // passed by value: no host pointer reaches the device
  memset(&ca, 0, sizeof(ca));
  for (int s = 0; s < ndep; ++s) ca.c[s] = coef[s];
  const int threads = 256;
  const int64_t blocks = (nc + 1 + threads - 1) / threads;
  cudaError_t e = pb::launch_pdl(pb::k_rho_epilogue, dim3((unsigned)blocks), dim3(threads), 0,
                                  (cudaStream_t)stream, bins, ca, ndep, nc, field_bc, left, right,
                                  rho, clear, status);
  if (e != cudaSuccess) return pb::cuda_status(e, "k_rho_epilogue");
  return PB_OK;
}

extern "C" int pb_rho_epilogue(const uint64_t *bins, const double *coef, int ndep, int64_t nc,
                               int field_bc, double *left, double *right, double *rho,
                               pb_status *status, void *stream) {
  return rho_epilogue(bins, coef, ndep, nc, field_bc, left, right, rho, nullptr, status, stream);
}

extern "C" int pb_density_step(uint64_t *bins, uint64_t *bins_next, pb_status *status,
                               const double *coef, int ndep, int64_t nc, int field_bc,
                               double *left, double *right, double *rho, void *stream) {
  if (bins_next == bins && bins != nullptr) {
    pb::set_error("pb_density_step: bins_next must not alias bins");
    return PB_ERR_INVALID;
  }
  if (ndep < 0 || ndep > PB_MAX_SPECIES || nc < 2 || !rho || !left || !right ||
      (ndep > 0 && (!bins || !coef)) ||
      (field_bc != PB_FIELD_PERIODIC && field_bc != PB_FIELD_DIRICHLET)) {
    pb::set_error("pb_density_step: bad arguments (nc=%lld ndep=%d)", (long long)nc, ndep);
    return PB_ERR_INVALID;
  }
  pb::CoefArgs ca;
  memset(&ca, 0, sizeof(ca));
  for (int s = 0; s < ndep; ++s) ca.c[s] = coef[s];
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  const int64_t b1 = (nc + threads - 1) / threads, b2 = (nc + 1 + threads - 1) / threads;
  cudaError_t e = pb::launch_pdl(pb::k_partials_clear, dim3((unsigned)b1), dim3(threads), 0, st, bins,
                                  ca, ndep, nc, left, right, bins_next, status);
  if (e != cudaSuccess) return pb::cuda_status(e, "k_partials_clear");
  e = pb::launch_pdl(pb::k_stitch, dim3((unsigned)b2), dim3(threads), 0, st, (const double *)left,
                     (const double *)right, nc, field_bc, rho, 2.0);
  if (e != cudaSuccess) return pb::cuda_status(e, "k_stitch");
  return PB_OK;
}

// ---------------------------------------------------------------------------
// Speed-of-light probe for the roofline: streams exactly the mover's bytes
// per species kind with a trivial update and no physics, 4 particles per
// thread, 256-bit accesses, full occupancy --
//   KICK   R x, vx, cell index   W x, vx
//   BORIS  R x, vx, vy, vz, cell W x, vx, vy, vz
//   DRIFT  R x, vx               W x
//   + yp   R vy, yp              W yp
// It measures what this read/write mix can reach on the part; the mover's
// achieved bandwidth is reported against the copy peak, not against this.
namespace pb {
__device__ __forceinline__ void sol_ld(const double *p, double &a, double &b, double &c, double &d) {
  asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void sol_st(double *p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

__global__ void __launch_bounds__(256) k_stream_sol(double *x, double *vx, double *vy, double *vz,
                                                    double *yp, const int32_t *cell,
                                                    const int8_t *cell8, int64_t n, int write_v,
                                                    int boris) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i + 3 < n; i += stride) {
    double a0, a1, a2, a3, b0, b1, b2, b3;
    sol_ld(x + i, a0, a1, a2, a3);
    sol_ld(vx + i, b0, b1, b2, b3);
    int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    if (cell8) {  // the mover's compressed cell index: 4 bytes per lane
      const int p = __ldcs(reinterpret_cast<const int *>(cell8 + i));
      c0 = p & 1; c1 = (p >> 8) & 1; c2 = (p >> 16) & 1; c3 = (p >> 24) & 1;
    } else if (cell) {
      const int4 c = __ldcs(reinterpret_cast<const int4 *>(cell + i));
      c0 = c.x; c1 = c.y; c2 = c.z; c3 = c.w;
    }
    a0 += b0 + c0; a1 += b1 + c1; a2 += b2 + c2; a3 += b3 + c3;
    sol_st(x + i, a0, a1, a2, a3);
    if (write_v) sol_st(vx + i, b0, b1, b2, b3);
    if (boris) {
      double y0, y1, y2, y3, z0, z1, z2, z3;
      sol_ld(vy + i, y0, y1, y2, y3);
      sol_ld(vz + i, z0, z1, z2, z3);
      sol_st(vy + i, y0 + z0, y1 + z1, y2 + z2, y3 + z3);
      sol_st(vz + i, z0 + b0, z1 + b1, z2 + b2, z3 + b3);
    }
    if (yp) {
      double y0, y1, y2, y3, w0, w1, w2, w3;
      sol_ld(yp + i, y0, y1, y2, y3);
      if (boris) {  // vy already read
        w0 = w1 = w2 = w3 = 1.0;
      } else {
        sol_ld(vy + i, w0, w1, w2, w3);
      }
      sol_st(yp + i, y0 + w0, y1 + w1, y2 + w2, y3 + w3);
    }
  }
}
}  // namespace pb

extern "C" int pb_stream_sol(const pb_species *sp, int nsp, void *stream) {
  int sms = 0;
  int rc = pb_device_sm_count(&sms);
  if (rc) return rc;
  for (int k = 0; k < nsp; ++k) {
    const pb_species &s = sp[k];
    if (s.kind == PB_KIND_INACTIVE || s.n < 4) continue;
    const bool charged = s.kind != PB_KIND_DRIFT;
    const bool boris = s.kind == PB_KIND_BORIS;
    pb::k_stream_sol<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(
        s.x, s.vx, s.vy, s.vz, s.yp, charged ? s.cell : nullptr, charged ? s.cell8 : nullptr,
        s.n & ~(int64_t)3, charged ? 1 : 0, boris ? 1 : 0);
  }
  PB_CHECK_LAUNCH("k_stream_sol");
  return PB_OK;
}

extern "C" int pb_stitch_rho(const double *left, const double *right, int64_t nc, int periodic,
                             double *rho, void *stream) {
  if (nc < 1 || !left || !right || !rho) {
    pb::set_error("pb_stitch_rho: bad arguments (nc=%lld)", (long long)nc);
    return PB_ERR_INVALID;
  }
  const int threads = 256;
  const int64_t blocks = (nc + 1 + threads - 1) / threads;
  pb::k_stitch<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      left, right, nc, periodic ? PB_FIELD_PERIODIC : PB_FIELD_DIRICHLET, rho, 1.0);
  PB_CHECK_LAUNCH("k_stitch");
  return PB_OK;
}
