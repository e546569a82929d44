// Device plasma loading with the reference's counter-based streams.
//
// init_plasma (pkg/src/picmc/core.py:292-352): per (species, cell) key
// derive(stream(seed, STREAM_INIT, isp), cell); slot s takes
//   x  = uniforms(key, s)
//   r1 = sqrt(-2 log(uniform_open(key, ppc0+4s))),  a1 = 2 pi uniform(key, ppc0+4s+1)
//   r2 = sqrt(-2 log(uniform_open(key, ppc0+4s+2))), a2 = 2 pi uniform(key, ppc0+4s+3)
//   vx = std*(r1 cos a1), vy = std*(r1 sin a1), vz = std*(r2 cos a2)
// splitmix64 is integer arithmetic (pkg/src/picmc/rng.py:56-116), so x is
// bit-exact; log/sin/cos are CUDA's (a few ulp from NumPy's).
#include "common.cuh"
#include "rng.cuh"

namespace pb {

__global__ void k_init(pb_species s, uint64_t skey, int64_t cell_lo,
                       int64_t ncells, int64_t ppc0, double vstd) {
  const double two_pi = 6.283185307179586;
  const int64_t total = ncells * ppc0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lc = i / ppc0;
    const uint64_t slot = (uint64_t)(i - lc * ppc0);
    const int64_t cell = cell_lo + lc;
    const uint64_t key = derive(skey, (uint64_t)cell);
    const uint64_t base = (uint64_t)ppc0 + 4 * slot;
    const double r1 = sqrt(-2.0 * log(uniform_open(key, base)));
    const double a1 = __dmul_rn(two_pi, uniform(key, base + 1));
    const double r2 = sqrt(-2.0 * log(uniform_open(key, base + 2)));
    const double a2 = __dmul_rn(two_pi, uniform(key, base + 3));
    s.x[i] = uniform(key, slot);
    s.vx[i] = __dmul_rn(vstd, __dmul_rn(r1, cos(a1)));
    s.vy[i] = __dmul_rn(vstd, __dmul_rn(r1, sin(a1)));
    s.vz[i] = __dmul_rn(vstd, __dmul_rn(r2, cos(a2)));
    if (s.yp) s.yp[i] = 0.0;
    s.cell[i] = (int32_t)cell;
  }
}

}  // namespace pb

extern "C" int pb_init_species(pb_species *sp, uint64_t species_key,
                               int64_t cell_lo, int64_t cell_hi, int64_t ppc0,
                               double vstd, void *stream) {
  if (!sp || !sp->x || !sp->vx || !sp->vy || !sp->vz || !sp->cell ||
      cell_hi < cell_lo || ppc0 < 0) {
    pb::set_error("pb_init_species: bad arguments");
    return PB_ERR_INVALID;
  }
  const int64_t total = (cell_hi - cell_lo) * ppc0;
  if (total == 0) return PB_OK;
  pb::k_init<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(
      *sp, species_key, cell_lo, cell_hi - cell_lo, ppc0, vstd);
  PB_CHECK_LAUNCH("k_init");
  return PB_OK;
}
