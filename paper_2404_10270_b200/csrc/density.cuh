// Density epilogue arithmetic shared by the epilogue kernels (abi.cu) and
// the fused field cycle (fields.cu): fixed-point bins -> weighted partials.
#pragma once

#include "common.cuh"

namespace pb {

// left/right per cell: species order, 0.0 + coef*L (fields.py:64-77).
__device__ __forceinline__ void weighted_partials(const uint64_t *__restrict__ bins,
                                                  const double *__restrict__ coef,
                                                  int ndep, int64_t nc, int64_t j,
                                                  double &left, double &right,
                                                  pb_status *st) {
  double l = 0.0, r = 0.0;
  for (int s = 0; s < ndep; ++s) {
    const uint64_t R = bins[(size_t)s * 2 * nc + j];
    const uint64_t C = bins[(size_t)s * 2 * nc + nc + j];
    if (C >= kMaxCellCount) flag_overflow(st, C);
    const uint64_t L = (C << kFracBits) - R;
    const double lraw = __dmul_rn(__ull2double_rn(L), kFracInv);
    const double rraw = __dmul_rn(__ull2double_rn(R), kFracInv);
    l = __dadd_rn(l, __dmul_rn(coef[s], lraw));
    r = __dadd_rn(r, __dmul_rn(coef[s], rraw));
  }
  left = l;
  right = r;
}

struct CoefArgs {
  double c[PB_MAX_SPECIES];
};

}  // namespace pb
