// Shared helpers for the sm_100a kernels of libpicmc_b200.
//
// Arithmetic discipline: the reference compiles its kernels with
// -ffp-contract=off (pkg/setup.py:9-12), so every expression that must match
// it bit for bit is spelled with explicit round-to-nearest intrinsics
// (__dadd_rn / __dmul_rn / __dsub_rn) and the whole library is additionally
// built with --fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/picmc_b200.h"

namespace pb {

// Thread-local error text for pb_last_error().
void set_error(const char *fmt, ...);
int cuda_status(cudaError_t err, const char *what);

#define PB_CHECK_LAUNCH(what)                                   \
  do {                                                          \
    cudaError_t e__ = cudaGetLastError();                       \
    if (e__ != cudaSuccess) return ::pb::cuda_status(e__, what); \
  } while (0)

constexpr int kFracBits = PB_DEPOSIT_FRAC_BITS;
constexpr double kFracScale = 281474976710656.0;       // 2^48
constexpr double kFracInv = 1.0 / 281474976710656.0;   // 2^-48
// Packed warp-scan payload: bits [0,56) = R sum, bits [56,64) = count.
constexpr int kCountShift = 56;
constexpr uint64_t kRMask = (uint64_t(1) << kCountShift) - 1;

// The fixed-point bins of one species in one cell hold R = sum round(x*2^48)
// <= C*2^48 and the epilogue forms C<<48: both wrap once a cell holds
// kMaxCellCount particles of one species (summed over ranks).  Every reader
// of the bins checks C against it and flags the step (PB_ERR_OVERFLOW, the
// largest count seen in pb_status.overflow) instead of producing a wrong rho.
constexpr uint64_t kMaxCellCount = uint64_t(1) << (64 - PB_DEPOSIT_FRAC_BITS);

__device__ __forceinline__ void flag_overflow(pb_status *st, uint64_t count) {
  if (!st) return;
  atomicMax(reinterpret_cast<unsigned long long *>(&st->overflow), (unsigned long long)count);
  atomicCAS(&st->code, PB_OK, PB_ERR_OVERFLOW);
}

// Quantise a cell-relative position in [0,1) to the deposit fixed point:
// round-to-nearest-even of x * 2^48 (exact: a power-of-two scale).  Adding
// 2^52 puts the value in the binade whose ulp is 1, so that single rounding
// IS the round-to-nearest-even to an integer and leaves it in the low
// mantissa bits -- bitwise __double2ull_rn, with a DADD in place of the
// F2I.U64.F64 conversion on the mover's per-particle path.
__device__ __forceinline__ uint64_t quantize(double x) {
  const double v = __dadd_rn(__dmul_rn(x, kFracScale), 4503599627370496.0);  // + 2^52
  return (uint64_t)__double_as_longlong(v) - 0x4330000000000000ull;
}

// Sum of per-particle fixed-point weights, packed with a count.
__device__ __forceinline__ uint64_t deposit_word(double x) {
  return (uint64_t(1) << kCountShift) | quantize(x);
}

__device__ __forceinline__ unsigned lane_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

// Python floor-mod for the periodic wrap (mover.py:156, `% nc_global`).
__device__ __forceinline__ int64_t floor_mod(int64_t a, int64_t m) {
  int64_t r = a % m;
  return r < 0 ? r + m : r;
}

// ---- programmatic dependent launch (PDL) ------------------------------------
// The per-step chain (density epilogue -> smoothing -> Poisson tiles -> E ->
// mover -> compaction) is a string of dependent kernels, most of them a few
// microseconds long.  Launched with programmatic stream serialisation, a
// kernel's successor is scheduled while it still runs: every CTA waits until
// the predecessor grid has completed and its writes are visible
// (griddepcontrol.wait) before touching memory, then lets its own dependent
// launch (launch_dependents) -- the same ordering as plain stream order,
// minus the launch gap, with at most one kernel queued ahead.  Both are
// no-ops without the launch attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// The two halves, for kernels that should hold their dependents back (a
// dependent launched early is resident beside the kernel; see
// k_field_fused).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();  // compile-time PB_PDL (default 1)

// Launch `kern` with programmatic stream serialisation (when enabled); the
// kernel must call pdl_enter() before its first global memory access.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace pb
