// mact_common.cuh — shared device helpers for libmact_cuda (sm_100a).
//
// Kernel-side coefficient block, PTX wrappers for the Blackwell bulk-copy
// engine (cp.async.bulk = TMA 1-D, SASS UBLKCP) and mbarriers, cheap
// float<->double bit conversions, and launch bookkeeping.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/mact_cuda.h"

namespace mact {

// Device-side invariant checks of the checked build (scripts/hazard_check.sh:
// MACT_NVCC_DEFS=-DMACT_CHECKS MACT_LIB_TAG=checks).  Shared-memory gather
// indices, DSMEM exchange sizes and ring positions are asserted there; a
// failure prints the condition and traps (the launch then reports an error).
// The product build compiles them away.
#ifdef MACT_CHECKS
#define MACT_DCHECK(cond)                                                                              \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("MACT_DCHECK %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x,        \
             (int)threadIdx.x, #cond);                                                                  \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define MACT_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

constexpr double kPi = 3.14159265358979311600;   // np.pi
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kSqrt2 = 1.4142135623730951;    // math.sqrt(2.0), approximants.py:21
constexpr double kSqrt3 = 1.7320508075688772;    // math.sqrt(3.0), approximants.py:22

// BT.709 / D65 constants (exact.py:21-40)
constexpr double kGammaKnee = 0.081, kGammaSlope = 4.5, kGammaOffset = 0.099,
                 kGammaScale = 1.099, kGammaPower = 1.0 / 0.45;
constexpr double kWhiteX = 0.950456, kWhiteY = 1.0, kWhiteZ = 1.089058;
constexpr double kLabKnee = 0.008856, kLabSlope = 7.787, kLabOffset = 16.0 / 116.0;
__host__ __device__ constexpr double rgb2xyz(int row, int col) {
  return row == 0 ? (col == 0 ? 0.412391 : col == 1 ? 0.357584 : 0.180481)
       : row == 1 ? (col == 0 ? 0.212639 : col == 1 ? 0.715169 : 0.072192)
                  : (col == 0 ? 0.019331 : col == 1 ? 0.119195 : 0.950532);
}

// RGB->XYZ rows pre-divided by the D65 white point, rounded once to fp32 --
// compile-time immediates (exact.py:21-66 fixes them; MactConfig cannot), so
// the FMAs take them as instruction operands instead of registers reloaded
// from the parameter bank.  KCoeffs::mxyz holds the same values (host check).
__host__ __device__ constexpr float kMxyz(int row, int col) {
  return (float)(rgb2xyz(row, col) / (row == 0 ? kWhiteX : row == 1 ? kWhiteY : kWhiteZ));
}

// Degree caps of the bundled sets: CIELAB rationals up to (4,4), the HSI
// refit and SCT polynomials up to 5.  Unused high coefficients are zero,
// which leaves Horner bit-identical (0*x + 0 = 0, then 0*x + a_n = a_n).
constexpr int kCbrtDeg = 4;
constexpr int kPolyDeg = 5;

// Segment table of the fp32 CIELAB lightness kernel (see KCoeffs::seg).
constexpr int kLabSegShift = 19;                                   // 16 segments per binade
constexpr uint32_t kLabSegMask = ~((1u << kLabSegShift) - 1u);
constexpr uint32_t kLabSegBase = 0x3C000000u >> kLabSegShift;      // 2^-7
constexpr int kLabSegs = (int)((0x3F800000u >> kLabSegShift) - kLabSegBase + 1);   // up to [1, 1.0625)
constexpr int kLabSegCopies = 8;   // bank-private smem copies: an 8-lane LDS.128 phase is conflict-free

// Kernel parameter block built on the host from MactCoeffs (passed by value
// as a __grid_constant__ parameter, so it lives in the constant bank and the
// FMAs take coefficients as c[][] operands — no registers, no globals).
struct KCoeffs {
  double cbrt_num[kCbrtDeg + 1];
  double cbrt_den[kCbrtDeg + 1];
  double hsi_d[kPolyDeg + 1], asin_d[kPolyDeg + 1], acos_d[kPolyDeg + 1],
      atanf_d[kPolyDeg + 1], atang_d[kPolyDeg + 1];
  float hsi[kPolyDeg + 1], asin[kPolyDeg + 1], acos[kPolyDeg + 1], atanf[kPolyDeg + 1],
      atang[kPolyDeg + 1];
  float mxyz[9];   // RGB->XYZ rows pre-divided by the white point (fp32)
  // Degree-(4,4) fast path.  With P' = P/p4, Q' = Q/q4 (monic) and k = p4/q4,
  //   f = P/Q = k P'/Q' = k (1 + (P' - Q')/Q') = k + s q,   q = D'(t)/Q'(t),
  // where D' is the monic cubic (P' - Q')/e3 and s = k e3.  One fp64 Horner
  // step fewer than evaluating P' (the t^4 terms cancel), and the constant k
  // disappears into the CIELAB epilogue:
  //   L* = 116 s qy + (116 k - 16),  a* = 500 s (qx - qy),  b* = 200 s (qy - qz).
  int32_t monic44;                  // 1 when the configuration is (4,4)
  double qm[4], dm[3];              // Q' = t^4 + qm3 t^3 + ...,  D' = t^3 + dm2 t^2 + ...
  double lin_s, lin_o;              // linear branch expressed in q: q = lin_s t + lin_o
  double l_s, l_o;                  // 116 s, 116 k - 16
  float a_s, b_s;                   // 500 s, 200 s
  // Segmented fp32 form of the same rational (any degrees), used when its
  // fit passed the host-side check (lab_seg = 1).  Segment i covers the fp32
  // values whose bits >> kLabSegShift equal kLabSegBase + i, i.e. 16
  // segments per binade from 2^-7 (below the knee 0.008856) to [1, 1.0625).
  // On it, R(t) ~= hi + u (c1 + u (c2 + u c3)) with u = t - t_seg exact:
  // seg[i] = (hi, c1, c2, c3).  The linear branch below the knee is
  // lin_hi + (lin_slope t + lin_lo).
  int32_t lab_seg;
  float lin_hi, lin_lo, lin_slope;
  float4 seg[kLabSegs];
};

// ---------------------------------------------------------------- Horner
template <int DEG>
__device__ __forceinline__ float horner_f(const float* c, float x) {
  float acc = c[DEG];
#pragma unroll
  for (int k = DEG - 1; k >= 0; --k) acc = fmaf(acc, x, c[k]);
  return acc;
}
template <int DEG>
__device__ __forceinline__ double horner_d(const double* c, double x) {
  double acc = c[DEG];
#pragma unroll
  for (int k = DEG - 1; k >= 0; --k) acc = fma(acc, x, c[k]);
  return acc;
}

// ------------------------------------------------- float <-> double bit moves
// Valid for positive normal inputs (and harmless garbage-but-finite for +0).
// They replace F2F.F64.F32 / F2F.F32.F64, which issue on the quarter-rate
// conversion pipe, by 2-3 integer ops on the ALU pipe.
__device__ __forceinline__ double f2d_pos(float f) {
  uint32_t b = __float_as_uint(f);
  uint32_t hi = (b >> 3) + 0x38000000u;
  uint32_t lo = b << 29;
  return __hiloint2double((int)hi, (int)lo);
}
// Truncating double->float for positive normal values inside float range.
__device__ __forceinline__ float d2f_pos_trunc(double d) {
  uint32_t hi = (uint32_t)__double2hiint(d) - 0x38000000u;
  uint32_t lo = (uint32_t)__double2loint(d);
  return __uint_as_float(__funnelshift_l(lo, hi, 3));
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// Byte k of w as an exact float (one PRMT builds 2^23 + byte, one FADD removes 2^23).
__device__ __forceinline__ float fbyte(uint32_t w, int k) {
  return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540u | (uint32_t)k)) - 8388608.0f;
}
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int k) {
  return __byte_perm(w, 0u, 0x4440u + (uint32_t)k);
}

// ------------------------------------------------ exact integer -> float
// Magic-number conversion for 0 <= v < 2^23 (IADD + FADD instead of I2F).
__device__ __forceinline__ float u2f_small(uint32_t v) {
  return __uint_as_float(v + 0x4B000000u) - 8388608.0f;
}

// ------------------------------------------------------------ PTX: mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Blocking wait on an mbarrier phase.  The suspend-time hint lets the
// hardware park the warp until the phase completes (instead of returning
// false after a short internal timeout and spinning through YIELD/BRA).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(0x100000u)
      : "memory");
}

// -------------------------------------------- PTX: bulk copy engine (TMA 1-D)
// global -> shared, completion signalled on an mbarrier (complete_tx::bytes).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global, bulk-group completion.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// Make generic-proxy shared-memory writes visible to the async (bulk) proxy.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------- host side
void count_launch(int k = 1);
// NVTX range around a library call (visible in Nsight Systems / `ncu --nvtx`);
// a few ns when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
int num_sms();
// cudaDevAttrReservedSharedMemoryPerBlock of the current device (cached).
int reserved_smem();
int make_kcoeffs(const MactCoeffs* c, KCoeffs* out);
// Sets the dynamic-smem attribute once per (kernel, device) and returns the
// persistent grid size occupancy x SM count (cached), or <= 0 on error.
int persistent_grid(const void* fn, int threads, size_t smem_bytes);
int grid_cap();   // MACT_GRID_CAP (debug): upper bound on persistent grids, in CTAs

}  // namespace mact
