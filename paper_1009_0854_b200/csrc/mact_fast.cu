// mact_fast.cu — K1-K3 (+ fused triple): the MACT fast transforms.
//
//   mact_lab_fast  <- mact.fast.rgb_to_lab_fast  (fast.py:86-115)
//   mact_hsi_fast  <- mact.fast.rgb_to_hsi_fast  (fast.py:118-148)
//   mact_sct_fast  <- mact.fast.rgb_to_sct_fast  (fast.py:151-203)
//   mact_all_fast  <- all three from one read of the pixels (BASELINE config 5)
//
// uint8 input runs the streaming kernel of mact_stream.cuh; real-valued
// input (the reference's float path, fast.py:96-99) runs a per-pixel fp64
// kernel that follows the reference formulas operation for operation.
#include "mact_pixel.cuh"
#include <type_traits>

#include "mact_stream.cuh"

namespace mact {

// ---------------------------------------------------------------- ops
// px(): one pixel (tail / unaligned kernel); px4w(): the 4 pixels packed in
// three input words (streaming kernel, warp-converged).  Both run the same
// arithmetic, so tile and tail results are bit-identical.
// GAMMA_TABLE rounded to fp32, generated from the oracle's fp64 table (the
// reference's numpy pow).  Loading it costs a CTA ~0.1 us; evaluating 256
// fp64 pow() per CTA cost ~0.9 us, 20 % of a 512^2 image (BASELINE C1).
__device__ const float kGammaF32[256] = {
#include "mact_gamma_table.inc"
};

// CIELAB op: both tables in one 64 KB-aligned shared block (PackedTab,
// mact_pixel.cuh), which the skeleton places at an aligned offset.
struct OpLab {
  static constexpr int NOUT = 1;
  using Params = KCoeffs;
  using Tab = PackedTab;
  struct alignas(128) Shared {
    static constexpr uint32_t kAlign = PackedTab::kBytes;
    float rows[256 * 64];   // row r: GAMMA_TABLE[r] (fast.py:35, fp32) x 32 lanes | segment r x 8 copies
  };
  static_assert(sizeof(Shared) == PackedTab::kBytes, "packed table is 256 rows of 256 B");
  static __device__ __forceinline__ void init(Shared* s, const Params& c) {
    for (int k = threadIdx.x; k < 256; k += blockDim.x) {   // L2-resident table, one row per thread
      const float v = __ldg(kGammaF32 + k);
      float4* row = reinterpret_cast<float4*>(s->rows + (k << 6));
#pragma unroll
      for (int j = 0; j < 8; ++j) row[(j + k) & 7] = make_float4(v, v, v, v);   // rotated: 8 rows, 8 bank groups
    }
    if (c.lab_seg) {   // warp-uniform parameter reads (one constant-cache broadcast per entry)
      const int lane = (int)(threadIdx.x & 31), nw = (int)(blockDim.x >> 5);
      for (int i = (int)(threadIdx.x >> 5); i < kLabSegs; i += nw) {
        const float4 v = c.seg[i];
        if (lane < 8) reinterpret_cast<float4*>(s->rows)[i * 16 + 8 + lane] = v;
      }
    }
  }
  static __device__ __forceinline__ Tab tab(const Shared* s, uint32_t lane, const Params&) {
    return Tab(s->rows, lane);
  }
  static __device__ __forceinline__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared* s,
                                            uint32_t lane, const Params& c, float (*o)[3]) {
    const Lab3 v = lab_fast_u8(r, g, b, tab(s, lane, c), c);
    o[0][0] = v.c0; o[0][1] = v.c1; o[0][2] = v.c2;
  }
  static __device__ __forceinline__ void px4w(uint32_t w0, uint32_t w1, uint32_t w2,
                                              const Shared* s, uint32_t lane, const Params& c,
                                              float (*o)[1][3]) {
    const Tab t = tab(s, lane, c);
    if (c.lab_seg || c.monic44) {
      float v[4][3];
      lab_fast_u8x4(w0, w1, w2, t, c, v);
#pragma unroll
      for (int q = 0; q < 4; ++q) { o[q][0][0] = v[q][0]; o[q][0][1] = v[q][1]; o[q][0][2] = v[q][2]; }
    } else {
      const uint32_t ch[12] = {byte_of(w0, 0), byte_of(w0, 1), byte_of(w0, 2), byte_of(w0, 3),
                               byte_of(w1, 0), byte_of(w1, 1), byte_of(w1, 2), byte_of(w1, 3),
                               byte_of(w2, 0), byte_of(w2, 1), byte_of(w2, 2), byte_of(w2, 3)};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const Lab3 v = lab_fast_u8(ch[3 * q], ch[3 * q + 1], ch[3 * q + 2], t, c);
        o[q][0][0] = v.c0; o[q][0][1] = v.c1; o[q][0][2] = v.c2;
      }
    }
  }
};

// 4 pixels of three words as exact floats: pixel q = bytes 3q, 3q+1, 3q+2.
__device__ __forceinline__ void words_to_rgbf(uint32_t w0, uint32_t w1, uint32_t w2, float (&f)[12]) {
  f[0] = fbyte(w0, 0); f[1] = fbyte(w0, 1); f[2] = fbyte(w0, 2); f[3] = fbyte(w0, 3);
  f[4] = fbyte(w1, 0); f[5] = fbyte(w1, 1); f[6] = fbyte(w1, 2); f[7] = fbyte(w1, 3);
  f[8] = fbyte(w2, 0); f[9] = fbyte(w2, 1); f[10] = fbyte(w2, 2); f[11] = fbyte(w2, 3);
}

template <int SPACE>
struct OpPoly {   // HSI / SCT: fp32 exact-integer formulation
  static constexpr int NOUT = 1;
  using Params = KCoeffs;
  struct Shared { int unused; };
  static __device__ __forceinline__ void init(Shared*, const Params&) {}
  static __device__ __forceinline__ Lab3 eval(float r, float g, float b, const Params& c) {
    return SPACE == MACT_SPACE_HSI ? hsi_fast_f(r, g, b, c) : sct_fast_f(r, g, b, c);
  }
  static __device__ __forceinline__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared*,
                                            uint32_t, const Params& c, float (*o)[3]) {
    const Lab3 v = eval(u2f_small(r), u2f_small(g), u2f_small(b), c);
    o[0][0] = v.c0; o[0][1] = v.c1; o[0][2] = v.c2;
  }
  static __device__ __forceinline__ void px4w(uint32_t w0, uint32_t w1, uint32_t w2, const Shared*,
                                              uint32_t, const Params& c, float (*o)[1][3]) {
    float f[12];
    words_to_rgbf(w0, w1, w2, f);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const Lab3 v = eval(f[3 * q], f[3 * q + 1], f[3 * q + 2], c);
      o[q][0][0] = v.c0; o[q][0][1] = v.c1; o[q][0][2] = v.c2;
    }
  }
};
using OpHsi = OpPoly<MACT_SPACE_HSI>;

// Calibration op: out = (r, g, b) as floats — the same 3 B in / 12 B out
// stream with no arithmetic, i.e. the achievable bandwidth ceiling of the
// skeleton on this I/O pattern (reported next to the roofline in bench.py).
struct OpExpand {
  static constexpr int NOUT = 1;
  using Params = KCoeffs;
  struct Shared { int unused; };
  static __device__ __forceinline__ void init(Shared*, const Params&) {}
  static __device__ __forceinline__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared*,
                                            uint32_t, const Params&, float (*o)[3]) {
    o[0][0] = u2f_small(r); o[0][1] = u2f_small(g); o[0][2] = u2f_small(b);
  }
  static __device__ __forceinline__ void px4w(uint32_t w0, uint32_t w1, uint32_t w2, const Shared*,
                                              uint32_t, const Params&, float (*o)[1][3]) {
    float f[12];
    words_to_rgbf(w0, w1, w2, f);
#pragma unroll
    for (int q = 0; q < 4; ++q) { o[q][0][0] = f[3 * q]; o[q][0][1] = f[3 * q + 1]; o[q][0][2] = f[3 * q + 2]; }
  }
};
using OpSct = OpPoly<MACT_SPACE_SCT>;

// Any subset of {Lab, HSI, SCT} from one read of the pixels (MASK bit 0 =
// Lab, 1 = HSI, 2 = SCT); outputs are packed in that order.  Config 5 runs
// all three, config 2 the HSI + SCT pair (no gamma table, no fp64).
template <int MASK>
struct OpMulti {
  static constexpr bool LAB = MASK & 1, HSI = MASK & 2, SCT = MASK & 4;
  static constexpr int NOUT = LAB + HSI + SCT;
  using Params = KCoeffs;
  struct NoShared { int unused; };
  using Shared = typename std::conditional<LAB, OpLab::Shared, NoShared>::type;
  static __device__ __forceinline__ void init(Shared* s, const Params& c) {
    if constexpr (LAB) OpLab::init(s, c);
  }
  static __device__ __forceinline__ void put(float* o, const Lab3& v) { o[0] = v.c0; o[1] = v.c1; o[2] = v.c2; }
  static __device__ __forceinline__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared* s,
                                            uint32_t lane, const Params& c, float (*o)[3]) {
    int k = 0;
    if constexpr (LAB) put(o[k++], lab_fast_u8(r, g, b, OpLab::tab(s, lane, c), c));
    if constexpr (HSI) put(o[k++], hsi_fast_u8(r, g, b, c));
    if constexpr (SCT) put(o[k++], sct_fast_u8(r, g, b, c));
  }
  static __device__ __forceinline__ void px4w(uint32_t w0, uint32_t w1, uint32_t w2,
                                              const Shared* s, uint32_t lane, const Params& c,
                                              float (*o)[NOUT][3]) {
    if constexpr (LAB) {
      float lab[4][1][3];
      OpLab::px4w(w0, w1, w2, s, lane, c, lab);
#pragma unroll
      for (int q = 0; q < 4; ++q) { o[q][0][0] = lab[q][0][0]; o[q][0][1] = lab[q][0][1]; o[q][0][2] = lab[q][0][2]; }
    }
    float f[12];
    words_to_rgbf(w0, w1, w2, f);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int k = LAB;
      if constexpr (HSI) put(o[q][k++], hsi_fast_f(f[3 * q], f[3 * q + 1], f[3 * q + 2], c));
      if constexpr (SCT) put(o[q][k++], sct_fast_f(f[3 * q], f[3 * q + 1], f[3 * q + 2], c));
    }
  }
};
using OpAll = OpMulti<7>;

// The "exact" transforms in fp32 with libdevice cbrtf / atanf / acosf /
// atan2f / sqrtf on the same streaming skeleton: the B200 comparator of the
// paper's Table 4 gain.  Formulas as exact.py:60-149.
template <int SPACE>
struct OpExactF32 {
  static constexpr int NOUT = 1;
  using Params = KCoeffs;
  struct NoShared { int unused; };
  using Shared = typename std::conditional<SPACE == MACT_SPACE_LAB, OpLab::Shared, NoShared>::type;
  static __device__ __forceinline__ void init(Shared* s, const Params& c) {
    if constexpr (SPACE == MACT_SPACE_LAB) OpLab::init(s, c);
  }
  static __device__ __forceinline__ float lab_f(float t) {
    return t > (float)kLabKnee ? cbrtf(t) : fmaf((float)kLabSlope, t, (float)kLabOffset);
  }
  static __device__ __forceinline__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared* s,
                                            uint32_t lane, const Params& c, float (*o)[3]) {
    if constexpr (SPACE == MACT_SPACE_LAB) {
      const PackedTab t(s->rows, lane);
      const float gr = t.gamma(r), gg = t.gamma(g), gb = t.gamma(b);
      const float fx = lab_f(lab_t(c, 0, gr, gg, gb));
      const float fy = lab_f(lab_t(c, 1, gr, gg, gb));
      const float fz = lab_f(lab_t(c, 2, gr, gg, gb));
      o[0][0] = fmaf(116.f, fy, -16.f);
      o[0][1] = 500.f * (fx - fy);
      o[0][2] = 200.f * (fy - fz);
    } else if constexpr (SPACE == MACT_SPACE_HSI) {
      const float rf = u2f_small(r) * (1.f / 255.f), gf = u2f_small(g) * (1.f / 255.f),
                  bf = u2f_small(b) * (1.f / 255.f);
      const float s3 = 1.7320508f;
      float h;
      if (r > b && g > b) h = (float)(kPi / 3.0) + atanf(s3 * (gf - rf) / ((gf - bf) + (rf - bf)));
      else if (g > r) h = (float)kPi + atanf(s3 * (bf - gf) / ((bf - rf) + (gf - rf)));
      else if (b > g) h = (float)(5.0 * kPi / 3.0) + atanf(s3 * (rf - bf) / ((rf - gf) + (bf - gf)));
      else h = r > b ? 0.f : __int_as_float(0x7fc00000);
      const float total = rf + gf + bf, low = fminf(fminf(rf, gf), bf);
      o[0][0] = h;
      o[0][1] = total > 0.f ? 1.f - 3.f * low / total : 0.f;
      o[0][2] = total * (1.f / 3.f);
    } else {
      const float rf = u2f_small(r), gf = u2f_small(g), bf = u2f_small(b);
      const float len = sqrtf(fmaf(rf, rf, fmaf(gf, gf, bf * bf)));
      o[0][0] = len;
      o[0][1] = len > 0.f ? acosf(fminf(fmaxf(bf / len, -1.f), 1.f)) : 0.f;
      o[0][2] = (r | g) ? atan2f(gf, rf) : __int_as_float(0x7fc00000);
    }
  }
  static __device__ __forceinline__ void px4w(uint32_t w0, uint32_t w1, uint32_t w2, const Shared* s,
                                              uint32_t lane, const Params& c, float (*o)[1][3]) {
    px4_each<OpExactF32>(w0, w1, w2, s, lane, c, o);
  }
};

// Real-valued input, fp64, reference formulas verbatim.
template <typename T>
__global__ void k_fast_real(int space, const T* __restrict__ in, float* __restrict__ out,
                            int64_t n, int planar, const __grid_constant__ KCoeffs c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double r = (double)in[3 * i], g = (double)in[3 * i + 1], b = (double)in[3 * i + 2];
    double o[3];
    if (space == MACT_SPACE_LAB) lab_fast_d(r, g, b, c, o);
    else if (space == MACT_SPACE_HSI) hsi_fast_d(r, g, b, c, o);
    else sct_fast_d(r, g, b, c, o);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (planar) out[k * n + i] = (float)o[k];
      else out[3 * i + k] = (float)o[k];
    }
  }
}

// ------------------------------------------------------------ launchers
// Tile configurations <Op, NW compute warps, G groups/lane, SIN input stages,
// NOB output buffers per warp> (DESIGN.md §Kernels has the smem/occupancy math).
// Overridable at build time for tuning (MACT_NVCC_DEFS, see build.py).
// CIELAB: 16+1 warps, G=4, 2 stages: 176 KB smem (32 KB bank-replicated gamma) -> 1 CTA/SM (R01 sweep: 250 Gpix/s)
#ifndef MACT_DIRECT_N
#define MACT_DIRECT_N (1 << 21)
#endif
#ifndef MACT_LAB_SMALL_N
#define MACT_LAB_SMALL_N (1 << 21)
#endif
#ifndef MACT_LAB_SNW
#define MACT_LAB_SNW 16
#endif
#ifndef MACT_LAB_NW
#define MACT_LAB_NW 16
#endif
#ifndef MACT_LAB_G
#define MACT_LAB_G 4
#endif
#ifndef MACT_LAB_SIN
#define MACT_LAB_SIN 2
#endif
#ifndef MACT_LAB_NOB
#define MACT_LAB_NOB 1
#endif
// HSI: 16+1 warps, G=4, 2 stages: 144 KB -> 1 CTA/SM (R01 sweep: 406 Gpix/s)
#ifndef MACT_HSI_NW
#define MACT_HSI_NW 16
#endif
#ifndef MACT_HSI_G
#define MACT_HSI_G 4
#endif
#ifndef MACT_HSI_SIN
#define MACT_HSI_SIN 2
#endif
#ifndef MACT_HSI_NOB
#define MACT_HSI_NOB 1
#endif
// SCT: 16+1 warps, G=2, 4 stages: 144 KB -> 1 CTA/SM (R01 sweep: 412 Gpix/s)
#ifndef MACT_SCT_NW
#define MACT_SCT_NW 16
#endif
#ifndef MACT_SCT_G
#define MACT_SCT_G 2
#endif
#ifndef MACT_SCT_SIN
#define MACT_SCT_SIN 4
#endif
#ifndef MACT_SCT_NOB
#define MACT_SCT_NOB 2
#endif
// fused triple: 16+1 warps, G=1, 2 stages: 116 KB -> 1 CTA/SM (R01 sweep: 127 G px-triples/s)
#ifndef MACT_ALL_NW
#define MACT_ALL_NW 16
#endif
#ifndef MACT_ALL_G
#define MACT_ALL_G 1
#endif
#ifndef MACT_ALL_SIN
#define MACT_ALL_SIN 8
#endif
#ifndef MACT_ALL_NOB
#define MACT_ALL_NOB 1
#endif
#define MACT_LAB_CFG MACT_LAB_NW, MACT_LAB_G, MACT_LAB_SIN, MACT_LAB_NOB
#define MACT_HSI_CFG MACT_HSI_NW, MACT_HSI_G, MACT_HSI_SIN, MACT_HSI_NOB
#define MACT_SCT_CFG MACT_SCT_NW, MACT_SCT_G, MACT_SCT_SIN, MACT_SCT_NOB
#define MACT_ALL_CFG MACT_ALL_NW, MACT_ALL_G, MACT_ALL_SIN, MACT_ALL_NOB
// HSI + SCT pair (config 2): fp32 only, 27 B/px
#ifndef MACT_HS_NW
#define MACT_HS_NW 16
#endif
#ifndef MACT_HS_G
#define MACT_HS_G 1
#endif
#ifndef MACT_HS_SIN
#define MACT_HS_SIN 4
#endif
#ifndef MACT_HS_NOB
#define MACT_HS_NOB 2
#endif
#define MACT_HS_CFG MACT_HS_NW, MACT_HS_G, MACT_HS_SIN, MACT_HS_NOB

template <typename T>
static int launch_real(int space, const T* in, float* out, int64_t n, int planar,
                       const KCoeffs& kc, cudaStream_t st) {
  if (n <= 0) return MACT_OK;
  int64_t grid = (n + 255) / 256;
  const int64_t cap = 8LL * num_sms();
  if (grid > cap) grid = cap;
  k_fast_real<T><<<(unsigned)grid, 256, 0, st>>>(space, in, out, n, planar, kc);
  count_launch();
  return check_launch("fast_real");
}

static int fast_entry(int space, const void* rgb, int in_dtype, float* out, int64_t n,
                      const MactCoeffs* c, int layout, void* stream) {
  if (n < 0 || (n > 0 && (rgb == nullptr || out == nullptr)) || c == nullptr)
    return set_error(MACT_EBADARG, "bad argument (n=%lld)", (long long)n);
  if (layout != MACT_LAYOUT_INTERLEAVED && layout != MACT_LAYOUT_PLANAR)
    return set_error(MACT_EBADARG, "unknown layout %d", layout);
  KCoeffs kc;
  if (int rc = make_kcoeffs(c, &kc)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int planar = layout == MACT_LAYOUT_PLANAR;
  Outs outs{{out, nullptr, nullptr}};
  const uint8_t* in = (const uint8_t*)rgb;
  // small interleaved HSI / SCT inputs (one image of up to a few Mpx): the
  // direct kernel, whose latency is one DRAM round trip (crossover measured on
  // B200: 2 Mpx).  CIELAB has no direct kernel: its tables must be staged in
  // shared memory (a parameter-bank gather runs at 30 Gpix/s), and with them
  // the small-tile streaming kernel is faster at every size (R01 sweep,
  // scripts/sweep_lab_sizes.py: 512^2 4.5 us vs 5.8 us).
  const bool direct = n < (int64_t)MACT_DIRECT_N && !planar && n % 4 == 0 &&
                      (uintptr_t)in % 16 == 0 && (uintptr_t)out % 16 == 0;
  switch (in_dtype) {
    case MACT_DTYPE_U8:
      if (space == MACT_SPACE_LAB) {
        // images below ~one tile per SM (C1: 512^2 = 32 tiles of 8192) take
        // smaller tiles so the work spreads over more SMs
        if (n < (int64_t)MACT_LAB_SMALL_N)
          return launch_stream_t<OpLab, MACT_LAB_SNW, 1, 2, 1>(in, outs, n, planar, kc, st, "lab_fast");
        return launch_stream_t<OpLab, MACT_LAB_CFG>(in, outs, n, planar, kc, st, "lab_fast");
      }
      if (space == MACT_SPACE_HSI)
        return direct ? launch_direct<OpHsi, 256>(in, outs, n, kc, st, "hsi_fast")
                      : launch_stream_t<OpHsi, MACT_HSI_CFG>(in, outs, n, planar, kc, st, "hsi_fast");
      return direct ? launch_direct<OpSct, 256>(in, outs, n, kc, st, "sct_fast")
                    : launch_stream_t<OpSct, MACT_SCT_CFG>(in, outs, n, planar, kc, st, "sct_fast");
    case MACT_DTYPE_F32:
      return launch_real<float>(space, (const float*)rgb, out, n, planar, kc, st);
    case MACT_DTYPE_F64:
      return launch_real<double>(space, (const double*)rgb, out, n, planar, kc, st);
    default:
      return set_error(MACT_EBADARG, "unsupported input dtype %d", in_dtype);
  }
}

}  // namespace mact

using namespace mact;

extern "C" int mact_lab_fast(const void* rgb, int in_dtype, float* out, int64_t n,
                             const MactCoeffs* c, int layout, void* stream) {
  return fast_entry(MACT_SPACE_LAB, rgb, in_dtype, out, n, c, layout, stream);
}
extern "C" int mact_hsi_fast(const void* rgb, int in_dtype, float* out, int64_t n,
                             const MactCoeffs* c, int layout, void* stream) {
  return fast_entry(MACT_SPACE_HSI, rgb, in_dtype, out, n, c, layout, stream);
}
extern "C" int mact_sct_fast(const void* rgb, int in_dtype, float* out, int64_t n,
                             const MactCoeffs* c, int layout, void* stream) {
  return fast_entry(MACT_SPACE_SCT, rgb, in_dtype, out, n, c, layout, stream);
}
extern "C" int mact_all_fast(const uint8_t* rgb, float* lab, float* hsi, float* sct, int64_t n,
                             const MactCoeffs* c, int layout, void* stream) {
  if (n < 0 || (n > 0 && rgb == nullptr) || c == nullptr)
    return set_error(MACT_EBADARG, "bad argument (n=%lld)", (long long)n);
  if (layout != MACT_LAYOUT_INTERLEAVED && layout != MACT_LAYOUT_PLANAR)
    return set_error(MACT_EBADARG, "unknown layout %d", layout);
  KCoeffs kc;
  if (int rc = make_kcoeffs(c, &kc)) return rc;
  const int mask = (lab != nullptr) | (hsi != nullptr) << 1 | (sct != nullptr) << 2;
  const int planar = layout == MACT_LAYOUT_PLANAR;
  cudaStream_t st = (cudaStream_t)stream;
  switch (mask) {
    case 0: return MACT_OK;
    case 1: return mact_lab_fast(rgb, MACT_DTYPE_U8, lab, n, c, layout, stream);
    case 2: return mact_hsi_fast(rgb, MACT_DTYPE_U8, hsi, n, c, layout, stream);
    case 4: return mact_sct_fast(rgb, MACT_DTYPE_U8, sct, n, c, layout, stream);
    case 3: return launch_stream_t<OpMulti<3>, MACT_ALL_CFG>(rgb, Outs{{lab, hsi, nullptr}}, n, planar, kc, st, "multi_fast");
    case 5: return launch_stream_t<OpMulti<5>, MACT_ALL_CFG>(rgb, Outs{{lab, sct, nullptr}}, n, planar, kc, st, "multi_fast");
    case 6: return launch_stream_t<OpMulti<6>, MACT_HS_CFG>(rgb, Outs{{hsi, sct, nullptr}}, n, planar, kc, st, "multi_fast");
    default: return launch_stream_t<OpAll, MACT_ALL_CFG>(rgb, Outs{{lab, hsi, sct}}, n, planar, kc, st, "all_fast");
  }
}

extern "C" int mact_exact_f32(int space, const uint8_t* rgb, float* out, int64_t n, int layout, void* stream) {
  if (space < 0 || space > 2) return set_error(MACT_EBADARG, "unknown space %d", space);
  if (n < 0 || (n > 0 && (!rgb || !out))) return set_error(MACT_EBADARG, "bad argument");
  if (layout != MACT_LAYOUT_INTERLEAVED && layout != MACT_LAYOUT_PLANAR)
    return set_error(MACT_EBADARG, "unknown layout %d", layout);
  if (n == 0) return MACT_OK;
  KCoeffs kc;
  MactCoeffs dflt{};
  dflt.cbrt_num_deg = dflt.cbrt_den_deg = 2;                // only mxyz is used; any valid degrees
  dflt.hsi_deg = 2; dflt.asin_deg = dflt.acos_deg = dflt.atan_deg = 4;
  dflt.cbrt_den[0] = 1.0;
  if (int rc = make_kcoeffs(&dflt, &kc)) return rc;
  Outs outs{{out, nullptr, nullptr}};
  const int planar = layout == MACT_LAYOUT_PLANAR;
  cudaStream_t st = (cudaStream_t)stream;
  if (space == MACT_SPACE_LAB)
    return launch_stream_t<OpExactF32<MACT_SPACE_LAB>, MACT_LAB_CFG>(rgb, outs, n, planar, kc, st, "exact_f32");
  if (space == MACT_SPACE_HSI)
    return launch_stream_t<OpExactF32<MACT_SPACE_HSI>, MACT_HSI_CFG>(rgb, outs, n, planar, kc, st, "exact_f32");
  return launch_stream_t<OpExactF32<MACT_SPACE_SCT>, MACT_SCT_CFG>(rgb, outs, n, planar, kc, st, "exact_f32");
}

extern "C" int mact_probe_expand(const uint8_t* rgb, float* out, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!rgb || !out))) return set_error(MACT_EBADARG, "bad argument");
  KCoeffs kc{};
  Outs outs{{out, nullptr, nullptr}};
  return launch_stream_t<OpExpand, MACT_HSI_CFG>(rgb, outs, n, 0, kc, (cudaStream_t)stream,
                                                "probe_expand");
}
