// mact_pixel.cuh — per-pixel device functions of the MACT path.
//
//   lab_fast_u8  <- fast.rgb_to_lab_fast integer path   (fast.py:86-115)
//   hsi_fast_u8  <- fast.rgb_to_hsi_fast                 (fast.py:118-148)
//   sct_fast_u8  <- fast.rgb_to_sct_fast                 (fast.py:151-203)
//   *_fast_d     <- the same functions on real-valued channels, fp64
//   *_exact_d    <- exact.rgb_to_*_exact                 (exact.py:52-149)
//   distances    <- exact.{lab,hsi}_distance, sct_distance_indirect (exact.py:163-190)
//
// Precision design:
//  * HSI and SCT run in fp32 with every branch predicate and every
//    numerator/denominator formed in exact integer arithmetic, so case
//    selection is bit-identical to the reference's fp64 compares.
//  * SCT's folded-arcsin argument uses the cancellation-free
//    1 - b/L = (r^2+g^2) / (L (L+b))  (H2).
//  * CIELAB: fp32 gamma table + fp32 3x3 (white folded in), then the rational
//    P/Q as a segmented fp32 cubic whose (hi, small part) split survives into
//    the a*, b* differences, so that 500 (fx - fy) does not amplify fp32
//    rounding (H1).  Configurations whose segment fit fails the host check
//    keep the fp64 evaluation (monic q = D'/Q' for (4,4), P/Q otherwise).
#pragma once

#include "mact_common.cuh"

namespace mact {

// ---------------------------------------------------------------- gamma
// inverse_gamma(i/255) exactly as exact.py:52-57 (fp64 pow).
__device__ __forceinline__ double inverse_gamma_d(double k) {
  return k < kGammaKnee ? k / kGammaSlope : pow((k + kGammaOffset) / kGammaScale, kGammaPower);
}

// -------------------------------------------------------------- CIELAB fast
__device__ __forceinline__ double rcp_approx_d(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// Lightness kernel f(t) (fast.py:110-115): t is the fp32 X/Xn, Y/Yn or Z/Zn.
// The rational P/Q is evaluated in fp64 Horner (approximants.py:55-82) and
// divided with MUFU.RCP64H + one Newton correction of the quotient
// (q1 = q0 + (P - q0 Q) y0, relative error ~e0^2), all in fp64, so f keeps
// ~1e-12 relative accuracy for the 500 (fx - fy) amplification (H1).
__device__ __forceinline__ double lab_f_fast(float t, const KCoeffs& c) {
  const double td = (double)t;                       // F2F on the XU pipe (1 issue slot)
  const double P = horner_d<kCbrtDeg>(c.cbrt_num, td);
  const double Q = horner_d<kCbrtDeg>(c.cbrt_den, td);
  const double y0 = rcp_approx_d(Q);
  const double q0 = P * y0;
  double f = fma(fma(-q0, Q, P), y0, q0);
  if (!(t > (float)kLabKnee)) f = fma(kLabSlope, td, kLabOffset);   // strict '>' (fast.py:114)
  return f;
}

struct Lab3 {
  float c0, c1, c2;
};

// Batched 4-pixel CIELAB for the default (4,4) rational in monic form.
// One warp vote decides whether any lane of the warp has a channel on the
// linear branch (t <= knee: ~0.04-0.3 % of colours per channel); only then
// is the linear value computed, so the common path has no selects.
// fp32 -> fp64 widening of t: F2F on the XU pipe costs 1 issue slot against 2
// for the ALU bit move (f2d_pos); the XU has headroom here (+2.5 % measured).
#ifndef MACT_T2D
#define MACT_T2D(x) ((double)(x))
#endif
__device__ __forceinline__ double monic4(const double* cm, double t) {
  double acc = t + cm[3];
  acc = fma(acc, t, cm[2]);
  acc = fma(acc, t, cm[1]);
  return fma(acc, t, cm[0]);
}
__device__ __forceinline__ double monic3(const double* cm, double t) {
  double acc = t + cm[2];
  acc = fma(acc, t, cm[1]);
  return fma(acc, t, cm[0]);
}
// q = D'(t)/Q'(t): MUFU.RCP64H seed + one fp64 Newton correction of the quotient.
__device__ __forceinline__ double lab_q(double td, const KCoeffs& c) {
  const double D = monic3(c.dm, td), Q = monic4(c.qm, td);
  const double y0 = rcp_approx_d(Q);
  const double q0 = D * y0;
  return fma(fma(-q0, Q, D), y0, q0);
}
__device__ __forceinline__ double lab_q_sel(float t, const KCoeffs& c) {
  return t > (float)kLabKnee ? lab_q(MACT_T2D(t), c) : fma(c.lin_s, (double)t, c.lin_o);
}
// CIELAB epilogue from the three q's: L* in fp64 (its two terms nearly cancel),
// a*, b* from an fp64 difference rounded once to fp32.
__device__ __forceinline__ void lab_from_q(double qx, double qy, double qz, const KCoeffs& c,
                                           float& L, float& A, float& B) {
  L = (float)fma(c.l_s, qy, c.l_o);
  A = c.a_s * (float)(qx - qy);
  B = c.b_s * (float)(qy - qz);
}

// ------------------------------------------ CIELAB fast, segmented fp32
// The rational R = P/Q as a piecewise cubic on 16 segments per binade of the
// fp32 t (KCoeffs::seg, fitted on the host to ~5e-9): with u = t - t_seg
// (exact: t_seg is t with the bits below the segment index cleared),
//   f = hi + d,   d = u (c1 + u (c2 + u c3)),
// and the epilogue keeps hi and d apart,
//   a* = 500 ((hx - hy) + (dx - dy)),  b* = 200 ((hy - hz) + (dy - dz)),
// so the 500x amplification of a* sees the rounding of the small parts d
// only (the hi differences are exact or rounded relative to the result).
// All fp32: no fp64 pipe, no XU.  Full-cube error vs the reference:
// 1.5e-5 / 5.6e-5 / 2.5e-5 on L*, a*, b* (tolerance 1e-4).
//
// Where the two tables (fp32 GAMMA_TABLE, segment table) are read from is a
// policy, so every kernel runs the same arithmetic:
//  * SmemTab<COPIES>: staged in shared memory; gamma replicated 32x (entry i
//    of lane l at float [i*32 + l], conflict-free), segment table in COPIES
//    bank-private copies (entry i of copy k at float4 [i*COPIES + k]);
//    addressed with 32-bit shared addresses off the lane's base.  The error
//    reduction kernel (static smem).
//  (A policy reading the segment entries straight from the parameter bank
//  -- no staging -- was measured at 30 Gpix/s: divergent constant-bank
//  gathers serialise.)
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
//  * PackedTab: both tables in ONE 64 KB block aligned to 64 KB in the
//    shared window, rows of 256 B: row r holds gamma entry r for the 32 lanes
//    in its first 128 B, and (rows 0..127) the 8 copies of segment entry r in
//    its last 128 B.  The gamma address of byte k of an input word is then
//    one PRMT (the byte lands in address bits 8..15 of the lane's base), and
//    the segment address of t one SHF + LOP3 (no clamp: t < 2^-7 wraps onto a
//    row the linear branch overrides).  The streaming CIELAB kernels.
template <int COPIES>
struct SmemTab {
  uint32_t gl, sa;   // gamma + lane*4, seg + (lane % COPIES)*16 (shared addresses)
  __device__ __forceinline__ SmemTab(const float* gamma_rep, const float4* seg, uint32_t lane)
      : gl(smem_u32(gamma_rep) + lane * 4), sa(smem_u32(seg) + (lane & (COPIES - 1)) * 16) {}
  __device__ __forceinline__ float gamma(uint32_t v) const { return lds_f32(gl + (v << 7)); }
  __device__ __forceinline__ float gamma_w(uint32_t w, int k) const { return gamma(byte_of(w, k)); }
  __device__ __forceinline__ float4 seg_t(uint32_t b) const {
    const uint32_t i = min((b >> kLabSegShift) - kLabSegBase, (uint32_t)(kLabSegs - 1));
    return lds_f32x4(sa + i * (COPIES * 16));
  }
};
struct PackedTab {
  static constexpr uint32_t kBytes = 65536;
  uint32_t gl, sa;   // table + lane*4, table + 128 + (lane % 8)*16 (shared addresses, table % 64K == 0)
  __device__ __forceinline__ PackedTab(const void* table, uint32_t lane)
      : gl(smem_u32(table) + lane * 4), sa(smem_u32(table) + 128 + (lane & 7) * 16) {}
  __device__ __forceinline__ float gamma(uint32_t v) const { return lds_f32(gl + (v << 8)); }
  __device__ __forceinline__ float gamma_w(uint32_t w, int k) const {
    return lds_f32(__byte_perm(w, gl, 0x7604u | ((uint32_t)k << 4)));
  }
  __device__ __forceinline__ float4 seg_t(uint32_t b) const {
    static_assert((kLabSegBase & 127u) == 0 && kLabSegs <= 128, "segment rows wrap mod 128");
    return lds_f32x4(((b >> (kLabSegShift - 8)) & 0x7F00u) | sa);
  }
};

template <class Tab>
__device__ __forceinline__ void lab_seg(float t, const Tab& tab, float& h, float& d) {
  const uint32_t b = __float_as_uint(t);
  const float4 e = tab.seg_t(b);
  const float u = t - __uint_as_float(b & kLabSegMask);
  h = e.x;
  d = u * fmaf(u, fmaf(u, e.w, e.z), e.y);
}
__device__ __forceinline__ void lab_seg_lin(float t, const KCoeffs& c, float& h, float& d) {
  h = c.lin_hi;
  d = fmaf(c.lin_slope, t, c.lin_lo);          // strict '>' keeps t = knee linear (fast.py:114)
}
__device__ __forceinline__ void lab_from_seg(float hx, float dx, float hy, float dy, float hz,
                                             float dz, float& L, float& A, float& B) {
  L = fmaf(116.f, dy, fmaf(116.f, hy, -16.f));
  A = 500.f * ((hx - hy) + (dx - dy));
  B = 200.f * ((hy - hz) + (dy - dz));
}
__device__ __forceinline__ float lab_t(const KCoeffs&, int row, float gr, float gg, float gb) {
  return fmaf(kMxyz(row, 2), gb, fmaf(kMxyz(row, 1), gg, kMxyz(row, 0) * gr));
}

// One pixel (tails, unaligned buffers, the fused error reduction).
template <class Tab>
__device__ __forceinline__ Lab3 lab_fast_u8(uint32_t r, uint32_t g, uint32_t b, const Tab& tab,
                                            const KCoeffs& c) {
  const float gr = tab.gamma(r), gg = tab.gamma(g), gb = tab.gamma(b);
  const float tx = lab_t(c, 0, gr, gg, gb), ty = lab_t(c, 1, gr, gg, gb), tz = lab_t(c, 2, gr, gg, gb);
  Lab3 o;
  if (c.lab_seg) {   // same arithmetic as lab_fast_u8x4 (bit-identical tile/tail paths)
    float h[3], d[3];
    const float t[3] = {tx, ty, tz};
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if (t[j] > (float)kLabKnee) lab_seg(t[j], tab, h[j], d[j]);
      else lab_seg_lin(t[j], c, h[j], d[j]);
    }
    lab_from_seg(h[0], d[0], h[1], d[1], h[2], d[2], o.c0, o.c1, o.c2);
    return o;
  }
  if (c.monic44) {   // same arithmetic as lab_fast_u8x4 (bit-identical tile/tail paths)
    lab_from_q(lab_q_sel(tx, c), lab_q_sel(ty, c), lab_q_sel(tz, c), c, o.c0, o.c1, o.c2);
    return o;
  }
  const double fx = lab_f_fast(tx, c), fy = lab_f_fast(ty, c), fz = lab_f_fast(tz, c);
  o.c0 = (float)fma(116.0, fy, -16.0);
  o.c1 = (float)(500.0 * (fx - fy));
  o.c2 = (float)(200.0 * (fy - fz));
  return o;
}

// 4 pixels (12 channels) per call, warp-converged.  Configurations that are
// neither segmented nor monic (4,4) take lab_fast_u8 per pixel (caller).
template <class Tab>
__device__ __forceinline__ void lab_fast_u8x4(uint32_t w0, uint32_t w1, uint32_t w2, const Tab& tab,
                                              const KCoeffs& c, float (*o)[3]) {
  float t[12];
  bool low = false;
  const uint32_t w[3] = {w0, w1, w2};
#pragma unroll
  for (int p = 0; p < 4; ++p) {   // channel j = 3p + q is byte j % 4 of word j / 4
    const float gr = tab.gamma_w(w[(3 * p) >> 2], (3 * p) & 3);
    const float gg = tab.gamma_w(w[(3 * p + 1) >> 2], (3 * p + 1) & 3);
    const float gb = tab.gamma_w(w[(3 * p + 2) >> 2], (3 * p + 2) & 3);
    t[3 * p] = lab_t(c, 0, gr, gg, gb);
    t[3 * p + 1] = lab_t(c, 1, gr, gg, gb);
    t[3 * p + 2] = lab_t(c, 2, gr, gg, gb);
  }
#pragma unroll
  for (int j = 0; j < 12; ++j) low |= !(t[j] > (float)kLabKnee);
  if (c.lab_seg) {
    float h[12], d[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) lab_seg(t[j], tab, h[j], d[j]);
    if (__any_sync(0xffffffffu, low)) {
#pragma unroll
      for (int j = 0; j < 12; ++j)
        if (!(t[j] > (float)kLabKnee)) lab_seg_lin(t[j], c, h[j], d[j]);
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
      lab_from_seg(h[3 * p], d[3 * p], h[3 * p + 1], d[3 * p + 1], h[3 * p + 2], d[3 * p + 2],
                   o[p][0], o[p][1], o[p][2]);
    return;
  }
  double q[12];
#pragma unroll
  for (int j = 0; j < 12; ++j) q[j] = lab_q(MACT_T2D(t[j]), c);
  if (__any_sync(0xffffffffu, low)) {
#pragma unroll
    for (int j = 0; j < 12; ++j)
      if (!(t[j] > (float)kLabKnee)) q[j] = fma(c.lin_s, (double)t[j], c.lin_o);
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
    lab_from_q(q[3 * p], q[3 * p + 1], q[3 * p + 2], c, o[p][0], o[p][1], o[p][2]);
}

// Reference-faithful fp64 evaluation on real-valued channels (float input
// path, fast.py:96-115), used for non-uint8 inputs.
__device__ __forceinline__ double lab_f_fast_d(double t, const KCoeffs& c) {
  const double P = horner_d<kCbrtDeg>(c.cbrt_num, t);
  const double Q = horner_d<kCbrtDeg>(c.cbrt_den, t);
  return t > kLabKnee ? P / Q : kLabSlope * t + kLabOffset;
}
__device__ __forceinline__ void lab_fast_d(double r, double g, double b, const KCoeffs& c,
                                           double* o) {
  const double gr = inverse_gamma_d(r / 255.0), gg = inverse_gamma_d(g / 255.0),
               gb = inverse_gamma_d(b / 255.0);
  const double x = rgb2xyz(0, 0) * gr + rgb2xyz(0, 1) * gg + rgb2xyz(0, 2) * gb;
  const double y = rgb2xyz(1, 0) * gr + rgb2xyz(1, 1) * gg + rgb2xyz(1, 2) * gb;
  const double z = rgb2xyz(2, 0) * gr + rgb2xyz(2, 1) * gg + rgb2xyz(2, 2) * gb;
  const double fx = lab_f_fast_d(x / kWhiteX, c), fy = lab_f_fast_d(y / kWhiteY, c),
               fz = lab_f_fast_d(z / kWhiteZ, c);
  o[0] = 116.0 * fy - 16.0;
  o[1] = 500.0 * (fx - fy);
  o[2] = 200.0 * (fy - fz);
}

// ----------------------------------------------------------------- HSI fast
// Kender case analysis (fast.py:131-146).  Channels arrive as exact
// integer-valued floats (0..255), so every compare, sum and difference below
// is exact and the case selection is bit-identical to the reference's fp64
// compares on r/255 etc.  Identities used (all exact on integers):
//   case1 (b strictly smallest)  <=>  b < min(r, g)
//   den of the active case = (sum of the other two) - 2 min = sum - 3 min
//   S = 1 - 3 min / sum = den / sum            (exact.py:95-101)
//   not case1..3  =>  g = b <= r, so case4 (h = 0) <=> den > 0, gray <=> den = 0
__device__ __forceinline__ Lab3 hsi_fast_f(float r, float g, float b, const KCoeffs& c) {
  const float mrg = fminf(r, g);
  const bool c1 = b < mrg;
  const bool c2 = !c1 & (g > r);
  const bool c3 = !c1 & !c2 & (b > g);
  const float sum = r + g + b;
  const float den = fmaf(-3.0f, fminf(mrg, b), sum);
  const float num = c1 ? g - r : (c2 ? b - g : r - b);
  const float base = c1 ? (float)(kPi / 3.0) : (c2 ? (float)kPi : (float)(5.0 * kPi / 3.0));
  const float x = num * rcp_approx(den);
  const float mag = horner_f<kPolyDeg>(c.hsi, fabsf(x));
  float h = base + (num < 0.0f ? -mag : mag);           // odd extension (fast.py:118-122)
  if (h < 0.0f) h += (float)kTwoPi;
  if (h >= (float)kTwoPi) h -= (float)kTwoPi;
  Lab3 o;
  o.c0 = (c1 | c2 | c3) ? h : (den > 0.0f ? 0.0f : __int_as_float(0x7fc00000));
  o.c1 = sum > 0.0f ? den * rcp_approx(sum) : 0.0f;
  o.c2 = sum * (float)(1.0 / 765.0);
  return o;
}

__device__ __forceinline__ double horner_dd(const double* cc, int deg, double x) {
  double acc = cc[deg];
  for (int k = deg - 1; k >= 0; --k) acc = acc * x + cc[k];
  return acc;
}

__device__ __forceinline__ void hsi_fast_d(double r, double g, double b, const KCoeffs& c,
                                           double* o) {
  r /= 255.0; g /= 255.0; b /= 255.0;
  const bool c1 = (r > b) && (g > b);
  const bool c2 = !c1 && (g > r);
  const bool c3 = !c1 && !c2 && (b > g);
  const bool c4 = !c1 && !c2 && !c3 && (r > b);
  double num = 0.0, den = 1.0, base = 0.0;
  if (c1) { num = g - r; den = (g - b) + (r - b); base = kPi / 3.0; }
  else if (c2) { num = b - g; den = (b - r) + (g - r); base = kPi; }
  else if (c3) { num = r - b; den = (r - g) + (b - g); base = 5.0 * kPi / 3.0; }
  const double x = num / den;
  const double mag = horner_dd(c.hsi_d, kPolyDeg, fabs(x));
  double h = base + (x < 0.0 ? -mag : mag);
  h = (c1 || c2 || c3) ? h : (c4 ? 0.0 : __longlong_as_double(0x7ff8000000000000ll));
  if (h < 0.0) h += kTwoPi;
  if (h >= kTwoPi) h -= kTwoPi;
  const double total = r + g + b;
  const double low = fmin(fmin(r, g), b);
  o[0] = h;
  o[1] = total > 0.0 ? 1.0 - 3.0 * low / total : 0.0;
  o[2] = total / 3.0;
}

// ----------------------------------------------------------------- SCT fast
// fast.py:151-203 on exact integer-valued float channels.
//  * |v|^2 = r^2+g^2+b^2 <= 195075 < 2^24 is exact; one MUFU.RSQ gives both
//    L = |v|^2 rsqrt(|v|^2) and b/L = b rsqrt(|v|^2).
//  * arccos branch: b/L >= 0.5 <=> 3 b^2 >= r^2 + g^2 (exact integer test);
//    the folded arcsin argument sqrt(1 - b/L) uses the cancellation-free
//    (r^2+g^2) / (L (L + b)) = (r^2+g^2) / (|v|^2 + b L).
//  * arctan: min(g,r)/max(g,r) with the direct/complement polynomial; both
//    polynomials are evaluated (FMA pipe) and selected, no divergence.
__device__ __forceinline__ Lab3 sct_fast_f(float r, float g, float b, const KCoeffs& c) {
  const float rg2 = fmaf(g, g, r * r);
  const float b2 = b * b;
  const float ss = rg2 + b2;
  const float rs = rsqrt_approx(ss);                    // inf at black, masked below
  const float L = ss * rs;
  // angle A = acos_fast(b / L)
  const bool upper = fmaf(3.0f, b2, -rg2) >= 0.0f;
  const float y = sqrt_approx(rg2 * rcp_approx(fmaf(b, L, ss)));
  const float pa_hi = horner_f<kPolyDeg>(c.asin, y);
  const float pa_lo = horner_f<kPolyDeg>(c.acos, b * rs);
  float ang_a = upper ? pa_hi : pa_lo;
  ang_a = ss > 0.0f ? fminf(fmaxf(ang_a, 0.0f), (float)(0.5 * kPi)) : 0.0f;
  // angle B = atan_unit_fast(g, r)
  const float lo = fminf(g, r), hi = fmaxf(g, r);
  const float t = lo * rcp_approx(hi);
  const float pf = horner_f<kPolyDeg>(c.atanf, t);
  const float pg = horner_f<kPolyDeg>(c.atang, t);
  float ang_b = fminf(fmaxf(g < r ? pf : pg, 0.0f), (float)(0.5 * kPi));
  Lab3 o;
  o.c0 = ss > 0.0f ? L : 0.0f;
  o.c1 = ang_a;
  o.c2 = hi > 0.0f ? ang_b : __int_as_float(0x7fc00000);
  return o;
}

__device__ __forceinline__ Lab3 hsi_fast_u8(uint32_t r, uint32_t g, uint32_t b, const KCoeffs& c) {
  return hsi_fast_f(u2f_small(r), u2f_small(g), u2f_small(b), c);
}
__device__ __forceinline__ Lab3 sct_fast_u8(uint32_t r, uint32_t g, uint32_t b, const KCoeffs& c) {
  return sct_fast_f(u2f_small(r), u2f_small(g), u2f_small(b), c);
}

__device__ __forceinline__ void sct_fast_d(double r, double g, double b, const KCoeffs& c,
                                           double* o) {
  const double len = sqrt(r * r + g * g + b * b);
  double a = 0.0;
  if (len > 0.0) {
    const double x = b / len;
    a = x < 0.5 ? horner_dd(c.acos_d, kPolyDeg, x)
                : horner_dd(c.asin_d, kPolyDeg, sqrt(fmax(1.0 - x, 0.0)));
  }
  double bb;
  if (g == 0.0 && r == 0.0) {
    bb = __longlong_as_double(0x7ff8000000000000ll);
  } else {
    const bool direct = g < r;
    const double arg = direct ? g / (r > 0.0 ? r : 1.0) : (g > 0.0 ? r / g : 0.0);
    bb = direct ? horner_dd(c.atanf_d, kPolyDeg, arg) : horner_dd(c.atang_d, kPolyDeg, arg);
    bb = fmin(fmax(bb, 0.0), 0.5 * kPi);
  }
  o[0] = len;
  o[1] = fmin(fmax(a, 0.0), 0.5 * kPi);
  o[2] = bb;
}

// ------------------------------------------------------------ exact, fp64
__device__ __forceinline__ double lab_f_exact(double t) {
  return t > kLabKnee ? cbrt(t) : kLabSlope * t + kLabOffset;
}
// linear-light channels -> L*a*b* (exact.py:60-83)
__device__ __forceinline__ void lab_from_linear(double gr, double gg, double gb, double* o) {
  const double x = rgb2xyz(0, 0) * gr + rgb2xyz(0, 1) * gg + rgb2xyz(0, 2) * gb;
  const double y = rgb2xyz(1, 0) * gr + rgb2xyz(1, 1) * gg + rgb2xyz(1, 2) * gb;
  const double z = rgb2xyz(2, 0) * gr + rgb2xyz(2, 1) * gg + rgb2xyz(2, 2) * gb;
  const double fx = lab_f_exact(x / kWhiteX), fy = lab_f_exact(y / kWhiteY),
               fz = lab_f_exact(z / kWhiteZ);
  o[0] = 116.0 * fy - 16.0;
  o[1] = 500.0 * (fx - fy);
  o[2] = 200.0 * (fy - fz);
}
__device__ __forceinline__ void lab_exact_d(double r, double g, double b, double* o) {
  lab_from_linear(inverse_gamma_d(r / 255.0), inverse_gamma_d(g / 255.0),
                  inverse_gamma_d(b / 255.0), o);
}
__device__ __forceinline__ void hsi_exact_d(double r, double g, double b, double* o) {
  r /= 255.0; g /= 255.0; b /= 255.0;
  const double s3 = 1.7320508075688772;       // np.sqrt(3.0)
  const bool c1 = (r > b) && (g > b);
  const bool c2 = !c1 && (g > r);
  const bool c3 = !c1 && !c2 && (b > g);
  const bool c4 = !c1 && !c2 && !c3 && (r > b);
  double h;
  if (c1) h = kPi / 3.0 + atan(s3 * (g - r) / ((g - b) + (r - b)));
  else if (c2) h = kPi + atan(s3 * (b - g) / ((b - r) + (g - r)));
  else if (c3) h = 5.0 * kPi / 3.0 + atan(s3 * (r - b) / ((r - g) + (b - g)));
  else h = c4 ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
  const double total = r + g + b;
  const double low = fmin(fmin(r, g), b);
  o[0] = h;
  o[1] = total > 0.0 ? 1.0 - 3.0 * low / total : 0.0;
  o[2] = total / 3.0;
}
// exact.rgb_to_hsi_arccos (exact.py:104-116): inverse-cosine hue formula.
__device__ __forceinline__ void hsi_arccos_d(double r, double g, double b, double* o) {
  r /= 255.0; g /= 255.0; b /= 255.0;
  const double num = 0.5 * ((r - g) + (r - b));
  const double den_sq = (r - g) * (r - g) + (r - b) * (g - b);
  const double ratio = num / sqrt(den_sq);
  double h = acos(fmin(fmax(ratio, -1.0), 1.0));
  if (b > g) h = kTwoPi - h;
  if (!(den_sq > 0.0)) h = __longlong_as_double(0x7ff8000000000000ll);
  const double total = r + g + b;
  const double low = fmin(fmin(r, g), b);
  o[0] = h;
  o[1] = total > 0.0 ? 1.0 - 3.0 * low / total : 0.0;
  o[2] = total / 3.0;
}
__device__ __forceinline__ void sct_exact_d(double r, double g, double b, double* o) {
  const double len = sqrt(r * r + g * g + b * b);
  o[0] = len;
  o[1] = len > 0.0 ? acos(fmin(fmax(b / len, -1.0), 1.0)) : 0.0;
  o[2] = (r == 0.0 && g == 0.0) ? __longlong_as_double(0x7ff8000000000000ll) : atan2(g, r);
}

// --------------------------------------------------------------- distances
__device__ __forceinline__ double lab_distance_d(const double* x, const double* y) {
  const double d0 = x[0] - y[0], d1 = x[1] - y[1], d2 = x[2] - y[2];
  return sqrt(d0 * d0 + d1 * d1 + d2 * d2);
}
__device__ __forceinline__ double hsi_distance_d(const double* x, const double* y) {
  const double hx = isnan(x[0]) ? 0.0 : x[0], hy = isnan(y[0]) ? 0.0 : y[0];
  double th = fabs(hx - hy);
  th = th > kPi ? kTwoPi - th : th;
  const double di = x[2] - y[2];
  const double d2 = x[1] * x[1] + y[1] * y[1] - 2.0 * x[1] * y[1] * cos(th) + di * di;
  return sqrt(fmax(d2, 0.0));
}
__device__ __forceinline__ void sct_to_rgb_d(const double* s, double* rgb) {
  const double bb = isnan(s[2]) ? 0.0 : s[2];
  double sa, ca, sb, cb;
  sincos(s[1], &sa, &ca);
  sincos(bb, &sb, &cb);
  rgb[0] = s[0] * sa * cb;
  rgb[1] = s[0] * sa * sb;
  rgb[2] = s[0] * ca;
}
__device__ __forceinline__ double sct_distance_d(const double* x, const double* y) {
  double rx[3], ry[3], lx[3], ly[3];
  sct_to_rgb_d(x, rx);
  sct_to_rgb_d(y, ry);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    rx[k] = fmin(fmax(rx[k], 0.0), 255.0);
    ry[k] = fmin(fmax(ry[k], 0.0), 255.0);
  }
  lab_exact_d(rx[0], rx[1], rx[2], lx);
  lab_exact_d(ry[0], ry[1], ry[2], ly);
  return lab_distance_d(lx, ly);
}
__device__ __forceinline__ double distance_d(int space, const double* x, const double* y) {
  return space == MACT_SPACE_LAB ? lab_distance_d(x, y)
       : space == MACT_SPACE_HSI ? hsi_distance_d(x, y)
                                 : sct_distance_d(x, y);
}

}  // namespace mact
