// mact_ref.cuh — the MACT fast transforms in the reference's own arithmetic
// (device side of the float64 fidelity mode, shared by mact_ref.cu and the
// fused error reduction): fp64, numpy's operation order, every +, *, /, sqrt
// rounded once (__d*_rn, no FMA contraction), Horner as
// approximants.eval_poly (approximants.py:55-71), the fp64 GAMMA_TABLE for
// 8-bit channels (fast.py:35).  Coefficients come from KCoeffs, whose unused
// high coefficients are zero, which leaves numpy's Horner bit-identical.
#pragma once

#include "mact_common.cuh"

namespace mact {
namespace ref {

static __device__ const double kGammaF64[256] = {
#include "mact_gamma_table64.inc"
};

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
// a / b for a constant divisor with rb = RN(1/b): q = RN(a rb), then one FMA
// correction (Markstein: the residual a - b q is exact and RN(q + r rb) is the
// correctly rounded quotient) -- 3 DP ops instead of the ~10 of a general
// division.  Used where the dividends are the 8-bit domain's (white-point
// division of the linear-light XYZ, /255 and /3 of integer channels), which the
// full-cube fidelity tests check bit for bit; non-finite values take dv.
__device__ __forceinline__ double dv_k(double a, double b, double rb) {
  const double q = __dmul_rn(a, rb);
  const double r = __fma_rn(-q, b, a);
  const double o = __fma_rn(r, rb, q);
  return isfinite(o) ? o : dv(a, b);
}
constexpr double kRcpWhiteX = 1.0 / kWhiteX, kRcpWhiteZ = 1.0 / kWhiteZ;
constexpr double kRcp255 = 1.0 / 255.0, kRcp3 = 1.0 / 3.0;

template <int DEG>
__device__ __forceinline__ double horner(const double* c, double x) {
  double acc = c[DEG];
#pragma unroll
  for (int i = DEG - 1; i >= 0; --i) acc = add(mul(acc, x), c[i]);
  return acc;
}

__device__ __forceinline__ double inverse_gamma(double k) {                // exact.py:52-57
  return k < kGammaKnee ? dv(k, kGammaSlope) : pow(dv(add(k, kGammaOffset), kGammaScale), kGammaPower);
}

__device__ __forceinline__ double lab_f_fast(double t, const KCoeffs& c) {  // fast.py:110-115
  const double den = horner<kCbrtDeg>(c.cbrt_den, t);
  const double q = dv(horner<kCbrtDeg>(c.cbrt_num, t), den);
  return t > kLabKnee ? q : add(mul(kLabSlope, t), kLabOffset);
}

__device__ __forceinline__ double atan_sqrt3(double x, const KCoeffs& c) {  // fast.py:118-122
  const double mag = horner<kPolyDeg>(c.hsi_d, fabs(x));
  return x < 0.0 ? -mag : mag;
}

__device__ __forceinline__ double acos_fast(double x, const KCoeffs& c) {   // fast.py:151-162
  const double d = sub(1.0, x);
  const double m = d != d ? d : (d > 0.0 ? d : 0.0);                       // np.maximum
  return x < 0.5 ? horner<kPolyDeg>(c.acos_d, x) : horner<kPolyDeg>(c.asin_d, __dsqrt_rn(m));
}

__device__ __forceinline__ double atan_unit(double g, double r, const KCoeffs& c) {  // fast.py:165-185
  double out;
  if (g < r) out = horner<kPolyDeg>(c.atanf_d, dv(g, r > 0.0 ? r : 1.0));
  else out = horner<kPolyDeg>(c.atang_d, g > 0.0 ? dv(r, g) : 0.0);
  return (g == 0.0 && r == 0.0) ? __longlong_as_double(0x7ff8000000000000ll) : out;
}

// fast.py:86-107 from linear-light channels
__device__ __forceinline__ void lab_fast(double r, double g, double b, const KCoeffs& c, double* o) {
  const double x = add(add(mul(rgb2xyz(0, 0), r), mul(rgb2xyz(0, 1), g)), mul(rgb2xyz(0, 2), b));
  const double y = add(add(mul(rgb2xyz(1, 0), r), mul(rgb2xyz(1, 1), g)), mul(rgb2xyz(1, 2), b));
  const double z = add(add(mul(rgb2xyz(2, 0), r), mul(rgb2xyz(2, 1), g)), mul(rgb2xyz(2, 2), b));
  static_assert(kWhiteY == 1.0, "y / Yw is y");
  const double fx = lab_f_fast(dv_k(x, kWhiteX, kRcpWhiteX), c), fy = lab_f_fast(y, c),
               fz = lab_f_fast(dv_k(z, kWhiteZ, kRcpWhiteZ), c);
  o[0] = sub(mul(116.0, fy), 16.0);
  o[1] = mul(500.0, sub(fx, fy));
  o[2] = mul(200.0, sub(fy, fz));
}

// fast.py:125-148 on raw channel values (0..255); U8: integer channels (the
// constant divisions take dv_k, checked on all 2^24 colours)
template <bool U8 = false>
__device__ __forceinline__ void hsi_fast(double r, double g, double b, const KCoeffs& c, double* o) {
  auto dvc = [](double a, double d, double rd) { return U8 ? dv_k(a, d, rd) : dv(a, d); };
  r = dvc(r, 255.0, kRcp255); g = dvc(g, 255.0, kRcp255); b = dvc(b, 255.0, kRcp255);
  const bool c1 = (r > b) && (g > b);
  const bool c2 = !c1 && (g > r);
  const bool c3 = !c1 && !c2 && (b > g);
  const bool c4 = !c1 && !c2 && !c3 && (r > b);
  const double num = c1 ? sub(g, r) : c2 ? sub(b, g) : c3 ? sub(r, b) : 0.0;
  const double den = c1 ? add(sub(g, b), sub(r, b)) : c2 ? add(sub(b, r), sub(g, r))
                   : c3 ? add(sub(r, g), sub(b, g)) : 1.0;
  const double base = c1 ? kPi / 3.0 : c2 ? kPi : c3 ? 5.0 * kPi / 3.0 : 0.0;
  double h = add(base, atan_sqrt3(dv(num, den), c));
  h = (c1 || c2 || c3) ? h : (c4 ? 0.0 : __longlong_as_double(0x7ff8000000000000ll));
  h = h < 0.0 ? add(h, kTwoPi) : h;
  h = h >= kTwoPi ? sub(h, kTwoPi) : h;
  const double total = add(add(r, g), b);                             // exact.py:95-101
  const double low = fmin(fmin(r, g), b);
  o[0] = h;
  o[1] = total > 0.0 ? sub(1.0, dv(mul(3.0, low), total)) : 0.0;
  o[2] = dvc(total, 3.0, kRcp3);
}

// fast.py:188-203 on raw channel values
__device__ __forceinline__ void sct_fast(double r, double g, double b, const KCoeffs& c, double* o) {
  const double len = __dsqrt_rn(add(add(mul(r, r), mul(g, g)), mul(b, b)));
  double a = len > 0.0 ? acos_fast(dv(b, len), c) : 0.0;
  double bb = atan_unit(g, r, c);
  a = fmin(fmax(a, 0.0), 0.5 * kPi);                                  // np.clip (finite here)
  if (!(bb != bb)) bb = fmin(fmax(bb, 0.0), 0.5 * kPi);               // NaN kept (fast.py:201-202)
  o[0] = len; o[1] = a; o[2] = bb;
}

}  // namespace ref
}  // namespace mact
