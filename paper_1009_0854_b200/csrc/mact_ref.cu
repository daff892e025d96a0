// mact_ref.cu — the MACT fast transforms evaluated exactly as the reference
// evaluates them: fp64, numpy's operation order, every +, *, /, sqrt rounded
// once (__d*_rn, no FMA contraction), Horner as approximants.eval_poly
// (approximants.py:55-71), the fp64 GAMMA_TABLE for 8-bit channels
// (fast.py:35).  For uint8 pixels the results are bit-identical to
// mact.fast.rgb_to_{lab,hsi,sct}_fast (fast.py:86-203); real-valued Lab
// inputs go through libdevice pow in inverse_gamma (within an ulp of libm),
// real HSI / SCT inputs stay bit-identical.
//
// This is the fidelity mode (out_dtype float64, 24 B/px out): the throughput
// path is mact_{lab,hsi,sct}_fast with fp32 outputs.
#include "mact_common.cuh"

namespace mact {

__device__ const double kGammaF64[256] = {
#include "mact_gamma_table64.inc"
};

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ double horner_np(const double* c, int deg, double x) {
  double acc = c[deg];
  for (int i = deg - 1; i >= 0; --i) acc = add(mul(acc, x), c[i]);
  return acc;
}

struct RefParams {
  double num[8], den[8], hsi[8], asin[8], acos[8], atanf[8], atang[8];
  int num_deg, den_deg, hsi_deg, asin_deg, acos_deg, atan_deg;
};

template <typename TI>
__device__ __forceinline__ double chan(const TI* p, int64_t i) { return (double)p[i]; }

// exact.inverse_gamma (exact.py:52-57): uint8 channels read the table, real ones evaluate it
template <typename TI>
__device__ __forceinline__ double lin(const TI* p, int64_t i) {
  if constexpr (sizeof(TI) == 1) {
    return kGammaF64[p[i]];
  } else {
    const double k = dv(chan(p, i), 255.0);
    return k < kGammaKnee ? dv(k, kGammaSlope) : pow(dv(add(k, kGammaOffset), kGammaScale), kGammaPower);
  }
}

__device__ __forceinline__ double lab_f_fast_np(double t, const RefParams& c) {   // fast.py:110-115
  const double den = horner_np(c.den, c.den_deg, t);
  const double q = dv(horner_np(c.num, c.num_deg, t), den);
  return t > kLabKnee ? q : add(mul(kLabSlope, t), kLabOffset);
}

__device__ __forceinline__ double atan_sqrt3_np(double x, const RefParams& c) {   // fast.py:118-122
  const double mag = horner_np(c.hsi, c.hsi_deg, fabs(x));
  return x < 0.0 ? -mag : mag;
}

__device__ __forceinline__ double acos_np(double x, const RefParams& c) {         // fast.py:151-162
  const double d = sub(1.0, x);
  const double m = d != d ? d : (d > 0.0 ? d : 0.0);                               // np.maximum
  return x < 0.5 ? horner_np(c.acos, c.acos_deg, x) : horner_np(c.asin, c.asin_deg, __dsqrt_rn(m));
}

__device__ __forceinline__ double atan_unit_np(double g, double r, const RefParams& c) {  // fast.py:165-185
  double out;
  if (g < r) out = horner_np(c.atanf, c.atan_deg, dv(g, r > 0.0 ? r : 1.0));
  else out = horner_np(c.atang, c.atan_deg, g > 0.0 ? dv(r, g) : 0.0);
  return (g == 0.0 && r == 0.0) ? __longlong_as_double(0x7ff8000000000000ll) : out;
}

template <int SPACE, typename TI>
__global__ void k_fast_ref(const __grid_constant__ RefParams c, const TI* __restrict__ in,
                           double* __restrict__ out, int64_t n, int planar) {
  const double kNaN = __longlong_as_double(0x7ff8000000000000ll);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double o0, o1, o2;
    if constexpr (SPACE == MACT_SPACE_LAB) {                       // fast.py:86-107
      const double r = lin(in, 3 * i), g = lin(in, 3 * i + 1), b = lin(in, 3 * i + 2);
      const double x = add(add(mul(rgb2xyz(0, 0), r), mul(rgb2xyz(0, 1), g)), mul(rgb2xyz(0, 2), b));
      const double y = add(add(mul(rgb2xyz(1, 0), r), mul(rgb2xyz(1, 1), g)), mul(rgb2xyz(1, 2), b));
      const double z = add(add(mul(rgb2xyz(2, 0), r), mul(rgb2xyz(2, 1), g)), mul(rgb2xyz(2, 2), b));
      const double fx = lab_f_fast_np(dv(x, kWhiteX), c), fy = lab_f_fast_np(dv(y, kWhiteY), c),
                   fz = lab_f_fast_np(dv(z, kWhiteZ), c);
      o0 = sub(mul(116.0, fy), 16.0);
      o1 = mul(500.0, sub(fx, fy));
      o2 = mul(200.0, sub(fy, fz));
    } else if constexpr (SPACE == MACT_SPACE_HSI) {                // fast.py:125-148
      const double r = dv(chan(in, 3 * i), 255.0), g = dv(chan(in, 3 * i + 1), 255.0),
                   b = dv(chan(in, 3 * i + 2), 255.0);
      const bool c1 = (r > b) && (g > b);
      const bool c2 = !c1 && (g > r);
      const bool c3 = !c1 && !c2 && (b > g);
      const bool c4 = !c1 && !c2 && !c3 && (r > b);
      const double num = c1 ? sub(g, r) : c2 ? sub(b, g) : c3 ? sub(r, b) : 0.0;
      const double den = c1 ? add(sub(g, b), sub(r, b)) : c2 ? add(sub(b, r), sub(g, r))
                       : c3 ? add(sub(r, g), sub(b, g)) : 1.0;
      const double base = c1 ? kPi / 3.0 : c2 ? kPi : c3 ? 5.0 * kPi / 3.0 : 0.0;
      double h = add(base, atan_sqrt3_np(dv(num, den), c));
      h = (c1 || c2 || c3) ? h : (c4 ? 0.0 : kNaN);
      h = h < 0.0 ? add(h, kTwoPi) : h;
      h = h >= kTwoPi ? sub(h, kTwoPi) : h;
      const double total = add(add(r, g), b);                       // exact.py:95-101
      const double low = fmin(fmin(r, g), b);
      o0 = h;
      o1 = total > 0.0 ? sub(1.0, dv(mul(3.0, low), total)) : 0.0;
      o2 = dv(total, 3.0);
    } else {                                                        // fast.py:188-203
      const double r = chan(in, 3 * i), g = chan(in, 3 * i + 1), b = chan(in, 3 * i + 2);
      const double len = __dsqrt_rn(add(add(mul(r, r), mul(g, g)), mul(b, b)));
      double a = len > 0.0 ? acos_np(dv(b, len), c) : 0.0;
      double bb = atan_unit_np(g, r, c);
      a = fmin(fmax(a, 0.0), 0.5 * kPi);                           // np.clip (a is never NaN here
      if (!(bb != bb)) bb = fmin(fmax(bb, 0.0), 0.5 * kPi);        //  for finite pixels)
      o0 = len; o1 = a; o2 = bb;
    }
    if (planar) {
      out[i] = o0; out[n + i] = o1; out[2 * n + i] = o2;
    } else {
      out[3 * i] = o0; out[3 * i + 1] = o1; out[3 * i + 2] = o2;
    }
  }
}

template <int SPACE, typename TI>
static int launch_ref(const RefParams& p, const TI* in, double* out, int64_t n, int planar, cudaStream_t st) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = 8LL * num_sms();
  if (g > cap) g = cap;
  k_fast_ref<SPACE, TI><<<(unsigned)g, 256, 0, st>>>(p, in, out, n, planar);
  count_launch();
  return check_launch("fast_f64");
}

template <typename TI>
static int ref_space(int space, const RefParams& p, const TI* in, double* out, int64_t n, int planar,
                     cudaStream_t st) {
  if (space == MACT_SPACE_LAB) return launch_ref<MACT_SPACE_LAB>(p, in, out, n, planar, st);
  if (space == MACT_SPACE_HSI) return launch_ref<MACT_SPACE_HSI>(p, in, out, n, planar, st);
  return launch_ref<MACT_SPACE_SCT>(p, in, out, n, planar, st);
}

}  // namespace mact

using namespace mact;

extern "C" int mact_fast_f64(int space, const void* rgb, int in_dtype, double* out, int64_t n,
                             const MactCoeffs* c, int layout, void* stream) {
  if (space < 0 || space > 2) return set_error(MACT_EBADARG, "unknown space %d", space);
  if (n < 0 || (n > 0 && (!rgb || !out)) || !c) return set_error(MACT_EBADARG, "bad argument");
  if (layout != MACT_LAYOUT_INTERLEAVED && layout != MACT_LAYOUT_PLANAR)
    return set_error(MACT_EBADARG, "unknown layout %d", layout);
  KCoeffs kc;                                   // validates the degree selection like the fp32 path
  if (int rc = make_kcoeffs(c, &kc)) return rc;
  if (n == 0) return MACT_OK;
  RefParams p;
  for (int k = 0; k < 8; ++k) {
    p.num[k] = c->cbrt_num[k]; p.den[k] = c->cbrt_den[k]; p.hsi[k] = c->atan_sqrt3[k];
    p.asin[k] = c->asin_half[k]; p.acos[k] = c->acos_half[k]; p.atanf[k] = c->atan_f[k];
    p.atang[k] = c->atan_g[k];
  }
  p.num_deg = c->cbrt_num_deg; p.den_deg = c->cbrt_den_deg; p.hsi_deg = c->hsi_deg;
  p.asin_deg = c->asin_deg; p.acos_deg = c->acos_deg; p.atan_deg = c->atan_deg;
  const int planar = layout == MACT_LAYOUT_PLANAR;
  cudaStream_t st = (cudaStream_t)stream;
  switch (in_dtype) {
    case MACT_DTYPE_U8: return ref_space(space, p, (const uint8_t*)rgb, out, n, planar, st);
    case MACT_DTYPE_F32: return ref_space(space, p, (const float*)rgb, out, n, planar, st);
    case MACT_DTYPE_F64: return ref_space(space, p, (const double*)rgb, out, n, planar, st);
  }
  return set_error(MACT_EBADARG, "unsupported input dtype %d", in_dtype);
}
