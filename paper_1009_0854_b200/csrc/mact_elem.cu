// mact_elem.cu — the reference's elementwise building blocks on fp64 device arrays.
//
//   mact_approx_eval <- fast.cbrt_fast / atan_sqrt3_fast / acos_fast / atan_unit_fast
//                       (fast.py:81-83, :118-122, :151-185) over
//                       approximants.eval_poly / eval_rational (approximants.py:55-82)
//   mact_poly_eval   <- approximants.eval_poly / eval_rational (approximants.py:55-82), any degree < 32
//   mact_exact_elem  <- exact.inverse_gamma / rgb_to_xyz / lab_f / xyz_to_lab (exact.py:52-83),
//                       lut.angular_lerp (lut.py:202-216)
//
// Horner runs exactly as numpy evaluates it (acc *= x; acc += c, each rounded:
// __dmul_rn / __dadd_rn, no FMA contraction), and +, *, /, sqrt are correctly
// rounded on both sides, so mact_approx_eval is bit-identical to the
// reference.  mact_exact_elem uses libdevice pow/cbrt (within 1-2 ulp of libm).
#include "mact_lut.cuh"

namespace mact {

struct ApproxParams {
  MactApproxSpec s;
};

__device__ __forceinline__ double horner_np(const double* c, int deg, double x) {
  double acc = c[deg];
  for (int i = deg - 1; i >= 0; --i) acc = __dadd_rn(__dmul_rn(acc, x), c[i]);
  return acc;
}

// np.maximum(d, 0.0): NaN propagates (C fmax would return 0)
__device__ __forceinline__ double max_np(double d) { return d != d ? d : (d > 0.0 ? d : 0.0); }

__global__ void k_approx(const __grid_constant__ ApproxParams p, const double* __restrict__ x,
                         const double* __restrict__ y, double* __restrict__ out, int64_t n,
                         int32_t* __restrict__ degenerate) {
  const MactApproxSpec& s = p.s;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    double r;
    switch (s.fn) {
      case MACT_FN_FORM:                                  // approximants.py:55-82
        if (s.b_deg < 0) {
          r = horner_np(s.a, s.a_deg, v);
        } else {
          const double den = horner_np(s.b, s.b_deg, v);
          if (fabs(den) < 1e-300 && degenerate) *degenerate = 1;
          r = __ddiv_rn(horner_np(s.a, s.a_deg, v), den);
        }
        break;
      case MACT_FN_ATAN_SQRT3: {                          // fast.py:118-122
        const double mag = horner_np(s.a, s.a_deg, fabs(v));
        r = v < 0.0 ? -mag : mag;
        break;
      }
      case MACT_FN_ACOS:                                  // fast.py:151-162
        r = v < 0.5 ? horner_np(s.a, s.a_deg, v)
                    : horner_np(s.b, s.b_deg, __dsqrt_rn(max_np(__dadd_rn(1.0, -v))));
        break;
      default: {                                          // MACT_FN_ATAN_UNIT, fast.py:165-185
        const double g = v, rr = y[i];
        if (g < rr) {
          r = horner_np(s.a, s.a_deg, __ddiv_rn(g, rr > 0.0 ? rr : 1.0));
        } else {
          r = horner_np(s.b, s.b_deg, g > 0.0 ? __ddiv_rn(rr, g) : 0.0);
        }
        if (g == 0.0 && rr == 0.0) r = __longlong_as_double(0x7ff8000000000000ll);
      }
    }
    out[i] = r;
  }
}

// approximants.eval_poly / eval_rational (approximants.py:55-82) for any
// Polynomial / Rational of degree < kPolyMax: numpy's Horner order, each step
// rounded twice (acc *= x; acc += c), the quotient rounded once.
struct PolyParams {
  MactPolySpec s;
};
__global__ void k_poly(const __grid_constant__ PolyParams p, const double* __restrict__ x,
                       double* __restrict__ out, int64_t n, int32_t* __restrict__ degenerate) {
  const MactPolySpec& s = p.s;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    const double num = horner_np(s.num, s.num_deg, v);
    if (s.den_deg < 0) {
      out[i] = num;
    } else {
      const double den = horner_np(s.den, s.den_deg, v);
      if (fabs(den) < 1e-300 && degenerate) *degenerate = 1;
      out[i] = __ddiv_rn(num, den);
    }
  }
}

__device__ __forceinline__ double inverse_gamma_np(double k) {    // exact.py:52-57
  return k < kGammaKnee ? __ddiv_rn(k, kGammaSlope)
                        : pow(__ddiv_rn(__dadd_rn(k, kGammaOffset), kGammaScale), kGammaPower);
}
__device__ __forceinline__ double lab_f_np(double t) {               // exact.py:69-72
  return t > kLabKnee ? cbrt(t) : __dadd_rn(__dmul_rn(kLabSlope, t), kLabOffset);
}

__global__ void k_exact_elem(int op, const double* __restrict__ a, const double* __restrict__ b,
                             const double* __restrict__ c, double* __restrict__ o0,
                             double* __restrict__ o1, double* __restrict__ o2, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (op >= MACT_ELEM_TARGET_CBRT) {                              // TargetFn.exact, approximants.py:101-115
      const double v = a[i];
      double r;
      switch (op) {
        case MACT_ELEM_TARGET_CBRT: r = cbrt(v); break;                          // np.cbrt
        case MACT_ELEM_TARGET_ATAN_SQRT3: r = atan(__dmul_rn(kSqrt3, v)); break;   // arctan(sqrt(3) x)
        case MACT_ELEM_TARGET_ASIN_HALF: r = __dmul_rn(2.0, asin(__ddiv_rn(v, kSqrt2))); break;
        case MACT_ELEM_TARGET_ACOS_HALF: r = acos(v); break;
        case MACT_ELEM_TARGET_ATAN_F: r = atan(v); break;
        default: r = __dadd_rn(__dmul_rn(0.5, kPi), -atan(v)); break;             // 0.5 pi - arctan(x)
      }
      o0[i] = r;
    } else if (op == MACT_ELEM_INVERSE_GAMMA) {
      o0[i] = inverse_gamma_np(a[i]);
    } else if (op == MACT_ELEM_LAB_F) {
      o0[i] = lab_f_np(a[i]);
    } else if (op == MACT_ELEM_ANGULAR_LERP) {
      o0[i] = angular_lerp_d(a[i], b[i], c[i]);
    } else if (op == MACT_ELEM_RGB_TO_XYZ) {                       // exact.py:60-66
      const double r = a[i], g = b[i], bb = c[i];
      double* o[3] = {o0, o1, o2};
#pragma unroll
      for (int row = 0; row < 3; ++row)
        o[row][i] = __dadd_rn(__dadd_rn(__dmul_rn(rgb2xyz(row, 0), r), __dmul_rn(rgb2xyz(row, 1), g)),
                              __dmul_rn(rgb2xyz(row, 2), bb));
    } else {                                                        // xyz_to_lab, exact.py:75-83
      const double fx = lab_f_np(__ddiv_rn(a[i], kWhiteX));
      const double fy = lab_f_np(__ddiv_rn(b[i], kWhiteY));
      const double fz = lab_f_np(__ddiv_rn(c[i], kWhiteZ));
      o0[3 * i] = __dadd_rn(__dmul_rn(116.0, fy), -16.0);
      o0[3 * i + 1] = __dmul_rn(500.0, __dadd_rn(fx, -fy));
      o0[3 * i + 2] = __dmul_rn(200.0, __dadd_rn(fy, -fz));
    }
  }
}

static unsigned elem_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = 8LL * num_sms();
  return (unsigned)(g < 1 ? 1 : g > cap ? cap : g);
}

}  // namespace mact

using namespace mact;

extern "C" int mact_approx_eval(const MactApproxSpec* spec, const double* x, const double* y,
                                double* out, int64_t n, int32_t* degenerate, void* stream) {
  if (!spec || n < 0 || (n > 0 && (!x || !out))) return set_error(MACT_EBADARG, "bad argument");
  if (spec->fn < MACT_FN_FORM || spec->fn > MACT_FN_ATAN_UNIT)
    return set_error(MACT_EBADARG, "unknown approximant function %d", spec->fn);
  if (spec->fn == MACT_FN_ATAN_UNIT && n > 0 && !y) return set_error(MACT_EBADARG, "atan_unit needs r");
  const bool two = spec->fn == MACT_FN_ACOS || spec->fn == MACT_FN_ATAN_UNIT;
  if (spec->a_deg < 0 || spec->a_deg > 7 || spec->b_deg > 7 || (two && spec->b_deg < 0))
    return set_error(MACT_EBADARG, "coefficient degrees out of range (%d, %d)", spec->a_deg, spec->b_deg);
  if (n == 0) return MACT_OK;
  ApproxParams p;
  p.s = *spec;
  k_approx<<<elem_grid(n), 256, 0, (cudaStream_t)stream>>>(p, x, y, out, n, degenerate);
  count_launch();
  return check_launch("approx_eval");
}

extern "C" int mact_exact_elem(int op, const double* in0, const double* in1, const double* in2,
                               double* out0, double* out1, double* out2, int64_t n, void* stream) {
  if (op < MACT_ELEM_INVERSE_GAMMA || op > MACT_ELEM_TARGET_ATAN_G)
    return set_error(MACT_EBADARG, "unknown elementwise op %d", op);
  const bool three_in = op == MACT_ELEM_RGB_TO_XYZ || op == MACT_ELEM_XYZ_TO_LAB ||
                        op == MACT_ELEM_ANGULAR_LERP;
  if (n < 0 || (n > 0 && (!in0 || !out0 || (three_in && (!in1 || !in2)) ||
                          (op == MACT_ELEM_RGB_TO_XYZ && (!out1 || !out2)))))
    return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  k_exact_elem<<<elem_grid(n), 256, 0, (cudaStream_t)stream>>>(op, in0, in1, in2, out0, out1, out2, n);
  count_launch();
  return check_launch("exact_elem");
}

extern "C" int mact_poly_eval(const MactPolySpec* spec, const double* x, double* out, int64_t n,
                              int32_t* degenerate, void* stream) {
  if (!spec || n < 0 || (n > 0 && (!x || !out))) return set_error(MACT_EBADARG, "bad argument");
  if (spec->num_deg < 0 || spec->num_deg >= MACT_POLY_MAX || spec->den_deg >= MACT_POLY_MAX)
    return set_error(MACT_EBADARG, "polynomial degrees out of range (%d, %d)", spec->num_deg, spec->den_deg);
  if (n == 0) return MACT_OK;
  PolyParams p;
  p.s = *spec;
  k_poly<<<elem_grid(n), 256, 0, (cudaStream_t)stream>>>(p, x, out, n, degenerate);
  count_launch();
  return check_launch("poly_eval");
}
