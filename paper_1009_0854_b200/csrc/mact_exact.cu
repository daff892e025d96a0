// mact_exact.cu — K5: fp64 ground-truth transforms, distances, pixel generators.
//
//   mact_exact        <- exact.rgb_to_{lab,hsi,sct}_exact (exact.py:86-149)
//   mact_sct_to_rgb   <- exact.sct_to_rgb                 (exact.py:152-160)
//   mact_distance     <- exact.lab_distance / hsi_distance / sct_distance_indirect
//                        (exact.py:163-190)
//   mact_cube_fill    <- harness.cube_chunk               (harness.py:35-46)
//   mact_call_counts  <- harness.call_probabilities       (harness.py:137-175)
//
// These are not on the roofline metric (the error path and lattice builds
// use them); they follow the reference formulas in fp64 with libdevice
// cbrt/pow/atan/acos/atan2/sincos.
#include <cmath>

#include "mact_pixel.cuh"

namespace mact {

template <typename T>
__device__ __forceinline__ double load_c(const T* p, int64_t i) { return (double)p[i]; }

__device__ __forceinline__ void exact_px(int space, double r, double g, double b, double* o) {
  if (space == MACT_SPACE_LAB) lab_exact_d(r, g, b, o);
  else if (space == MACT_SPACE_HSI) hsi_exact_d(r, g, b, o);
  else if (space == MACT_SPACE_SCT) sct_exact_d(r, g, b, o);
  else hsi_arccos_d(r, g, b, o);
}

template <typename TI, typename TO>
__global__ void k_exact(int space, const TI* __restrict__ in, TO* __restrict__ out, int64_t n) {
  __shared__ double gamma[256];
  // uint8 input: exact.rgb_to_lab_exact evaluates inverse_gamma(r/255) — the
  // same 256 values, so tabulate them once per CTA.
  const bool u8 = sizeof(TI) == 1;
  if (u8 && space == MACT_SPACE_LAB) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) gamma[i] = inverse_gamma_d(i / 255.0);
    __syncthreads();
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double o[3];
    if (u8 && space == MACT_SPACE_LAB) {
      lab_from_linear(gamma[(int)in[3 * i]], gamma[(int)in[3 * i + 1]], gamma[(int)in[3 * i + 2]], o);
    } else {
      exact_px(space, load_c(in, 3 * i), load_c(in, 3 * i + 1), load_c(in, 3 * i + 2), o);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) out[3 * i + k] = (TO)o[k];
  }
}

__global__ void k_sct_to_rgb(const double* __restrict__ s, double* __restrict__ rgb, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    sct_to_rgb_d(s + 3 * i, rgb + 3 * i);
}

template <typename TX, typename TY>
__global__ void k_distance(int space, const TX* __restrict__ x, const TY* __restrict__ y,
                           double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double a[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      a[k] = (double)x[3 * i + k];
      b[k] = (double)y[3 * i + k];
    }
    out[i] = distance_d(space, a, b);
  }
}

// 4 pixels (12 bytes, 3 words) per thread; pixel i = (i>>16, i>>8 & 255, i & 255)
__global__ void k_cube_fill(uint8_t* __restrict__ rgb, int64_t start, int64_t n) {
  const int64_t ngroups = n / 4;
  const bool aligned = ((uintptr_t)rgb % 4) == 0;
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < (n + 3) / 4;
       gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = gi * 4;
    if (aligned && gi < ngroups) {
      uint32_t b[12];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t idx = (uint32_t)((start + p0 + k) & 0xFFFFFF);
        b[3 * k] = idx >> 16;
        b[3 * k + 1] = (idx >> 8) & 255u;
        b[3 * k + 2] = idx & 255u;
      }
      uint32_t* w = reinterpret_cast<uint32_t*>(rgb + 3 * p0);
      w[0] = b[0] | b[1] << 8 | b[2] << 16 | b[3] << 24;
      w[1] = b[4] | b[5] << 8 | b[6] << 16 | b[7] << 24;
      w[2] = b[8] | b[9] << 8 | b[10] << 16 | b[11] << 24;
    } else {
      for (int k = 0; k < 4 && p0 + k < n; ++k) {
        const uint32_t idx = (uint32_t)((start + p0 + k) & 0xFFFFFF);
        rgb[3 * (p0 + k)] = (uint8_t)(idx >> 16);
        rgb[3 * (p0 + k) + 1] = (uint8_t)(idx >> 8);
        rgb[3 * (p0 + k) + 2] = (uint8_t)idx;
      }
    }
  }
}

// harness.call_probabilities (harness.py:137-175) as exact counts over the
// cube.  One thread per (r, g) walks b = 0..255.  The lightness-kernel test
// keeps the reference's fp64 evaluation order, m0*gamma[r] + (m1*gamma[g] +
// m2*gamma[b]) > knee*white (harness.py:146-156), with explicit _rn ops so no
// FMA contraction changes a rounding; gamma[] is the host-libm table (the
// reference's numpy pow), not libdevice pow, so a value within an ulp of the
// threshold cannot flip.  Integer counts -> atomics are order-independent.
struct CallParams {
  double gamma[256];
};

__global__ void __launch_bounds__(256) k_call_counts(const __grid_constant__ CallParams p,
                                                     unsigned long long* __restrict__ counts) {
  __shared__ double m[3][3], thr[3];
  if (threadIdx.x < 9) m[threadIdx.x / 3][threadIdx.x % 3] = rgb2xyz(threadIdx.x / 3, threadIdx.x % 3);
  if (threadIdx.x < 3)
    thr[threadIdx.x] = __dmul_rn(kLabKnee, threadIdx.x == 0 ? kWhiteX : threadIdx.x == 1 ? kWhiteY : kWhiteZ);
  __syncthreads();
  const int rg = blockIdx.x * blockDim.x + threadIdx.x;          // grid covers 65536 exactly
  const int r = rg >> 8, g = rg & 255;
  uint32_t cx = 0, cy = 0, cz = 0, casin = 0;
  double tr[3], tg[3];
#pragma unroll
  for (int row = 0; row < 3; ++row) {
    tr[row] = __dmul_rn(m[row][0], p.gamma[r]);
    tg[row] = __dmul_rn(m[row][1], p.gamma[g]);
  }
  const int rg2 = r * r + g * g;
  for (int b = 0; b < 256; ++b) {
    const double gb = p.gamma[b];
    cx += __dadd_rn(tr[0], __dadd_rn(tg[0], __dmul_rn(m[0][2], gb))) > thr[0];
    cy += __dadd_rn(tr[1], __dadd_rn(tg[1], __dmul_rn(m[1][2], gb))) > thr[1];
    cz += __dadd_rn(tr[2], __dadd_rn(tg[2], __dmul_rn(m[2][2], gb))) > thr[2];
    casin += 3 * b * b >= rg2;
  }
  const uint32_t catan = (r | g) ? 256u : 0u;
  uint32_t v[5] = {cx, cy, cz, casin, catan};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < 5; ++k) atomicAdd(&counts[k < 4 ? k : 5], (unsigned long long)v[k]);
  }
}

__global__ void k_call_counts_finish(unsigned long long* counts) {
  counts[4] = (1ull << 24) - counts[3];                           // arccos = complement
}

static unsigned grid_for(int64_t n, int per_sm = 8) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)per_sm * num_sms();
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

template <typename TI>
static int exact_out(int space, const TI* in, void* out, int out_dtype, int64_t n, cudaStream_t st) {
  if (out_dtype == MACT_DTYPE_F64)
    k_exact<TI, double><<<grid_for(n), 256, 0, st>>>(space, in, (double*)out, n);
  else if (out_dtype == MACT_DTYPE_F32)
    k_exact<TI, float><<<grid_for(n), 256, 0, st>>>(space, in, (float*)out, n);
  else
    return set_error(MACT_EBADARG, "unsupported output dtype %d", out_dtype);
  count_launch();
  return check_launch("exact");
}

template <typename TX>
static int dist_y(int space, const TX* x, const void* y, int y_dtype, double* out, int64_t n,
                  cudaStream_t st) {
  if (y_dtype == MACT_DTYPE_F64)
    k_distance<TX, double><<<grid_for(n), 256, 0, st>>>(space, x, (const double*)y, out, n);
  else if (y_dtype == MACT_DTYPE_F32)
    k_distance<TX, float><<<grid_for(n), 256, 0, st>>>(space, x, (const float*)y, out, n);
  else
    return set_error(MACT_EBADARG, "unsupported dtype %d", y_dtype);
  count_launch();
  return check_launch("distance");
}

}  // namespace mact

using namespace mact;

extern "C" int mact_exact(int space, const void* rgb, int in_dtype, void* out, int out_dtype,
                          int64_t n, void* stream) {
  NvtxRange range("mact_exact");
  if (space < 0 || space > MACT_SPACE_HSI_ARCCOS) return set_error(MACT_EBADARG, "unknown space %d", space);
  if (n < 0 || (n > 0 && (!rgb || !out))) return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (in_dtype) {
    case MACT_DTYPE_U8: return exact_out(space, (const uint8_t*)rgb, out, out_dtype, n, st);
    case MACT_DTYPE_F32: return exact_out(space, (const float*)rgb, out, out_dtype, n, st);
    case MACT_DTYPE_F64: return exact_out(space, (const double*)rgb, out, out_dtype, n, st);
    default: return set_error(MACT_EBADARG, "unsupported input dtype %d", in_dtype);
  }
}

extern "C" int mact_sct_to_rgb(const double* sct, double* rgb, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!sct || !rgb))) return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  k_sct_to_rgb<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(sct, rgb, n);
  count_launch();
  return check_launch("sct_to_rgb");
}

extern "C" int mact_distance(int space, const void* x, int x_dtype, const void* y, int y_dtype,
                             double* out, int64_t n, void* stream) {
  if (space < 0 || space > 2) return set_error(MACT_EBADARG, "unknown space %d", space);
  if (n < 0 || (n > 0 && (!x || !y || !out))) return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (x_dtype == MACT_DTYPE_F64) return dist_y(space, (const double*)x, y, y_dtype, out, n, st);
  if (x_dtype == MACT_DTYPE_F32) return dist_y(space, (const float*)x, y, y_dtype, out, n, st);
  return set_error(MACT_EBADARG, "unsupported dtype %d", x_dtype);
}

extern "C" int mact_call_counts(unsigned long long* counts, void* stream) {
  if (!counts) return set_error(MACT_EBADARG, "bad argument");
  static const CallParams params = [] {
    CallParams q;
    for (int i = 0; i < 256; ++i) {          // exact.inverse_gamma(i / 255) (exact.py:52-57), host libm
      const double k = i / 255.0;
      q.gamma[i] = k < kGammaKnee ? k / kGammaSlope : std::pow((k + kGammaOffset) / kGammaScale, kGammaPower);
    }
    return q;
  }();
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(counts, 0, 6 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return set_error(MACT_ECUDA, "call_counts: %s", cudaGetErrorString(e));
  k_call_counts<<<256, 256, 0, st>>>(params, counts);
  k_call_counts_finish<<<1, 1, 0, st>>>(counts);
  count_launch(2);
  return check_launch("call_counts");
}

extern "C" int mact_cube_fill(uint8_t* rgb, int64_t start, int64_t n, void* stream) {
  if (n < 0 || start < 0 || (n > 0 && !rgb)) return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  k_cube_fill<<<grid_for((n + 3) / 4), 256, 0, (cudaStream_t)stream>>>(rgb, start, n);
  count_launch();
  return check_launch("cube_fill");
}
