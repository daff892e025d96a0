// mact_exact.cu — K5: fp64 ground-truth transforms, distances, pixel generators.
//
//   mact_exact        <- exact.rgb_to_{lab,hsi,sct}_exact (exact.py:86-149)
//   mact_sct_to_rgb   <- exact.sct_to_rgb                 (exact.py:152-160)
//   mact_distance     <- exact.lab_distance / hsi_distance / sct_distance_indirect
//                        (exact.py:163-190)
//   mact_cube_fill    <- harness.cube_chunk               (harness.py:35-46)
//
// These are not on the roofline metric (the error path and lattice builds
// use them); they follow the reference formulas in fp64 with libdevice
// cbrt/pow/atan/acos/atan2/sincos.
#include "mact_pixel.cuh"

namespace mact {

template <typename T>
__device__ __forceinline__ double load_c(const T* p, int64_t i) { return (double)p[i]; }

__device__ __forceinline__ void exact_px(int space, double r, double g, double b, double* o) {
  if (space == MACT_SPACE_LAB) lab_exact_d(r, g, b, o);
  else if (space == MACT_SPACE_HSI) hsi_exact_d(r, g, b, o);
  else sct_exact_d(r, g, b, o);
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
  if (space < 0 || space > 2) return set_error(MACT_EBADARG, "unknown space %d", space);
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

extern "C" int mact_cube_fill(uint8_t* rgb, int64_t start, int64_t n, void* stream) {
  if (n < 0 || start < 0 || (n > 0 && !rgb)) return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  k_cube_fill<<<grid_for((n + 3) / 4), 256, 0, (cudaStream_t)stream>>>(rgb, start, n);
  count_launch();
  return check_launch("cube_fill");
}
