// mact_ref.cu — the float64 fidelity mode of the fast transforms
// (mact_fast_f64): the reference's own arithmetic (mact_ref.cuh), bit-identical
// to mact.fast.rgb_to_{lab,hsi,sct}_fast (fast.py:86-203) for uint8 pixels and
// for real-valued HSI / SCT pixels; real-valued Lab inputs go through libdevice
// pow in inverse_gamma (within an ulp of libm).  The throughput path is
// mact_{lab,hsi,sct}_fast with fp32 outputs.
#include "mact_ref.cuh"

namespace mact {

template <typename TI>
__device__ __forceinline__ double chan(const TI* p, int64_t i) { return (double)p[i]; }

// exact.inverse_gamma (exact.py:52-57): uint8 channels read the table, real ones evaluate it
template <typename TI>
__device__ __forceinline__ double lin(const TI* p, int64_t i) {
  if constexpr (sizeof(TI) == 1) return ref::kGammaF64[p[i]];
  else return ref::inverse_gamma(ref::dv(chan(p, i), 255.0));
}

template <int SPACE, typename TI>
__global__ void k_fast_ref(const __grid_constant__ KCoeffs c, const TI* __restrict__ in,
                           double* __restrict__ out, int64_t n, int planar) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double o[3];
    if constexpr (SPACE == MACT_SPACE_LAB) ref::lab_fast(lin(in, 3 * i), lin(in, 3 * i + 1), lin(in, 3 * i + 2), c, o);
    else if constexpr (SPACE == MACT_SPACE_HSI)
      ref::hsi_fast<sizeof(TI) == 1>(chan(in, 3 * i), chan(in, 3 * i + 1), chan(in, 3 * i + 2), c, o);
    else ref::sct_fast(chan(in, 3 * i), chan(in, 3 * i + 1), chan(in, 3 * i + 2), c, o);
    if (planar) {
      out[i] = o[0]; out[n + i] = o[1]; out[2 * n + i] = o[2];
    } else {
      out[3 * i] = o[0]; out[3 * i + 1] = o[1]; out[3 * i + 2] = o[2];
    }
  }
}

template <int SPACE, typename TI>
static int launch_ref(const KCoeffs& p, const TI* in, double* out, int64_t n, int planar, cudaStream_t st) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = 8LL * num_sms();
  if (g > cap) g = cap;
  k_fast_ref<SPACE, TI><<<(unsigned)g, 256, 0, st>>>(p, in, out, n, planar);
  count_launch();
  return check_launch("fast_f64");
}

template <typename TI>
static int ref_space(int space, const KCoeffs& p, const TI* in, double* out, int64_t n, int planar,
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
  const int planar = layout == MACT_LAYOUT_PLANAR;
  cudaStream_t st = (cudaStream_t)stream;
  switch (in_dtype) {
    case MACT_DTYPE_U8: return ref_space(space, kc, (const uint8_t*)rgb, out, n, planar, st);
    case MACT_DTYPE_F32: return ref_space(space, kc, (const float*)rgb, out, n, planar, st);
    case MACT_DTYPE_F64: return ref_space(space, kc, (const double*)rgb, out, n, planar, st);
  }
  return set_error(MACT_EBADARG, "unsupported input dtype %d", in_dtype);
}
