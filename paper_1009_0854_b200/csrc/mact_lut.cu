// mact_lut.cu — K4: 3D-LUT build, node selection and interpolation.
//
//   mact_lut_build   <- lut.build_lut        (lut.py:77-95)
//   mact_lut_nodes   <- lut.node_weights     (lut.py:115-199)
//   mact_lut_interp  <- lut.interpolate(..., variant="standard") for the linear
//                       CIELAB destination   (lut.py:231-246, :341-350)
//
// Device lattice format: (n^3, 4) fp32, r-major, node = (c0, c1, c2, 0) so a
// node is one 16-byte load.  Interpolation runs inside the streaming skeleton
// (mact_stream.cuh).  For grids 9^3 and 17^3 the lattice is staged once per
// persistent CTA into shared memory (17^3 x 16 B = 78.6 KB): one LDS.128 per
// node.  33^3 (575 KB) exceeds a CTA's 227 KB and is gathered with LDG.128
// through L1/L2 (the lattice stays L2-resident).
#include "mact_lut.cuh"
#include "mact_pixel.cuh"
#include "mact_stream.cuh"

namespace mact {

struct LutParams {
  const float4* lat;   // (n^3, 4) fp32, r-major, padded
};

template <int N, int METHOD>
struct OpLut {
  static constexpr int NOUT = 1;
  static constexpr bool SMEM = N <= 17;
  using Params = LutParams;
  struct Shared {
    float4 lat[SMEM ? N * N * N : 1];
  };
  static __device__ __forceinline__ void init(Shared* s, const Params& p) {
    if constexpr (SMEM) {
      for (int i = threadIdx.x; i < N * N * N; i += blockDim.x)
        s->lat[i] = __ldg(p.lat + i);
    }
  }
  static __device__ __forceinline__ float3 node(const Shared* s, const Params& p, int i) {
    if constexpr (SMEM) {
      const float4 v = s->lat[i];
      return make_float3(v.x, v.y, v.z);
    } else {
      const float4 v = __ldg(p.lat + i);
      return make_float3(v.x, v.y, v.z);
    }
  }
  static __device__ __forceinline__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared* s,
                                            uint32_t, const Params& p, float (*o)[3]) {
    constexpr int K = LutK<METHOD>::K;
    int idx[K];
    float w[K];
    lut_nodes<N, METHOD>(r, g, b, idx, w);
    float3 v = node(s, p, idx[0]);
    float a0 = w[0] * v.x, a1 = w[0] * v.y, a2 = w[0] * v.z;
#pragma unroll
    for (int j = 1; j < K; ++j) {
      v = node(s, p, idx[j]);
      a0 = fmaf(w[j], v.x, a0);
      a1 = fmaf(w[j], v.y, a1);
      a2 = fmaf(w[j], v.z, a2);
    }
    o[0][0] = a0; o[0][1] = a1; o[0][2] = a2;
  }
  // 4 pixels: all node indices first, then every node load, then the FMAs, so
  // 4*K independent gathers are in flight per thread (L2 latency for 33^3,
  // LDS latency for the smem lattice).  Trilinear (K = 8) goes 2 pixels at a
  // time to bound register pressure.
  static __device__ __forceinline__ void px4w(uint32_t w0, uint32_t w1, uint32_t w2,
                                              const Shared* s, uint32_t lane, const Params& p,
                                              float (*o)[1][3]) {
    constexpr int K = LutK<METHOD>::K;
    constexpr int PB = K > 6 ? 2 : 4;                 // pixels per batch
    const uint32_t ch[12] = {byte_of(w0, 0), byte_of(w0, 1), byte_of(w0, 2), byte_of(w0, 3),
                             byte_of(w1, 0), byte_of(w1, 1), byte_of(w1, 2), byte_of(w1, 3),
                             byte_of(w2, 0), byte_of(w2, 1), byte_of(w2, 2), byte_of(w2, 3)};
#pragma unroll
    for (int q0 = 0; q0 < 4; q0 += PB) {
      int idx[PB][K];
      float w[PB][K];
      float3 v[PB][K];
#pragma unroll
      for (int q = 0; q < PB; ++q)
        lut_nodes<N, METHOD>(ch[3 * (q0 + q)], ch[3 * (q0 + q) + 1], ch[3 * (q0 + q) + 2], idx[q], w[q]);
#pragma unroll
      for (int q = 0; q < PB; ++q)
#pragma unroll
        for (int j = 0; j < K; ++j) v[q][j] = node(s, p, idx[q][j]);
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        float a0 = w[q][0] * v[q][0].x, a1 = w[q][0] * v[q][0].y, a2 = w[q][0] * v[q][0].z;
#pragma unroll
        for (int j = 1; j < K; ++j) {
          a0 = fmaf(w[q][j], v[q][j].x, a0);
          a1 = fmaf(w[q][j], v[q][j].y, a1);
          a2 = fmaf(w[q][j], v[q][j].z, a2);
        }
        o[q0 + q][0][0] = a0; o[q0 + q][0][1] = a1; o[q0 + q][0][2] = a2;
      }
    }
  }
};

// ------------------------------------------------------- angular destinations
// lut.py:202-262.  Components flagged in MASK (bit c: component c is an angle —
// HSI hue, both SCT angles) are blended on the circle; the others take the
// standard weighted sum.  Simplex methods use the weight-blended circular mean
// of their nodes (_circular_blend, lut.py:219-228); trilinear cascades
// pairwise angular_lerp along r, then g, then b (lut.py:249-262).  A vanishing
// blended direction (hypot < 1e-12) falls back to the heaviest node (first
// maximum weight) or to theta0, wrapped into [0, 2 pi).
//
// Near the gray axis the circular mean is a sum of almost-cancelling unit
// vectors, so it is evaluated like the reference: fp64 lattice (n^3, 3),
// fp64 weights (exact integer products / 255^k), fp64 sincos/atan2.  This
// destination is not on the throughput metric; a per-pixel kernel suffices.
__device__ __forceinline__ double fmod2pi_d(double a) {
  a = fmod(a, kTwoPi);
  return a < 0.0 ? a + kTwoPi : a;
}
__device__ __forceinline__ double angular_lerp_d(double t0, double t1, double a) {
  double s0, c0, s1, c1;
  sincos(t0, &s0, &c0);
  sincos(t1, &s1, &c1);
  const double c = (1.0 - a) * c0 + a * c1, s = (1.0 - a) * s0 + a * s1;
  if (hypot(c, s) < 1e-12) return fmod2pi_d(t0);
  const double out = atan2(s, c);
  return out < 0.0 ? out + kTwoPi : out;
}

template <int N, int METHOD>
__global__ void k_lut_angular(const double* __restrict__ lat, int mask, const uint8_t* __restrict__ rgb,
                              float* __restrict__ out, int64_t n, int planar) {
  constexpr int K = LutK<METHOD>::K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
    int idx[K];
    double w[K];
    lut_nodes<N, METHOD, double>(r, g, b, idx, w);
    double res[3];
    for (int comp = 0; comp < 3; ++comp) {
      if (!((mask >> comp) & 1)) {
        double a = 0.0;
        for (int j = 0; j < K; ++j) a += w[j] * lat[3 * idx[j] + comp];
        res[comp] = a;
      } else if (METHOD == MACT_LUT_TRILINEAR) {
        int br, bg, bb, rr, rg, rb;
        lut_locate<N>(r, br, rr);
        lut_locate<N>(g, bg, rg);
        lut_locate<N>(b, bb, rb);
        const double dr = rr / 255.0, dg = rg / 255.0, db = rb / 255.0;
        double v[8];
        for (int j = 0; j < 8; ++j) v[j] = lat[3 * idx[j] + comp];   // corner c = r<<2|g<<1|b
        const double r00 = angular_lerp_d(v[0], v[4], dr), r01 = angular_lerp_d(v[1], v[5], dr);
        const double r10 = angular_lerp_d(v[2], v[6], dr), r11 = angular_lerp_d(v[3], v[7], dr);
        res[comp] = angular_lerp_d(angular_lerp_d(r00, r10, dg), angular_lerp_d(r01, r11, dg), db);
      } else {
        double c = 0.0, sn = 0.0, wmax = w[0], heavy = lat[3 * idx[0] + comp];
        for (int j = 0; j < K; ++j) {
          const double t = lat[3 * idx[j] + comp];
          double sj, cj;
          sincos(t, &sj, &cj);
          c += w[j] * cj;
          sn += w[j] * sj;
          if (w[j] > wmax) { wmax = w[j]; heavy = t; }
        }
        if (hypot(c, sn) < 1e-12) {
          res[comp] = fmod2pi_d(heavy);
        } else {
          const double o = atan2(sn, c);
          res[comp] = o < 0.0 ? o + kTwoPi : o;
        }
      }
    }
    for (int comp = 0; comp < 3; ++comp) {
      if (planar) out[comp * n + i] = (float)res[comp];
      else out[3 * i + comp] = (float)res[comp];
    }
  }
}

// ---------------------------------------------------------------- build
__global__ void k_lut_build(int space, int n, double* __restrict__ f64, float* __restrict__ f32) {
  const int total = n * n * n;
  const double spacing = 255.0 / (n - 1);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int ir = i / (n * n), ig = (i / n) % n, ib = i % n;
    double o[3];
    const double r = ir * spacing, g = ig * spacing, b = ib * spacing;   // lattice_coordinates
    if (space == MACT_SPACE_LAB) lab_exact_d(r, g, b, o);
    else if (space == MACT_SPACE_HSI) hsi_exact_d(r, g, b, o);
    else sct_exact_d(r, g, b, o);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double v = isnan(o[k]) ? 0.0 : o[k];                        // nan_to_num (lut.py:92)
      if (f64) f64[3 * i + k] = v;
      if (f32) f32[4 * i + k] = (float)v;
    }
    if (f32) f32[4 * i + 3] = 0.0f;
  }
}

// --------------------------------------------------------------- nodes
template <int N, int METHOD>
__global__ void k_lut_nodes(const uint8_t* __restrict__ rgb, int64_t n, int32_t* __restrict__ nodes,
                            float* __restrict__ weights) {
  constexpr int K = LutK<METHOD>::K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int idx[K];
    float w[K];
    lut_nodes<N, METHOD>(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], idx, w);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      nodes[i * K + j] = idx[j];
      weights[i * K + j] = w[j];
    }
  }
}

template <int N, int METHOD>
static int launch_interp(const float* lat, const uint8_t* rgb, float* out, int64_t n, int planar,
                         cudaStream_t st) {
  Outs outs{{out, nullptr, nullptr}};
  LutParams p{reinterpret_cast<const float4*>(lat)};
  // 17^3: 78.6 KB lattice + 9 KB in + 12 KB out -> 2 CTA/SM (16 compute warps);
  // 33^3 gathers from L2, so more warps in flight: 16 per CTA, 3 CTA/SM.
  if constexpr (N == 33)
    return launch_stream_t<OpLut<N, METHOD>, 16, 1, 3, 1>(rgb, outs, n, planar, p, st, "lut_interp");
  else
    return launch_stream_t<OpLut<N, METHOD>, 8, (N <= 9 ? 2 : 1), 3, 1>(rgb, outs, n, planar, p, st,
                                                                         "lut_interp");
}

template <int N>
static int interp_grid(int method, const float* lat, const uint8_t* rgb, float* out, int64_t n,
                       int planar, cudaStream_t st) {
  switch (method) {
    case MACT_LUT_TRILINEAR: return launch_interp<N, MACT_LUT_TRILINEAR>(lat, rgb, out, n, planar, st);
    case MACT_LUT_PRISM: return launch_interp<N, MACT_LUT_PRISM>(lat, rgb, out, n, planar, st);
    case MACT_LUT_PYRAMIDAL: return launch_interp<N, MACT_LUT_PYRAMIDAL>(lat, rgb, out, n, planar, st);
    case MACT_LUT_TETRAHEDRAL: return launch_interp<N, MACT_LUT_TETRAHEDRAL>(lat, rgb, out, n, planar, st);
  }
  return set_error(MACT_EBADARG, "unknown interpolation method %d", method);
}

template <int N>
static int interp_ang(int method, int mask, const double* lat, const uint8_t* rgb, float* out,
                      int64_t n, int planar, cudaStream_t st) {
  int64_t g = (n + 255) / 256;
  if (g > 8LL * num_sms()) g = 8LL * num_sms();
  switch (method) {
    case MACT_LUT_TRILINEAR: k_lut_angular<N, MACT_LUT_TRILINEAR><<<(unsigned)g, 256, 0, st>>>(lat, mask, rgb, out, n, planar); break;
    case MACT_LUT_PRISM: k_lut_angular<N, MACT_LUT_PRISM><<<(unsigned)g, 256, 0, st>>>(lat, mask, rgb, out, n, planar); break;
    case MACT_LUT_PYRAMIDAL: k_lut_angular<N, MACT_LUT_PYRAMIDAL><<<(unsigned)g, 256, 0, st>>>(lat, mask, rgb, out, n, planar); break;
    case MACT_LUT_TETRAHEDRAL: k_lut_angular<N, MACT_LUT_TETRAHEDRAL><<<(unsigned)g, 256, 0, st>>>(lat, mask, rgb, out, n, planar); break;
    default: return set_error(MACT_EBADARG, "unknown interpolation method %d", method);
  }
  count_launch();
  return check_launch("lut_interp_angular");
}

template <int N>
static int nodes_grid(int method, const uint8_t* rgb, int64_t n, int32_t* nodes, float* w,
                      cudaStream_t st) {
  int64_t g = (n + 255) / 256;
  if (g > 8LL * num_sms()) g = 8LL * num_sms();
  switch (method) {
    case MACT_LUT_TRILINEAR: k_lut_nodes<N, MACT_LUT_TRILINEAR><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_PRISM: k_lut_nodes<N, MACT_LUT_PRISM><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_PYRAMIDAL: k_lut_nodes<N, MACT_LUT_PYRAMIDAL><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_TETRAHEDRAL: k_lut_nodes<N, MACT_LUT_TETRAHEDRAL><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    default: return set_error(MACT_EBADARG, "unknown interpolation method %d", method);
  }
  count_launch();
  return check_launch("lut_nodes");
}

}  // namespace mact

using namespace mact;

extern "C" int mact_lut_build(int space, int grid_n, double* lattice_f64, float* lattice_f32,
                              void* stream) {
  if (space < 0 || space > 2) return set_error(MACT_EBADARG, "unknown destination space %d", space);
  if (grid_n != 9 && grid_n != 17 && grid_n != 33)
    return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
  if (!lattice_f64 && !lattice_f32) return set_error(MACT_EBADARG, "no output lattice");
  const int total = grid_n * grid_n * grid_n;
  k_lut_build<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(space, grid_n, lattice_f64,
                                                                     lattice_f32);
  count_launch();
  return check_launch("lut_build");
}

extern "C" int mact_lut_interp(const float* lattice, int grid_n, int method, const uint8_t* rgb,
                               float* out, int64_t n, int layout, void* stream) {
  if (n < 0 || (n > 0 && (!lattice || !rgb || !out))) return set_error(MACT_EBADARG, "bad argument");
  if ((uintptr_t)lattice % 16) return set_error(MACT_EBADARG, "lattice must be 16-byte aligned");
  if (layout != MACT_LAYOUT_INTERLEAVED && layout != MACT_LAYOUT_PLANAR)
    return set_error(MACT_EBADARG, "unknown layout %d", layout);
  const int planar = layout == MACT_LAYOUT_PLANAR;
  cudaStream_t st = (cudaStream_t)stream;
  switch (grid_n) {
    case 9: return interp_grid<9>(method, lattice, rgb, out, n, planar, st);
    case 17: return interp_grid<17>(method, lattice, rgb, out, n, planar, st);
    case 33: return interp_grid<33>(method, lattice, rgb, out, n, planar, st);
  }
  return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
}

extern "C" int mact_lut_nodes(int grid_n, int method, const uint8_t* rgb, int64_t n,
                              int32_t* nodes, float* weights, void* stream) {
  if (n < 0 || (n > 0 && (!rgb || !nodes || !weights))) return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (grid_n) {
    case 9: return nodes_grid<9>(method, rgb, n, nodes, weights, st);
    case 17: return nodes_grid<17>(method, rgb, n, nodes, weights, st);
    case 33: return nodes_grid<33>(method, rgb, n, nodes, weights, st);
  }
  return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
}

extern "C" int mact_lut_interp_angular(const double* lattice64, int grid_n, int method,
                                       int angular_mask, const uint8_t* rgb, float* out, int64_t n,
                                       int layout, void* stream) {
  if (n < 0 || (n > 0 && (!lattice64 || !rgb || !out))) return set_error(MACT_EBADARG, "bad argument");
  if (angular_mask < 0 || angular_mask > 7) return set_error(MACT_EBADARG, "bad angular mask %d", angular_mask);
  if (layout != MACT_LAYOUT_INTERLEAVED && layout != MACT_LAYOUT_PLANAR)
    return set_error(MACT_EBADARG, "unknown layout %d", layout);
  if (n == 0) return MACT_OK;
  const int planar = layout == MACT_LAYOUT_PLANAR;
  cudaStream_t st = (cudaStream_t)stream;
  switch (grid_n) {
    case 9: return interp_ang<9>(method, angular_mask, lattice64, rgb, out, n, planar, st);
    case 17: return interp_ang<17>(method, angular_mask, lattice64, rgb, out, n, planar, st);
    case 33: return interp_ang<33>(method, angular_mask, lattice64, rgb, out, n, planar, st);
  }
  return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
}
