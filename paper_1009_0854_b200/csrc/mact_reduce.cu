// mact_reduce.cu — K6: fused candidate + exact + metric + reduction.
//
// Semantics follow harness.measure_error (harness.py:71-122): per pixel the
// space's distance (DISTANCES, harness.py:28-32 -> exact.py:163-190) between
// the candidate and the exact transform; statistics {sum, max, first argmax,
// count}.  COMPONENT mode reports per-component |candidate - exact| (hue
// circular, NaN-exact pixels excluded and counted).
//
// Determinism: a fixed grid (persistent, capped), each thread visits a fixed
// ascending index sequence, warp/block trees in a fixed shape, per-block
// partials folded by one block in block order.  Ties on the maximum keep the
// LOWEST global index, matching np.argmax + strict '>' across chunks.
#include <cstring>

#include "mact_lut.cuh"
#include "mact_pixel.cuh"
#include "mact_ref.cuh"

namespace mact {

constexpr int kRedThreads = 256;
constexpr int kRedSegCopies = 4;
constexpr int kRedMaxBlocks = 2048;

struct Acc {
  double sum, max;
  unsigned long long count, argmax, nan;
};

__device__ __forceinline__ void acc_init(Acc& a) {
  a.sum = 0.0; a.max = -1.0; a.count = 0; a.argmax = ~0ull; a.nan = 0;
}
__device__ __forceinline__ void acc_push(Acc& a, double d, unsigned long long gidx) {
  if (isnan(d)) { a.nan++; return; }
  a.sum += d;
  a.count++;
  if (d > a.max) { a.max = d; a.argmax = gidx; }
}
__device__ __forceinline__ void acc_merge(Acc& a, const Acc& b) {
  a.sum += b.sum;
  a.count += b.count;
  a.nan += b.nan;
  if (b.max > a.max || (b.max == a.max && b.argmax < a.argmax)) { a.max = b.max; a.argmax = b.argmax; }
}
__device__ __forceinline__ Acc acc_shfl(const Acc& a, int off) {
  Acc b;
  b.sum = __shfl_down_sync(0xffffffffu, a.sum, off);
  b.max = __shfl_down_sync(0xffffffffu, a.max, off);
  b.count = __shfl_down_sync(0xffffffffu, a.count, off);
  b.argmax = __shfl_down_sync(0xffffffffu, a.argmax, off);
  b.nan = __shfl_down_sync(0xffffffffu, a.nan, off);
  return b;
}

// Block-wide reduction of NC accumulators; result valid in thread 0.
template <int NC>
__device__ void block_reduce(Acc (&a)[NC]) {
  __shared__ Acc sh[kRedThreads / 32][NC];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < NC; ++c)
    for (int off = 16; off > 0; off >>= 1) acc_merge(a[c], acc_shfl(a[c], off));
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < NC; ++c) sh[wid][c] = a[c];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      a[c] = sh[0][c];
      for (int w = 1; w < kRedThreads / 32; ++w) acc_merge(a[c], sh[w][c]);
    }
  }
}

struct RedParams {
  MactErrSpec spec;
  KCoeffs c;
  const uint8_t* rgb;
  int64_t cube_start;
  int64_t n;
  int64_t index_base;
};

template <int N>
__device__ __forceinline__ void lut_value(const float* lat, int method, uint32_t r, uint32_t g,
                                          uint32_t b, double* o) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f;
  const float4* lat4 = reinterpret_cast<const float4*>(lat);   // (n^3, 4) padded lattice
  auto acc = [&](const int* idx, const float* w, int k) {
    for (int j = 0; j < k; ++j) {
      const float4 v = __ldg(lat4 + idx[j]);
      if (j == 0) { a0 = w[0] * v.x; a1 = w[0] * v.y; a2 = w[0] * v.z; }
      else { a0 = fmaf(w[j], v.x, a0); a1 = fmaf(w[j], v.y, a1); a2 = fmaf(w[j], v.z, a2); }
    }
  };
  if (method == MACT_LUT_TRILINEAR) { int i[8]; float w[8]; lut_nodes<N, MACT_LUT_TRILINEAR>(r, g, b, i, w); acc(i, w, 8); }
  else if (method == MACT_LUT_PRISM) { int i[6]; float w[6]; lut_nodes<N, MACT_LUT_PRISM>(r, g, b, i, w); acc(i, w, 6); }
  else if (method == MACT_LUT_PYRAMIDAL) { int i[5]; float w[5]; lut_nodes<N, MACT_LUT_PYRAMIDAL>(r, g, b, i, w); acc(i, w, 5); }
  else { int i[4]; float w[4]; lut_nodes<N, MACT_LUT_TETRAHEDRAL>(r, g, b, i, w); acc(i, w, 4); }
  o[0] = a0; o[1] = a1; o[2] = a2;
}

template <typename T>
__device__ __forceinline__ void load3(const void* p, int64_t i, double* o) {
  const T* q = reinterpret_cast<const T*>(p) + 3 * i;
  o[0] = (double)q[0]; o[1] = (double)q[1]; o[2] = (double)q[2];
}

template <int NC>
__global__ void __launch_bounds__(kRedThreads) k_err(const __grid_constant__ RedParams p,
                                                     MactErrStats* __restrict__ parts) {
  // the reference's fp64 GAMMA_TABLE (fast.py:35, exact.py:52-57 at i/255) and its fp32 rounding
  __shared__ float gamma_rep[256 * 32];
  __shared__ double gamma_d[256];
  __shared__ float4 seg[kLabSegs * kRedSegCopies];   // KCoeffs::seg (fewer copies: static smem cap)
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) gamma_rep[i] = (float)ref::kGammaF64[i >> 5];
  if (p.c.lab_seg)
    for (int i = (int)(threadIdx.x >> 5); i < kLabSegs; i += kRedThreads / 32) {
      const float4 v = p.c.seg[i];
      if ((threadIdx.x & 31) < kRedSegCopies) seg[i * kRedSegCopies + (threadIdx.x & 31)] = v;
    }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) gamma_d[i] = ref::kGammaF64[i];
  __syncthreads();
  const MactErrSpec& s = p.spec;
  const uint32_t lane = threadIdx.x & 31;
  Acc a[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc_init(a[c]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r, g, b;
    if (p.rgb) {
      r = p.rgb[3 * i]; g = p.rgb[3 * i + 1]; b = p.rgb[3 * i + 2];
    } else {
      const uint32_t idx = (uint32_t)((p.cube_start + i) & 0xFFFFFF);
      r = idx >> 16; g = (idx >> 8) & 255u; b = idx & 255u;
    }
    double cand[3], ref[3];
    if (s.candidate == MACT_CAND_FAST) {
      Lab3 v;
      if (s.space == MACT_SPACE_LAB) v = lab_fast_u8(r, g, b, SmemTab<kRedSegCopies>(gamma_rep, seg, lane), p.c);
      else if (s.space == MACT_SPACE_HSI) v = hsi_fast_u8(r, g, b, p.c);
      else v = sct_fast_u8(r, g, b, p.c);
      cand[0] = v.c0; cand[1] = v.c1; cand[2] = v.c2;
    } else if (s.candidate == MACT_CAND_FAST_F64) {        // the reference's own arithmetic
      if (s.space == MACT_SPACE_LAB) ref::lab_fast(gamma_d[r], gamma_d[g], gamma_d[b], p.c, cand);
      else if (s.space == MACT_SPACE_HSI) ref::hsi_fast<true>((double)r, (double)g, (double)b, p.c, cand);
      else ref::sct_fast((double)r, (double)g, (double)b, p.c, cand);
    } else if (s.candidate == MACT_CAND_LUT) {
      if (s.lut_grid_n == 9) lut_value<9>(s.lut_lattice, s.lut_method, r, g, b, cand);
      else if (s.lut_grid_n == 17) lut_value<17>(s.lut_lattice, s.lut_method, r, g, b, cand);
      else lut_value<33>(s.lut_lattice, s.lut_method, r, g, b, cand);
    } else {
      if (s.cand_dtype == MACT_DTYPE_F64) load3<double>(s.cand_array, i, cand);
      else load3<float>(s.cand_array, i, cand);
    }
    if (s.ref_array) {
      if (s.ref_dtype == MACT_DTYPE_F64) load3<double>(s.ref_array, i, ref);
      else load3<float>(s.ref_array, i, ref);
    } else if (s.space == MACT_SPACE_LAB) {
      lab_from_linear(gamma_d[r], gamma_d[g], gamma_d[b], ref);
    } else if (s.space == MACT_SPACE_HSI) {
      hsi_exact_d((double)r, (double)g, (double)b, ref);
    } else {
      sct_exact_d((double)r, (double)g, (double)b, ref);
    }
    const unsigned long long gi = (unsigned long long)(p.index_base + i);
    if constexpr (NC == 1) {
      acc_push(a[0], distance_d(s.space, cand, ref), gi);
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double d = fabs(cand[c] - ref[c]);
        if (s.space == MACT_SPACE_HSI && c == 0) d = fmin(d, kTwoPi - d);
        acc_push(a[c], (isnan(cand[c]) || isnan(ref[c])) ? __longlong_as_double(0x7ff8000000000000ll) : d, gi);
      }
    }
  }
  block_reduce<NC>(a);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      MactErrStats o;
      o.sum = a[c].sum; o.max = a[c].max; o.count = a[c].count; o.argmax = a[c].argmax;
      o.nan_count = a[c].nan; o._pad = 0;
      parts[(size_t)blockIdx.x * NC + c] = o;
    }
  }
}

template <int NC>
__global__ void __launch_bounds__(kRedThreads) k_err_final(const MactErrStats* __restrict__ parts,
                                                           int nblocks, MactErrStats* __restrict__ out) {
  Acc a[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc_init(a[c]);
  // each thread folds a contiguous, fixed block range in order
  const int per = (nblocks + kRedThreads - 1) / kRedThreads;
  const int lo = threadIdx.x * per, hi = min(nblocks, lo + per);
  for (int bk = lo; bk < hi; ++bk) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const MactErrStats& q = parts[(size_t)bk * NC + c];
      Acc b;
      b.sum = q.sum; b.max = q.max; b.count = q.count; b.argmax = q.argmax; b.nan = q.nan_count;
      acc_merge(a[c], b);
    }
  }
  block_reduce<NC>(a);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      MactErrStats o;
      o.sum = a[c].sum; o.max = a[c].max; o.count = a[c].count; o.argmax = a[c].argmax;
      o.nan_count = a[c].nan; o._pad = 0;
      out[c] = o;
    }
  }
}

}  // namespace mact

using namespace mact;

extern "C" size_t mact_err_workspace_bytes(void) {
  return (size_t)kRedMaxBlocks * 3 * sizeof(MactErrStats);
}

extern "C" int mact_err_reduce(const MactErrSpec* spec, const MactCoeffs* c, const uint8_t* rgb,
                               int64_t cube_start, int64_t n, int64_t index_base,
                               MactErrStats* out, void* workspace, void* stream) {
  NvtxRange range("mact_err_reduce");
  if (!spec || !out || !workspace) return set_error(MACT_EBADARG, "bad argument");
  if (spec->space < 0 || spec->space > 2) return set_error(MACT_EBADARG, "unknown space %d", spec->space);
  if (n <= 0) return set_error(MACT_EBADARG, "empty population");
  if (!rgb && cube_start < 0) return set_error(MACT_EBADARG, "no pixels (rgb NULL, cube_start < 0)");
  if (spec->candidate == MACT_CAND_LUT) {
    if (!spec->lut_lattice) return set_error(MACT_EBADARG, "LUT candidate without lattice");
    if (spec->lut_grid_n != 9 && spec->lut_grid_n != 17 && spec->lut_grid_n != 33)
      return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
    if (spec->lut_method < 0 || spec->lut_method > 3)
      return set_error(MACT_EBADARG, "unknown interpolation method %d", spec->lut_method);
  } else if (spec->candidate == MACT_CAND_ARRAY) {
    if (!spec->cand_array) return set_error(MACT_EBADARG, "array candidate without data");
  } else if (spec->candidate != MACT_CAND_FAST && spec->candidate != MACT_CAND_FAST_F64) {
    return set_error(MACT_EBADARG, "unknown candidate kind %d", spec->candidate);
  }
  if (spec->candidate != MACT_CAND_ARRAY && !rgb && cube_start < 0)
    return set_error(MACT_EBADARG, "candidate needs pixels");
  RedParams p;
  p.spec = *spec;
  if (spec->candidate == MACT_CAND_FAST || spec->candidate == MACT_CAND_FAST_F64) {
    if (int rc = make_kcoeffs(c, &p.c)) return rc;
  } else {
    memset(&p.c, 0, sizeof p.c);
  }
  p.rgb = rgb;
  p.cube_start = cube_start;
  p.n = n;
  p.index_base = index_base;
  cudaStream_t st = (cudaStream_t)stream;
  const bool comp = spec->metric == MACT_METRIC_COMPONENT;
  const void* fn = comp ? (const void*)k_err<3> : (const void*)k_err<1>;
  int64_t grid = persistent_grid(fn, kRedThreads, 0);
  if (grid <= 0) return MACT_ECUDA;
  if (grid > kRedMaxBlocks) grid = kRedMaxBlocks;
  const int64_t need = (n + kRedThreads - 1) / kRedThreads;
  if (grid > need) grid = need;
  MactErrStats* parts = (MactErrStats*)workspace;
  if (comp) {
    k_err<3><<<(unsigned)grid, kRedThreads, 0, st>>>(p, parts);
    k_err_final<3><<<1, kRedThreads, 0, st>>>(parts, (int)grid, out);
  } else {
    k_err<1><<<(unsigned)grid, kRedThreads, 0, st>>>(p, parts);
    k_err_final<1><<<1, kRedThreads, 0, st>>>(parts, (int)grid, out);
  }
  count_launch(2);
  return check_launch("err_reduce");
}
