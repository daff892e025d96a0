// mact_stream.cuh — persistent streaming skeleton shared by every per-pixel
// kernel of the path (MACT transforms and LUT interpolators).
//
// Data layout in HBM: packed interleaved uint8 RGB in (3 B/px, the
// reference's (...,3) C-order layout), fp32 out interleaved (N,3) or planar
// (3,N).  The path is HBM-bound (15 B/px algorithmic traffic per transform),
// so the kernel is built around the Blackwell bulk-copy engine:
//
//   * one CTA per SM slot, grid-stride over tiles of TP pixels;
//   * thread 0 streams input tiles global->smem with cp.async.bulk into an
//     SIN-deep mbarrier ring (3*TP bytes each, no register staging, no LSU
//     instructions for the loads);
//   * all threads read their 4-pixel groups from smem (3 x LDS.32, stride-3
//     words: conflict-free), compute, and write fp32 results to one of two
//     output staging buffers (STS.128, conflict-free);
//   * thread 0 drains each output tile smem->global with cp.async.bulk
//     bulk_group stores (12*TP bytes per output, 4*TP per plane), double
//     buffered against compute with wait_group.read.
//
// Tiles that are not whole (the tail) and unaligned buffers go through the
// per-pixel generic kernel.
#pragma once

#include "mact_common.cuh"

namespace mact {

// Op concept:
//   static constexpr int NOUT;              // 1 or 3 output triples per pixel
//   using Params;                           // __grid_constant__ parameter block
//   struct Shared;                          // per-CTA shared state (tables)
//   static __device__ void init(Shared*, const Params&);   // all threads, then __syncthreads
//   static __device__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared*,
//                             uint32_t lane, const Params&, float (*o)[3]);

struct Outs {
  float* o[3];
};

template <class Op, int TP, int SIN>
struct StreamSmem {
  static constexpr int IN_BYTES = TP * 3;
  static constexpr int OUT_FLOATS = TP * 3;                    // per output triple-array
  static constexpr size_t in_off = 0;
  static constexpr size_t out_off = (size_t)SIN * IN_BYTES;
  static constexpr size_t bar_off = out_off + 2ull * Op::NOUT * OUT_FLOATS * 4;
  static constexpr size_t sh_off = (bar_off + SIN * 8 + 127) / 128 * 128;
  static constexpr size_t bytes = sh_off + sizeof(typename Op::Shared);
};

template <class Op, int TP, int NT, int SIN>
__global__ void __launch_bounds__(NT) k_stream(const uint8_t* __restrict__ in, Outs outs,
                                                int64_t n, int64_t ntiles, int planar,
                                                const __grid_constant__ typename Op::Params p) {
  using L = StreamSmem<Op, TP, SIN>;
  constexpr int NOUT = Op::NOUT;
  constexpr int G = TP / (4 * NT);                 // 4-pixel groups per thread per tile
  static_assert(TP % (4 * NT) == 0, "tile must split into 4-pixel groups");
  static_assert((TP * 3) % 16 == 0, "bulk copies need 16-byte multiples");
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* in_s = smem + L::in_off;
  float* out_s = reinterpret_cast<float*>(smem + L::out_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bar_off);
  auto* sh = reinterpret_cast<typename Op::Shared*>(smem + L::sh_off);
  const uint32_t tid = threadIdx.x, lane = tid & 31;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < SIN; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  Op::init(sh, p);
  __syncthreads();

  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t my_tiles = ntiles > first ? (ntiles - first + stride - 1) / stride : 0;
  if (tid == 0) {
    for (int s = 0; s < SIN && s < my_tiles; ++s) {
      const int64_t t = first + s * stride;
      mbar_arrive_expect_tx(&bars[s], L::IN_BYTES);
      bulk_g2s(in_s + s * L::IN_BYTES, in + t * L::IN_BYTES, L::IN_BYTES, &bars[s]);
    }
  }

  for (int64_t i = 0; i < my_tiles; ++i) {
    const int64_t t = first + i * stride;
    const int s = (int)(i % SIN);
    mbar_wait(&bars[s], (uint32_t)((i / SIN) & 1));
    const uint32_t* wsrc = reinterpret_cast<const uint32_t*>(in_s + s * L::IN_BYTES);
    uint32_t w[G][3];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int q = (g * NT + (int)tid) * 3;
      w[g][0] = wsrc[q];
      w[g][1] = wsrc[q + 1];
      w[g][2] = wsrc[q + 2];
    }
    const int ob = (int)(i & 1);
    if (tid == 0) bulk_wait_read<1>();            // tile i-2's stores have read buffer ob
    __syncthreads();                              // input stage s consumed; buffer ob free
    if (tid == 0 && i + SIN < my_tiles) {
      const int64_t tn = first + (i + SIN) * stride;
      mbar_arrive_expect_tx(&bars[s], L::IN_BYTES);
      bulk_g2s(in_s + s * L::IN_BYTES, in + tn * L::IN_BYTES, L::IN_BYTES, &bars[s]);
    }
    float* ob_s = out_s + (size_t)ob * NOUT * L::OUT_FLOATS;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t w0 = w[g][0], w1 = w[g][1], w2 = w[g][2];
      float o[4][NOUT][3];
      Op::px(byte_of(w0, 0), byte_of(w0, 1), byte_of(w0, 2), sh, lane, p, o[0]);
      Op::px(byte_of(w0, 3), byte_of(w1, 0), byte_of(w1, 1), sh, lane, p, o[1]);
      Op::px(byte_of(w1, 2), byte_of(w1, 3), byte_of(w2, 0), sh, lane, p, o[2]);
      Op::px(byte_of(w2, 1), byte_of(w2, 2), byte_of(w2, 3), sh, lane, p, o[3]);
      const int grp = g * NT + (int)tid;          // 4-pixel group index inside the tile
#pragma unroll
      for (int k = 0; k < NOUT; ++k) {
        float* base = ob_s + k * L::OUT_FLOATS;
        if (!planar) {
          float4* d = reinterpret_cast<float4*>(base + grp * 12);
          d[0] = make_float4(o[0][k][0], o[0][k][1], o[0][k][2], o[1][k][0]);
          d[1] = make_float4(o[1][k][1], o[1][k][2], o[2][k][0], o[2][k][1]);
          d[2] = make_float4(o[2][k][2], o[3][k][0], o[3][k][1], o[3][k][2]);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            *reinterpret_cast<float4*>(base + c * TP + grp * 4) =
                make_float4(o[0][k][c], o[1][k][c], o[2][k][c], o[3][k][c]);
        }
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < NOUT; ++k) {
        float* dst = outs.o[k];
        if (dst == nullptr) continue;
        const float* src = ob_s + k * L::OUT_FLOATS;
        if (!planar) {
          bulk_s2g(dst + t * (int64_t)TP * 3, src, TP * 12);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) bulk_s2g(dst + c * n + t * (int64_t)TP, src + c * TP, TP * 4);
        }
      }
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait<0>();
}

// Per-pixel fallback for the tail tile and unaligned buffers.
template <class Op, int NT>
__global__ void __launch_bounds__(NT) k_generic(const uint8_t* __restrict__ in, Outs outs,
                                                 int64_t start, int64_t n, int planar,
                                                 const __grid_constant__ typename Op::Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  auto* sh = reinterpret_cast<typename Op::Shared*>(smem);
  Op::init(sh, p);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  for (int64_t i = start + blockIdx.x * (int64_t)NT + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * NT) {
    const uint8_t* q = in + 3 * i;
    float o[Op::NOUT][3];
    Op::px(q[0], q[1], q[2], sh, lane, p, o);
#pragma unroll
    for (int k = 0; k < Op::NOUT; ++k) {
      float* dst = outs.o[k];
      if (dst == nullptr) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (planar) dst[c * n + i] = o[k][c];
        else dst[3 * i + c] = o[k][c];
      }
    }
  }
}

// Host launcher: persistent bulk-copy kernel over whole tiles, generic kernel
// for the tail (or everything, when a buffer is not 16-byte aligned).
template <class Op, int TP, int NT, int SIN>
inline int launch_stream_t(const uint8_t* in, Outs outs, int64_t n, int planar,
                         const typename Op::Params& p, cudaStream_t st, const char* name) {
  if (n <= 0) return MACT_OK;
  using L = StreamSmem<Op, TP, SIN>;
  bool aligned = ((uintptr_t)in % 16) == 0;
  for (int k = 0; k < Op::NOUT; ++k) {
    if (outs.o[k] && ((uintptr_t)outs.o[k] % 16) != 0) aligned = false;
  }
  if (planar && (n % 4) != 0) aligned = false;
  int64_t ntiles = aligned ? n / TP : 0;
  if (ntiles > 0) {
    auto kfn = k_stream<Op, TP, NT, SIN>;
    int64_t grid = persistent_grid((const void*)kfn, NT, L::bytes);
    if (grid <= 0) return MACT_ECUDA;
    if (grid > ntiles) grid = ntiles;
    kfn<<<(unsigned)grid, NT, L::bytes, st>>>(in, outs, n, ntiles, planar, p);
    count_launch();
    int rc2 = check_launch(name);
    if (rc2) return rc2;
  }
  const int64_t done = ntiles * TP;
  if (done < n) {
    const int64_t rem = n - done;
    auto kfn = k_generic<Op, 256>;
    const size_t sb = sizeof(typename Op::Shared);
    const int64_t cap = persistent_grid((const void*)kfn, 256, sb);
    if (cap <= 0) return MACT_ECUDA;
    int64_t grid = (rem + 255) / 256;
    if (grid > cap) grid = cap;
    kfn<<<(unsigned)grid, 256, sb, st>>>(in, outs, done, n, planar, p);
    count_launch();
    return check_launch(name);
  }
  return MACT_OK;
}

}  // namespace mact
