// mact_stream.cuh — persistent, warp-specialised streaming skeleton shared by
// every per-pixel kernel of the path (MACT transforms and LUT interpolators).
//
// Data layout in HBM: packed interleaved uint8 RGB in (3 B/px, the
// reference's (...,3) C-order layout), fp32 out interleaved (N,3) or planar
// (3,N).  The path is HBM-bound (15 B/px algorithmic traffic per transform),
// so data moves with the Blackwell bulk-copy engine (cp.async.bulk, SASS
// UBLKCP) and the SMs only compute:
//
//   * CTA = NW compute warps + 1 producer warp, persistent, grid-stride over
//     tiles of TP = NW * 128 * G pixels;
//   * producer (one lane): streams input tiles global->smem into an SIN-deep
//     ring; full[s] completes on the transaction bytes, empty[s] collects one
//     arrival per compute warp before stage s is refilled;
//   * compute warp w owns the contiguous slice [w*WPX, (w+1)*WPX) of each tile
//     (WPX = 128*G); lane l takes 4-pixel groups g*32 + l: 3 x LDS.32 at a
//     stride of 3 words (conflict-free), results to the warp's own staging
//     buffer with STS.128 (conflict-free), then lane 0 drains the slice with
//     one bulk store per output array (WPX*12 B, or 3 planes of WPX*4 B).
//     Output buffers are NOB-deep per warp and recycled with
//     cp.async.bulk.wait_group.read — no CTA-wide barrier anywhere in the loop.
//
// WAR across proxies: a compute warp arrives on empty[s] only after its
// results derived from stage s were written to smem and made visible to the
// async proxy, so the producer's refill can never overtake a pending LDS.
//
// Tiles that are not whole (the tail) and unaligned buffers go through the
// per-pixel generic kernel.
#pragma once

#include <type_traits>

#include "mact_common.cuh"

namespace mact {

// Op concept:
//   static constexpr int NOUT;              // 1 or 3 output triples per pixel
//   using Params;                           // __grid_constant__ parameter block
//   struct Shared;                          // per-CTA shared state (tables)
//   static __device__ void init(Shared*, const Params&);   // all threads, then __syncthreads
//   static __device__ void px(r, g, b, const Shared*, lane, const Params&, float (*o)[3]);
//   static __device__ void px4w(w0, w1, w2, const Shared*, lane, const Params&,
//                               float (*o)[NOUT][3]);   // 4 packed pixels, warp-converged

struct Outs {
  float* o[3];
};

// Default 4-pixel batch: unpack the three words, four independent px() calls.
template <class Op>
__device__ __forceinline__ void px4_each(uint32_t w0, uint32_t w1, uint32_t w2,
                                         const typename Op::Shared* sh, uint32_t lane,
                                         const typename Op::Params& p, float (*o)[Op::NOUT][3]) {
  Op::px(byte_of(w0, 0), byte_of(w0, 1), byte_of(w0, 2), sh, lane, p, o[0]);
  Op::px(byte_of(w0, 3), byte_of(w1, 0), byte_of(w1, 1), sh, lane, p, o[1]);
  Op::px(byte_of(w1, 2), byte_of(w1, 3), byte_of(w2, 0), sh, lane, p, o[2]);
  Op::px(byte_of(w2, 1), byte_of(w2, 2), byte_of(w2, 3), sh, lane, p, o[3]);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Alignment an Op's Shared block needs in the shared-memory window
// (Shared::kAlign; default 128).  Blocks aligned beyond 128 B are placed at
// a fixed offset computed for the dynamic-smem window starting at
// kDynSmemBase (sm_90 / sm_100 reserve the first 1 KB of every CTA's window);
// the kernels check the resulting address and trap if the assumption breaks.
constexpr uint32_t kDynSmemBase = 0x400;
template <class T, class = void>
struct ShAlign { static constexpr uint32_t v = 128; };
template <class T>
struct ShAlign<T, std::void_t<decltype(T::kAlign)>> { static constexpr uint32_t v = T::kAlign; };

// Optional per-thread context an Op derives once from its staged tables
// (Op::Ctx, Op::ctx(sh, p)) and the streaming kernel keeps in registers for
// the whole tile loop (Op::px4w_ctx); Ops without one use px4w.
template <class Op, class = void>
struct HasCtx : std::false_type {};
template <class Op>
struct HasCtx<Op, std::void_t<typename Op::Ctx>> : std::true_type {};

// Ops that run as 2-CTA clusters (Op::kCluster = true: the pair shares its
// staged tables through distributed shared memory) replace the CTA barrier
// after Op::init with a cluster barrier, and keep every CTA resident until
// its partner is done reading its shared memory.
template <class Op, class = void>
struct IsCluster : std::false_type {};
template <class Op>
struct IsCluster<Op, std::void_t<decltype(Op::kCluster)>> : std::integral_constant<bool, Op::kCluster> {};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class Op, int NW, int G, int SIN, int NOB>
struct WsLayout {
  using Sh = typename Op::Shared;
  static constexpr uint32_t A = ShAlign<Sh>::v;
  static constexpr int WPX = 128 * G;                 // pixels per warp slice
  static constexpr int TP = NW * WPX;                 // pixels per tile
  static constexpr int IN_BYTES = TP * 3;
  static constexpr int OUT_FLOATS = WPX * 3;          // one output array of one slice
  static constexpr size_t in_off = 0;
  static constexpr size_t out_warp = (size_t)NOB * Op::NOUT * OUT_FLOATS * 4;
  // A <= 128: [in stages][out slices][barriers][Shared]
  // A  > 128: [in stages][barriers] ... [Shared at the aligned offset][out slices]
  static constexpr size_t in_end = (size_t)SIN * IN_BYTES;
  static constexpr size_t bar_off = A <= 128 ? in_end + NW * out_warp : in_end;
  static constexpr size_t sh_off = A <= 128 ? (bar_off + 2 * SIN * 8 + 127) / 128 * 128
                                            : (A - kDynSmemBase % A) % A;
  static constexpr size_t out_off = A <= 128 ? in_end : sh_off + sizeof(Sh);
  static constexpr size_t bytes = A <= 128 ? sh_off + sizeof(Sh) : out_off + NW * out_warp;
  static_assert(A <= 128 || bar_off + 2 * SIN * 8 <= sh_off, "stages overlap the aligned tables");
  static constexpr int threads = 32 * (NW + 1);
};
// Shared block of a per-pixel kernel at the start of dynamic smem, aligned at run time.
template <class Op>
__device__ __forceinline__ typename Op::Shared* shared_block(uint8_t* smem) {
  constexpr uint32_t A = ShAlign<typename Op::Shared>::v;
  if constexpr (A <= 128) return reinterpret_cast<typename Op::Shared*>(smem);
  const uint32_t pad = (A - (smem_u32(smem) & (A - 1))) & (A - 1);
  return reinterpret_cast<typename Op::Shared*>(smem + pad);
}
template <class Op>
constexpr size_t shared_block_bytes() {
  constexpr uint32_t A = ShAlign<typename Op::Shared>::v;
  return sizeof(typename Op::Shared) + (A <= 128 ? 0 : A);
}

template <class Op, int NW, int G, int SIN, int NOB>
__global__ void __launch_bounds__(32 * (NW + 1)) k_ws(const uint8_t* __restrict__ in, Outs outs,
                                                       int64_t n, int64_t ntiles, int planar,
                                                       const __grid_constant__ typename Op::Params p) {
  using L = WsLayout<Op, NW, G, SIN, NOB>;
  constexpr int NOUT = Op::NOUT;
  static_assert((L::IN_BYTES % 16) == 0 && (L::OUT_FLOATS * 4) % 16 == 0, "bulk copies need 16 B");
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* in_s = smem + L::in_off;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::bar_off);
  uint64_t* empty = full + SIN;
  auto* sh = reinterpret_cast<typename Op::Shared*>(smem + L::sh_off);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (L::A > 128) {
    if (smem_u32(sh) & (L::A - 1)) __trap();            // window base differs from kDynSmemBase
  }

  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int64_t my_tiles = ntiles > first ? (ntiles - first + stride - 1) / stride : 0;
  // The producer lane initialises the mbarriers and issues the first SIN tile
  // loads before the CTA stages its tables, so the DRAM latency of the first
  // tiles overlaps Op::init (one-tile-per-CTA launches: small images).
  const bool producer = warp == NW && lane == 0;
  const int64_t pre = my_tiles < SIN ? my_tiles : SIN;
  if (producer) {
#pragma unroll
    for (int s = 0; s < SIN; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
    for (int64_t i = 0; i < pre; ++i) {
      mbar_arrive_expect_tx(&full[i], L::IN_BYTES);
      bulk_g2s(in_s + (size_t)i * L::IN_BYTES, in + (first + i * stride) * L::IN_BYTES, L::IN_BYTES, &full[i]);
    }
  }
  Op::init(sh, p);
  constexpr bool CL = IsCluster<Op>::value;
  if constexpr (CL) cluster_sync_all();
  else __syncthreads();

  if (warp == NW) {                                       // ---- producer warp
    if (lane == 0) {
      // ring position (stage s, its use count) maintained incrementally: no
      // 64-bit divisions by SIN in the loop
      int s = (int)(pre % SIN);
      uint32_t ph = (uint32_t)(pre / SIN);
      int64_t t = first + pre * stride;
      for (int64_t i = pre; i < my_tiles; ++i, t += stride) {
        if (i >= SIN) mbar_wait(&empty[s], (ph - 1) & 1);
        mbar_arrive_expect_tx(&full[s], L::IN_BYTES);
        bulk_g2s(in_s + (size_t)s * L::IN_BYTES, in + t * L::IN_BYTES, L::IN_BYTES, &full[s]);
        if (++s == SIN) { s = 0; ++ph; }
      }
    }
    __syncwarp();
    if constexpr (CL) cluster_sync_all();                 // the partner may still read our tables
    return;
  }

  // ---- compute warps
  float* out_w = reinterpret_cast<float*>(smem + L::out_off + warp * L::out_warp);
  const auto ctx = [&] {
    if constexpr (HasCtx<Op>::value) return Op::ctx(sh, p);
    else return 0;
  }();
  int s = 0, ob = 0;                                      // ring stage and output buffer of tile i
  uint32_t ph = 0;                                        // use count of stage s, mod 2
  int64_t t = first;
  for (int64_t i = 0; i < my_tiles; ++i, t += stride) {
    float* ob_s = out_w + (size_t)ob * NOUT * L::OUT_FLOATS;
    if (lane == 0) bulk_wait_read<NOB - 1>();             // this buffer's last store has read it
    __syncwarp();
    mbar_wait(&full[s], ph & 1);
    const uint32_t* wsrc =
        reinterpret_cast<const uint32_t*>(in_s + (size_t)s * L::IN_BYTES) + warp * (L::WPX / 4) * 3;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int grp = g * 32 + (int)lane;                 // 4-pixel group inside the warp slice
      float o[4][NOUT][3];
      if constexpr (HasCtx<Op>::value)
        Op::px4w_ctx(wsrc[3 * grp], wsrc[3 * grp + 1], wsrc[3 * grp + 2], sh, lane, p, ctx, o);
      else
        Op::px4w(wsrc[3 * grp], wsrc[3 * grp + 1], wsrc[3 * grp + 2], sh, lane, p, o);
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
            *reinterpret_cast<float4*>(base + c * L::WPX + grp * 4) =
                make_float4(o[0][k][c], o[1][k][c], o[2][k][c], o[3][k][c]);
        }
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      const int64_t px0 = t * L::TP + (int64_t)warp * L::WPX;
#pragma unroll
      for (int k = 0; k < NOUT; ++k) {
        float* dst = outs.o[k];
        if (dst == nullptr) continue;
        const float* src = ob_s + k * L::OUT_FLOATS;
        if (!planar) {
          bulk_s2g(dst + px0 * 3, src, L::WPX * 12);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) bulk_s2g(dst + c * n + px0, src + c * L::WPX, L::WPX * 4);
        }
      }
      bulk_commit();
      mbar_arrive(&empty[s]);                             // stage s fully consumed by this warp
    }
    if (++s == SIN) { s = 0; ++ph; }
    if constexpr (NOB > 1) ob = ob + 1 == NOB ? 0 : ob + 1;
  }
  if (lane == 0) bulk_wait<0>();
  __syncwarp();
  if constexpr (CL) cluster_sync_all();
}

// Per-pixel fallback for the tail tile and unaligned buffers.
template <class Op, int NT>
__global__ void __launch_bounds__(NT) k_generic(const uint8_t* __restrict__ in, Outs outs,
                                                 int64_t start, int64_t n, int planar,
                                                 const __grid_constant__ typename Op::Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  auto* sh = shared_block<Op>(smem);
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

// Small inputs (one image of a few Mpx): no producer warp, no mbarriers, no
// staging -- each thread loads its 4 pixels (3 words), runs Op::px4w and
// stores 3 float4, so the latency of a launch is one DRAM round trip plus
// the arithmetic.  Interleaved output, 16-byte aligned buffers, n % 4 == 0.
template <class Op, int NT>
__global__ void __launch_bounds__(NT) k_direct(const uint8_t* __restrict__ in, Outs outs, int64_t ngroups,
                                               const __grid_constant__ typename Op::Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  auto* sh = shared_block<Op>(smem);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(in);
  const int64_t stride = (int64_t)gridDim.x * NT;
  int64_t gi = blockIdx.x * (int64_t)NT + threadIdx.x;
  // the first group's loads are in flight while the CTA stages its tables
  uint32_t w0 = 0, w1 = 0, w2 = 0;
  if (gi < ngroups) { w0 = __ldg(w + 3 * gi); w1 = __ldg(w + 3 * gi + 1); w2 = __ldg(w + 3 * gi + 2); }
  Op::init(sh, p);
  __syncthreads();
  for (; gi < ngroups; gi += stride) {
    float o[4][Op::NOUT][3];
    Op::px4w(w0, w1, w2, sh, lane, p, o);
    if (gi + stride < ngroups) {
      const uint32_t* q = w + 3 * (gi + stride);
      w0 = __ldg(q); w1 = __ldg(q + 1); w2 = __ldg(q + 2);
    }
#pragma unroll
    for (int k = 0; k < Op::NOUT; ++k) {
      if (outs.o[k] == nullptr) continue;
      float4* d = reinterpret_cast<float4*>(outs.o[k] + 12 * gi);
      d[0] = make_float4(o[0][k][0], o[0][k][1], o[0][k][2], o[1][k][0]);
      d[1] = make_float4(o[1][k][1], o[1][k][2], o[2][k][0], o[2][k][1]);
      d[2] = make_float4(o[2][k][2], o[3][k][0], o[3][k][1], o[3][k][2]);
    }
  }
}

template <class Op, int NT>
inline int launch_direct(const uint8_t* in, Outs outs, int64_t n, const typename Op::Params& p,
                         cudaStream_t st, const char* name) {
  NvtxRange range(name);
  auto kfn = k_direct<Op, NT>;
  const size_t sb = shared_block_bytes<Op>();
  const int64_t cap = persistent_grid((const void*)kfn, NT, sb);
  if (cap <= 0) return MACT_ECUDA;
  const int64_t ngroups = n / 4;
  int64_t grid = (ngroups + NT - 1) / NT;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  kfn<<<(unsigned)grid, NT, sb, st>>>(in, outs, ngroups, p);
  count_launch();
  return check_launch(name);
}

// Host launcher: whole tiles on k_ws, the remainder (or everything, when a
// buffer is not 16-byte aligned) on k_generic.
template <class Op, int NW, int G, int SIN, int NOB>
inline int launch_stream_t(const uint8_t* in, Outs outs, int64_t n, int planar,
                           const typename Op::Params& p, cudaStream_t st, const char* name) {
  if (n <= 0) return MACT_OK;
  NvtxRange range(name);
  using L = WsLayout<Op, NW, G, SIN, NOB>;
  bool aligned = ((uintptr_t)in % 16) == 0;
  for (int k = 0; k < Op::NOUT; ++k)
    if (outs.o[k] && ((uintptr_t)outs.o[k] % 16) != 0) aligned = false;
  if (planar && (n % 4) != 0) aligned = false;
  const int64_t ntiles = aligned ? n / L::TP : 0;
  if constexpr (L::A > 128) {   // the aligned-table layout assumes kDynSmemBase (the kernel traps otherwise)
    if (reserved_smem() != (int)kDynSmemBase)
      return set_error(MACT_ECUDA, "%s: %d B reserved shared memory per block, layout assumes %u", name,
                       reserved_smem(), kDynSmemBase);
  }
  if (ntiles > 0) {
    auto kfn = k_ws<Op, NW, G, SIN, NOB>;
    int64_t grid = persistent_grid((const void*)kfn, L::threads, L::bytes);
    if (grid <= 0) return MACT_ECUDA;
    if (grid > ntiles) grid = ntiles;
    kfn<<<(unsigned)grid, L::threads, L::bytes, st>>>(in, outs, n, ntiles, planar, p);
    count_launch();
    if (int rc = check_launch(name)) return rc;
  }
  const int64_t done = ntiles * L::TP;
  if (done < n) {
    auto kfn = k_generic<Op, 256>;
    const size_t sb = shared_block_bytes<Op>();
    const int64_t cap = persistent_grid((const void*)kfn, 256, sb);
    if (cap <= 0) return MACT_ECUDA;
    int64_t grid = (n - done + 255) / 256;
    if (grid > cap) grid = cap;
    kfn<<<(unsigned)grid, 256, sb, st>>>(in, outs, done, n, planar, p);
    count_launch();
    return check_launch(name);
  }
  return MACT_OK;
}

}  // namespace mact
