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
// persistent CTA into shared memory: 9^3 as 8 bank-private float4 copies
// (conflict-free LDS.128), 17^3 as 64-bit fixed-point nodes (LutQuant below:
// one LDS.64 per node, 38 KB) or, for lattices whose value range is too wide
// for that format, as two planes, (c0, c1) float2 and c2 float (59 KB): one
// LDS.64 + one LDS.32 per node.  Random gathers are bank-conflict bound: on
// B200 a random warp LDS.64 costs 5.2 smem cycles, LDS.64 + LDS.32 7.9, one
// LDS.128 of a padded float4 node 9.4 (tools/ldsbench.cu).  33^3 exceeds a
// CTA's 227 KB even as fixed-point nodes (287 KB): CTAs come in pairs, each
// holding half of the r-planes (148 KB) and interpolating the pixels whose
// cell lies in its half, results scattered straight to global memory
// (k_lut33_split; the cluster version with a DSMEM exchange, k_lut33_pair, and
// the component-split CTAs, k_lut33_comp / k_lut33_planar, remain selectable).
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include <cooperative_groups.h>

#include "mact_lut.cuh"
#include "mact_pixel.cuh"
#include "mact_stream.cuh"

#ifndef MACT_LUT_NW
#define MACT_LUT_NW 16
#endif
#ifndef MACT_LUT_NW_TRI17     // 17^3 trilinear (93 KB pair lattice, one CTA per SM): 24 or 31 warps measured slower (138 vs 153 Gpix/s)
#define MACT_LUT_NW_TRI17 16
#endif
#ifndef MACT_LUT_SIN
#define MACT_LUT_SIN 3
#endif
// 17^3 tile shape (R02 sweep on C3, tri / prism / pyr / tet): G = 2 groups of 128 pixels per warp and tile
// 162 / 174 / 196 / 226 against 156 / 176 / 199 / 230 for G = 1, so trilinear (one CTA per SM) takes 2 and the
// others 1; two output staging buffers per warp (NOB = 2) 171 / 192 / 222: slower; SIN = 2 with NOB = 2 the same.
#ifndef MACT_LUT_G
#define MACT_LUT_G 1
#endif
#ifndef MACT_LUT_G_TRI17      // with G = 2: 12 / 20 / 24 warps 144 / 146 / 149 against 162 Gpix/s for 16
#define MACT_LUT_G_TRI17 2
#endif
#ifndef MACT_LUT_NOB
#define MACT_LUT_NOB 1
#endif
#ifndef MACT_LUT33_TRI_PB
#define MACT_LUT33_TRI_PB 1
#endif

namespace mact {

struct LutParams {
  const float4* lat;   // (n^3, 4) fp32, r-major, padded
};

// ---------------------------------------------- 64-bit fixed-point lattice
// Node = (q0 | q1 << 21 | q2 << 42), q_c in 21 / 21 / 22 bits, value
// v_c = lo_c + S_c q_c.  Decoding ORs q_c into the mantissa of 2^23 (exact
// float F = 2^23 + q_c) and takes ONE fma: fmaf(F, S_c, K_c) with
// K_c = lo_c - S_c 2^23 chosen exactly representable (rounded down from
// min_c - S_c 2^23, so lo_c <= min_c), i.e. S_c q_c + lo_c rounded once.
// Enabled only when every half-step S_c / 2 <= kLutQuantTol (CIELAB 17^3:
// 2.4e-5 / 4.4e-5 / 2.4e-5 on L*, a*, b*), so an interpolated value moves by
// at most sum|w| * 4.4e-5 (sum|w| = 1 for trilinear / prism / tetrahedral,
// <= 1.5 for the pyramid) -- inside the 1e-4 north-star tolerance.  Other
// lattices (wider ranges, non-finite values) keep the fp32 planes.
constexpr double kLutQuantTol = 5e-5;
struct LutQuant {
  float s[3], k[3];
  float s255[3];   // S_c / 255 (the 17^3 trilinear lerps scale code differences by S_c rb / 255)
  int on;
};
// q_c = rint((v_c - lo_c) / S_c), the quotient taken as a product with the
// fp64 reciprocal (|error| ~1e-9 codes: any rounding of it keeps |v - v'| <=
// S_c / 2 + 1e-9 S_c); identical in every CTA.
__device__ __forceinline__ uint2 lut_quant_pack(const LutQuant& q, float4 v) {
  const double lo0 = (double)q.k[0] + (double)q.s[0] * 8388608.0;
  const double lo1 = (double)q.k[1] + (double)q.s[1] * 8388608.0;
  const double lo2 = (double)q.k[2] + (double)q.s[2] * 8388608.0;
  const uint32_t q0 = (uint32_t)__double2uint_rn(((double)v.x - lo0) * (1.0 / (double)q.s[0]));
  const uint32_t q1 = (uint32_t)__double2uint_rn(((double)v.y - lo1) * (1.0 / (double)q.s[1]));
  const uint32_t q2 = (uint32_t)__double2uint_rn(((double)v.z - lo2) * (1.0 / (double)q.s[2]));
  return make_uint2(q0 | (q1 << 21), (q1 >> 11) | (q2 << 10));
}
// A node as (c0, c1) + c2, so the (c0, c1) pair can use Blackwell's packed
// fp32x2 FMA (FFMA2: one issue, each lane rounded exactly like FFMA).
struct Node2 {
  float2 xy;
  float z;
};
// (x & 0x1FFFFF) | 0x4B000000 as ONE LOP3: with both constants visible ptxas
// emits two LOP3 (an instruction takes one immediate), so the magic comes from
// constant memory, which it does not fold -- it is loaded into a register once
// per kernel.  Read-only, never written.
#ifndef MACT_LUT_FUSED_LOP
#define MACT_LUT_FUSED_LOP 1
#endif
static __constant__ uint32_t kLutMagic23 = 0x4B000000u;
__device__ __forceinline__ uint32_t lut_field21(uint32_t x) {
#if MACT_LUT_FUSED_LOP
  uint32_t r;
  asm("lop3.b32 %0, %1, 0x1FFFFF, %2, 0xEA;" : "=r"(r) : "r"(x), "r"(kLutMagic23));
  return r;
#else
  return (x & 0x1FFFFFu) | 0x4B000000u;
#endif
}
__device__ __forceinline__ uint32_t mad_hi_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;   // hi(a * b) + c on the FMA pipe (IMAD.HI), where a shift + add would take the ALU pipe
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
// F_c = 2^23 + q_c of one node (exact floats), the integer part of the decode below.
__device__ __forceinline__ void lut_quant_f(uint2 w, float2& f01, float& f2) {
  uint32_t t0;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(t0) : "r"(w.x), "r"(1u << 11));
  f01.x = __uint_as_float(mad_hi_u32(t0, 1u << 21, 0x4B000000u));
  f01.y = __uint_as_float(lut_field21(__funnelshift_r(w.x, w.y, 21)));
  f2 = __uint_as_float(mad_hi_u32(w.y, 1u << 22, 0x4B000000u));
}
__device__ __forceinline__ Node2 lut_quant_unpack2(const LutQuant& q, uint2 w) {
  // The kernel is ALU-pipe bound, so q0 and q2 are extracted on the FMA pipe
  // (IMAD / IMAD.HI) rather than with LOP3 / SHF: 17^3 tetrahedral +5 %.
  // (ptxas turns these mad.hi by powers of two into LEA.HI; forcing IMAD.HI measured slower)
  uint32_t t0;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(t0) : "r"(w.x), "r"(1u << 11));       // q0 to the top bits
  const float f0 = __uint_as_float(mad_hi_u32(t0, 1u << 21, 0x4B000000u));
  // (q1 on the FMA pipe as well -- three IMADs -- measured within +-1 %: kept on the ALU)
  const float f1 = __uint_as_float(lut_field21(__funnelshift_r(w.x, w.y, 21)));
  const float f2 = __uint_as_float(mad_hi_u32(w.y, 1u << 22, 0x4B000000u));   // (w.y >> 10) + 2^23 bits
  Node2 n;
  n.xy = __ffma2_rn(make_float2(f0, f1), make_float2(q.s[0], q.s[1]), make_float2(q.k[0], q.k[1]));
  n.z = fmaf(f2, q.s[2], q.k[2]);
  return n;
}
// Per-component min / max of the lattice (block reduction, exact) and the
// quantisation parameters; all threads of the CTA, ends with __syncthreads.
__device__ __forceinline__ void lut_quant_setup(const float4* lat, int nn, LutQuant* out, float (*red)[6]) {
  float m[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  bool finite = true;
  for (int i = threadIdx.x; i < nn; i += blockDim.x) {
    const float4 v = __ldg(lat + i);
    finite &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z);
    m[0] = fminf(m[0], v.x); m[1] = fminf(m[1], v.y); m[2] = fminf(m[2], v.z);
    m[3] = fmaxf(m[3], v.x); m[4] = fmaxf(m[4], v.y); m[5] = fmaxf(m[5], v.z);
  }
  if (!finite) m[0] = NAN;
  const int any_nan = __syncthreads_or(!finite);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const float x = __shfl_xor_sync(0xffffffffu, m[c], o);
      m[c] = c < 3 ? fminf(m[c], x) : fmaxf(m[c], x);
    }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < 6; ++c) red[warp][c] = m[c];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w)
      for (int c = 0; c < 6; ++c) m[c] = c < 3 ? fminf(m[c], red[w][c]) : fmaxf(m[c], red[w][c]);
    LutQuant q;
    q.on = !any_nan;
    const int bits[3] = {21, 21, 22};
    for (int c = 0; c < 3; ++c) {
      const double lo = m[c], range = (double)m[c + 3] - lo;
      // two spare codes: lo_c sits below min_c by less than one step
      const float sc = __double2float_ru(fmax(range, 1e-30) / (double)((1u << bits[c]) - 3u));
      const float kc = __double2float_rd(lo - (double)sc * 8388608.0);
      q.s[c] = sc;
      q.k[c] = kc;
      q.s255[c] = (float)((double)sc / 255.0);
      const double top = ((double)m[c + 3] - ((double)kc + (double)sc * 8388608.0)) / (double)sc;
      if (!((double)sc * 0.5 <= kLutQuantTol) || !isfinite(kc) || !(top <= (double)(1u << bits[c]) - 1.5))
        q.on = 0;
    }
    *out = q;
  }
  __syncthreads();
}

template <int N, int METHOD>
struct OpLut {
  static constexpr int NOUT = 1;
  static constexpr bool SMEM = N <= 17;
  using Params = LutParams;
  // 9^3: bank-private copies.  An LDS.128 warp access is served 8 lanes per
  // phase, one 16-byte bank group per lane when conflict-free; node i of lane
  // slot k = lane & 7 lives at float4 index 8 i + k, so the 8 lanes of a
  // phase always hit 8 different groups (8 x 729 x 16 B = 93 KB).  (The
  // fixed-point node below with 16 copies -- conflict-free LDS.64 -- was
  // measured slower here: 172-229 against 210-308 Gpix/s; without conflicts
  // to save, the decode's 8 integer/FMA ops per node cost more issue.)
  static constexpr bool PRIV = N <= 9;
  // 17^3: 64-bit fixed-point nodes when the lattice's value ranges allow it
  // (LutQuant; one LDS.64 per node instead of LDS.64 + LDS.32), else the
  // fp32 planes.  The choice is made per CTA from the lattice itself, by the
  // same deterministic arithmetic in every CTA.
  static constexpr bool PACK = SMEM && !PRIV;
  // 17^3 trilinear: b-pair entries e = (node e, node e + 1), 16 bytes, so the 8
  // corners of a cell are 4 LDS.128 (random LDS.128 9.4 smem cycles against
  // 2 x 5.2 for the two LDS.64 it replaces) and the interpolation runs as 7
  // lerps instead of 8 weight products (tri_px below).
  static constexpr bool PAIR = PACK && METHOD == MACT_LUT_TRILINEAR;
  // Cell location is the reference's (lut.py:98-105): for byte pixels
  // min(p (n-1) div 255, n-2) is the shift p >> 4 (lut_locate), p = 255 in cell
  // n-2 at offset 255 -- no clamp, no ghost planes (R01 staged 18^3 nodes to
  // avoid the clamp of the /255 magic; the shift needs neither).
  static constexpr int NG = N;
  static constexpr int NNG = NG * NG * NG;
  static __device__ __forceinline__ void locate_g(uint32_t r, uint32_t g, uint32_t b, int& bf, int& rr,
                                                  int& rg, int& rb) {
    int br, bg, bb;
    lut_locate<N>(r, br, rr);
    lut_locate<N>(g, bg, rg);
    lut_locate<N>(b, bb, rb);
    bf = (br * NG + bg) * NG + bb;
  }
  struct Shared {
    float4 lat[PRIV ? 8 * N * N * N : 1];
    union {
      struct {
        float2 c01[PACK ? NNG : 1];
        float c2[PACK ? NNG : 1];
      } f;
      uint2 pk[PACK && !PAIR ? NNG : 1];
      uint4 pk2[PAIR ? NNG : 1];
    } u;
    LutQuant q;
    float red[32][6];
  };
  static __device__ __forceinline__ void init(Shared* s, const Params& p) {
    if constexpr (PRIV) {
      for (int i = threadIdx.x; i < 8 * N * N * N; i += blockDim.x) s->lat[i] = __ldg(p.lat + (i >> 3));
    } else if constexpr (PACK) {
      lut_quant_setup(p.lat, N * N * N, &s->q, s->red);   // ends with __syncthreads
      const LutQuant q = s->q;
      for (int i = threadIdx.x; i < NNG; i += blockDim.x) {
        const float4 v = __ldg(p.lat + i);
        if (q.on && PAIR) {   // node i and its b neighbour (the last b plane pairs with itself; never used)
          const float4 v1 = __ldg(p.lat + min(i + 1, NNG - 1));
          const uint2 a = lut_quant_pack(q, v), b = lut_quant_pack(q, v1);
          s->u.pk2[i] = make_uint4(a.x, a.y, b.x, b.y);
        } else if (q.on) {
          s->u.pk[i] = lut_quant_pack(q, v);
        } else {
          s->u.f.c01[i] = make_float2(v.x, v.y);
          s->u.f.c2[i] = v.z;
        }
      }
    }
  }
  // PK: the CTA's lattice is in the fixed-point format (decided once per call site, not per node)
  template <bool PK = false>
  static __device__ __forceinline__ Node2 node(const Shared* s, const Params& p, int i, uint32_t lane,
                                               const LutQuant& q) {
    MACT_DCHECK(i >= 0 && i < (PRIV || !SMEM ? N * N * N : NNG));
    if constexpr (PRIV) {
      const float4 v = s->lat[(i << 3) | (lane & 7)];
      return Node2{make_float2(v.x, v.y), v.z};
    } else if constexpr (PACK) {   // 32-bit shared addresses: one LEA per node
      if constexpr (PK) {
        uint2 w;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y)
                     : "r"(smem_u32(s->u.pk) + ((uint32_t)i << 3)));
        return lut_quant_unpack2(q, w);
      }
      float2 v;
      asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y)
                   : "r"(smem_u32(s->u.f.c01) + ((uint32_t)i << 3)));
      return Node2{v, lds_f32(smem_u32(s->u.f.c2) + ((uint32_t)i << 2))};
    } else {
      const float4 v = __ldg(p.lat + i);
      return Node2{make_float2(v.x, v.y), v.z};
    }
  }
  static __device__ __forceinline__ LutQuant quant(const Shared* s) {
    if constexpr (PACK) return s->q;
    else return LutQuant{};
  }
  // Cell location and node selection of one pixel exactly as the interpolation
  // kernels run it (mact_lut_nodes_timed emits them for the parity tests): the
  // reference's cell, the reference's simplex; only the tetrahedral zero-weight
  // middle node under ties may be another corner (lut_nodes_at, TIES = false).
  template <bool = true>
  static __device__ __forceinline__ void select(uint32_t r, uint32_t g, uint32_t b,
                                                int (&idx)[LutK<METHOD>::K], float (&w)[LutK<METHOD>::K]) {
    lut_nodes<N, METHOD, float, false>(r, g, b, idx, w);
  }
  static __device__ __forceinline__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared* s,
                                            uint32_t lane, const Params& p, float (*o)[3]) {
    constexpr int K = LutK<METHOD>::K;
    int idx[K];
    float w[K];
    const LutQuant q = quant(s);
    if constexpr (PAIR) {
      if (q.on) {
        const uint32_t c[1][3] = {{r, g, b}};
        tri_px<1>(c, s, q, o);
        return;
      }
    }
    if (q.on) select<true>(r, g, b, idx, w);
    else select<false>(r, g, b, idx, w);
    auto nd = [&](int i) { return q.on ? node<true>(s, p, i, lane, q) : node<false>(s, p, i, lane, q); };
    Node2 v = nd(idx[0]);
    float2 a01 = __fmul2_rn(make_float2(w[0], w[0]), v.xy);
    float a2 = w[0] * v.z;
#pragma unroll
    for (int j = 1; j < K; ++j) {   // out += w_j V[node_j], node order (lut.py:233-236); FFMA2 = two FFMAs
      v = nd(idx[j]);
      a01 = __ffma2_rn(make_float2(w[j], w[j]), v.xy, a01);
      a2 = fmaf(w[j], v.z, a2);
    }
    o[0][0] = a01.x; o[0][1] = a01.y; o[0][2] = a2;
  }
  // 4 pixels: all node indices first, then every node load, then the FMAs, so
  // 4*K independent gathers are in flight per thread (L2 latency for 33^3,
  // LDS latency for the smem lattice).  Trilinear (K = 8) goes 2 pixels at a
  // time to bound register pressure.
  using Ctx = LutQuant;   // kept in registers by the streaming kernel
  static __device__ __forceinline__ Ctx ctx(const Shared* s, const Params&) { return quant(s); }
  static __device__ __forceinline__ void px4w_ctx(uint32_t w0, uint32_t w1, uint32_t w2,
                                                  const Shared* s, uint32_t lane, const Params& p,
                                                  const Ctx& qt, float (*o)[1][3]) {
    if constexpr (PAIR) {
      if (qt.on) {
        const uint32_t c[4][3] = {{byte_of(w0, 0), byte_of(w0, 1), byte_of(w0, 2)},
                                  {byte_of(w0, 3), byte_of(w1, 0), byte_of(w1, 1)},
                                  {byte_of(w1, 2), byte_of(w1, 3), byte_of(w2, 0)},
                                  {byte_of(w2, 1), byte_of(w2, 2), byte_of(w2, 3)}};
        float r[4][3];
        tri_px<4>(c, s, qt, r);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          o[t][0][0] = r[t][0]; o[t][0][1] = r[t][1]; o[t][0][2] = r[t][2];
        }
        return;
      }
    }
    if (PACK && qt.on) px4w_t<PACK>(w0, w1, w2, s, lane, p, qt, o);
    else px4w_t<false>(w0, w1, w2, s, lane, p, qt, o);
  }
  // 17^3 trilinear on the b-pair entries.  Along b the lerp runs on the codes:
  // D = F(b-node) - F(a-node) is exact (integers below 2^24), so
  //   P_c = (S_c F_a + K_c) + (S_c rb / 255) D_c
  // is the decoded a-node plus one rounded correction; then g and r lerp the
  // decoded values, P0 + t (P1 - P0).  Rounding stays far below the fixed-point
  // half-step.  All loads of the batch are issued before any math.
  template <int PB>
  static __device__ __forceinline__ void tri_px(const uint32_t (&c)[PB][3], const Shared* s, const LutQuant& q,
                                                float (*o)[3]) {
    constexpr uint32_t SR = NG * NG * 16u, SG = NG * 16u;   // byte strides of the pair entries
    constexpr float inv255 = 1.0f / 255.0f;
    uint4 e[PB][4];
    float tb[PB], tg[PB], tr[PB];
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      int bf, rr, rg, rb;
      locate_g(c[t][0], c[t][1], c[t][2], bf, rr, rg, rb);
      tb[t] = (float)rb;
      tg[t] = (float)rg * inv255;
      tr[t] = (float)rr * inv255;
      MACT_DCHECK(bf >= 0 && bf + NG * NG + NG < NNG);
      const uint32_t a = smem_u32(s->u.pk2) + ((uint32_t)bf << 4);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t ak = a + (k >> 1) * SR + (k & 1) * SG;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(e[t][k].x), "=r"(e[t][k].y), "=r"(e[t][k].z), "=r"(e[t][k].w) : "r"(ak));
      }
    }
    const float2 s01 = make_float2(q.s[0], q.s[1]), k01 = make_float2(q.k[0], q.k[1]);
    const float2 m1 = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      const float2 st01 = __fmul2_rn(make_float2(q.s255[0], q.s255[1]), make_float2(tb[t], tb[t]));
      const float st2 = q.s255[2] * tb[t];
      float2 p01[4];
      float p2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 fa01, fb01;
        float fa2, fb2;
        lut_quant_f(make_uint2(e[t][k].x, e[t][k].y), fa01, fa2);
        lut_quant_f(make_uint2(e[t][k].z, e[t][k].w), fb01, fb2);
        const float2 va01 = __ffma2_rn(fa01, s01, k01);
        const float va2 = fmaf(fa2, q.s[2], q.k[2]);
        p01[k] = __ffma2_rn(st01, __ffma2_rn(fa01, m1, fb01), va01);
        p2[k] = fmaf(st2, fb2 - fa2, va2);
      }
      const float2 g2 = make_float2(tg[t], tg[t]);
      const float2 q0 = __ffma2_rn(g2, __ffma2_rn(p01[0], m1, p01[1]), p01[0]);
      const float2 q1 = __ffma2_rn(g2, __ffma2_rn(p01[2], m1, p01[3]), p01[2]);
      const float q02 = fmaf(tg[t], p2[1] - p2[0], p2[0]);
      const float q12 = fmaf(tg[t], p2[3] - p2[2], p2[2]);
      const float2 r01 = __ffma2_rn(make_float2(tr[t], tr[t]), __ffma2_rn(q0, m1, q1), q0);
      o[t][0] = r01.x;
      o[t][1] = r01.y;
      o[t][2] = fmaf(tr[t], q12 - q02, q02);
    }
  }
  static __device__ __forceinline__ void px4w(uint32_t w0, uint32_t w1, uint32_t w2,
                                              const Shared* s, uint32_t lane, const Params& p,
                                              float (*o)[1][3]) {
    px4w_ctx(w0, w1, w2, s, lane, p, quant(s), o);
  }
  template <bool PK>
  static __device__ __forceinline__ void px4w_t(uint32_t w0, uint32_t w1, uint32_t w2,
                                                const Shared* s, uint32_t lane, const Params& p,
                                                const LutQuant& qt, float (*o)[1][3]) {
    constexpr int K = LutK<METHOD>::K;
    constexpr int PB = K > 6 ? 2 : 4;                 // pixels per batch
    const uint32_t ch[12] = {byte_of(w0, 0), byte_of(w0, 1), byte_of(w0, 2), byte_of(w0, 3),
                             byte_of(w1, 0), byte_of(w1, 1), byte_of(w1, 2), byte_of(w1, 3),
                             byte_of(w2, 0), byte_of(w2, 1), byte_of(w2, 2), byte_of(w2, 3)};
#pragma unroll
    for (int q0 = 0; q0 < 4; q0 += PB) {
      int idx[PB][K];
      float w[PB][K];
      Node2 v[PB][K];
#pragma unroll
      for (int q = 0; q < PB; ++q) select<PK>(ch[3 * (q0 + q)], ch[3 * (q0 + q) + 1], ch[3 * (q0 + q) + 2], idx[q], w[q]);
#pragma unroll
      for (int q = 0; q < PB; ++q)
#pragma unroll
        for (int j = 0; j < K; ++j) v[q][j] = node<PK>(s, p, idx[q][j], lane, qt);
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        float2 a01 = __fmul2_rn(make_float2(w[q][0], w[q][0]), v[q][0].xy);
        float a2 = w[q][0] * v[q][0].z;
#pragma unroll
        for (int j = 1; j < K; ++j) {
          a01 = __ffma2_rn(make_float2(w[q][j], w[q][j]), v[q][j].xy, a01);
          a2 = fmaf(w[q][j], v[q][j].z, a2);
        }
        o[q0 + q][0][0] = a01.x; o[q0 + q][0][1] = a01.y; o[q0 + q][0][2] = a2;
      }
    }
  }
};

// ------------------------------------------------- 33^3: r-split CTA pairs
// The 33^3 lattice as 64-bit fixed-point nodes (LutQuant) is 287 KB -- more
// than one CTA's 227 KB -- but HALF of it by r-planes is not: a 2-CTA cluster
// holds planes 0..16 in rank 0 and planes 16..32 in rank 1 (17 x 33^2 x 8 B =
// 148 KB each, plane 16 in both).  A cell with base_r <= 15 (r <= 127) has
// all its nodes in rank 0's planes, one with base_r >= 16 (r >= 128) all in
// rank 1's, so the pixel's bit 7 of r names the CTA that can interpolate it
// from its OWN shared memory.  (Gathering the other half's nodes through
// distributed shared memory instead -- ld.shared::cluster per node -- measured
// 22-43 Gpix/s: DSMEM serves scattered 8-byte requests slowly; it is used
// here only for one contiguous bulk copy per warp and slice.)
//
// Warp w of rank 0 and warp w of rank 1 work on the same 128-pixel slices
// (lane L holds pixels 4L..4L+3, 12 bytes; rank 0 owns the output of pixels
// 0..63 = lanes 0..15, rank 1 of 64..127).  Per slice, each warp:
//   1. loads the slice (3 words per lane, prefetched one slice ahead) and
//      compacts ITS pixels (r >> 7 == rank) into a list, in pixel order, with
//      ballots and prefix popcounts;
//   2. interpolates the list, 32 entries per round (the 17^3 code: integer
//      cell location and selection, LDS.64 fixed-point nodes, FFMA2), writing
//      each result to `res` in list order -- entries of half 1 shifted by
//      pad = -T0 mod 4, so the partner's part of the list is a 16-byte
//      aligned run (rank 0 ships entries T0.., rank 1 entries 0..T0-1);
//   3. ships that run with ONE bulk copy into the partner warp's `recv`
//      (cp.async.bulk shared::cta -> shared::cluster, completing on the
//      partner's mbarrier);
//   4. merges its half on the 16 lanes that hold it (a pixel's rank among
//      ours / theirs comes from the same ballots) and stores it with STG.128;
//   5. tells the partner its `recv` is free (remote mbarrier arrive).
// Both sides know every count from the same input bytes, so the receiver
// arms its barrier with exactly the bytes the sender will ship.  Selection
// runs once per pixel; each CTA does half the interpolation work plus
// ~1/4 of the output bytes over DSMEM (bulk).  2.9 KB of buffers per warp
// leave room for 24 warps next to the 148 KB of planes.
constexpr int kL33Planes = 17;
constexpr int kL33Plane = 33 * 33;
#ifndef MACT_LUT33_NW
#define MACT_LUT33_NW 24
#endif
constexpr int kP33NW = MACT_LUT33_NW;          // warps per CTA (smem: 148 KB planes + 2.9 KB per warp)
constexpr int kP33Slice = 128;                 // pixels per warp slice
constexpr int kP33Half = 64;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// local shared -> a cluster peer's shared, completing bytes on the peer's mbarrier
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                               uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}
// Relaxed: the arrive only says "your bulk copy may overwrite my recv now"; every
// read of recv has already returned (its values fed the STGs issued before), so
// no fence is needed -- and .release.cluster compiles to MEMBAR.ALL.GPU, which
// waits for those just-issued global stores (15 % of the kernel's stall samples).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Selection of one pixel on the 33^3 lattice, as the pair kernel runs it.
template <int METHOD>
struct Lut33Sel {
  template <bool = true>
  static __device__ __forceinline__ void select(uint32_t r, uint32_t g, uint32_t b,
                                                int (&idx)[LutK<METHOD>::K], float (&w)[LutK<METHOD>::K]) {
    int br, bg, bb, rr, rg, rb;
    lut_locate<33>(r, br, rr);
    lut_locate<33>(g, bg, rg);
    lut_locate<33>(b, bb, rb);
    lut_nodes_at<33, METHOD, float, false>((br * 33 + bg) * 33 + bb, rr, rg, rb, idx, w);
  }
};

struct alignas(16) P33Warp {
  uint32_t list[kP33Slice];         // packed r | g << 8 | b << 16 of this CTA's pixels, slice order
  float recv[kP33Half * 3];         // the partner's results for my half, its list order
  float res[(kP33Slice + 5) * 3];   // my results, list order, half-1 entries shifted by pad (+ bulk slack)
};
struct P33Shared {
  P33Warp wb[kP33NW];
  uint2 pk[kL33Planes * kL33Plane];
  uint64_t rfull[kP33NW];       // my recv landed (partner's bulk copy + my expect_tx arrive)
  uint64_t sfree[kP33NW];       // the partner consumed what I sent (its remote arrive)
  LutQuant q;
  float red[32][6];
};
constexpr size_t kP33Smem = sizeof(P33Shared);

// node value: fixed-point from my planes (PK) or fp32 from the L2 lattice
template <bool PK>
__device__ __forceinline__ Node2 p33_node(uint32_t pk_base, const float4* lat4, const LutQuant& q, int i) {
  if constexpr (PK) {
    uint2 w;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "r"(pk_base + ((uint32_t)i << 3)));
    return lut_quant_unpack2(q, w);
  } else {
    const float4 t = __ldg(lat4 + i);
    return Node2{make_float2(t.x, t.y), t.z};
  }
}

// Interpolate list entries lane + 32 q (q < Q) into res (entry j at j + pad if j >= T0).
template <int METHOD, bool PK>
__device__ __forceinline__ void p33_rounds(P33Warp& B, int M, int T0, int pad, uint32_t rank, uint32_t lane,
                                           uint32_t pk_base, const float4* lat4, const LutQuant& q) {
  constexpr int K = LutK<METHOD>::K;
#ifndef MACT_P33_PB
#define MACT_P33_PB 1
#endif
  // entries per lane in flight: M ~ 64 entries per 128-px slice, so rounds of
  // 32 x PB waste lanes on the last round (PB = 2: 50-75 % use when M > 64)
  constexpr int PB = K > 6 ? 1 : MACT_P33_PB;
  const int Q = (M + 31) >> 5;
  for (int q0 = 0; q0 < Q; q0 += PB) {
    int idx[PB][K];
    float w[PB][K];
    Node2 v[PB][K];
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      const int j = (int)lane + 32 * (q0 + t);
      // padding lanes take a colour of MY half (r = 128 rank): a node outside my
      // planes would address shared memory outside the CTA's window
      const uint32_t e = j < M ? B.list[j] : (rank << 7);
      Lut33Sel<METHOD>::template select<true>(e & 0xFFu, (e >> 8) & 0xFFu, e >> 16, idx[t], w[t]);
    }
#pragma unroll
    for (int t = 0; t < PB; ++t)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        MACT_DCHECK(!PK || (uint32_t)(idx[t][k] - 16 * kL33Plane * (int)rank) < (uint32_t)(kL33Planes * kL33Plane));
        v[t][k] = p33_node<PK>(pk_base, lat4, q, idx[t][k]);
      }
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      float2 a01 = __fmul2_rn(make_float2(w[t][0], w[t][0]), v[t][0].xy);
      float a2 = w[t][0] * v[t][0].z;
#pragma unroll
      for (int k = 1; k < K; ++k) {   // out += w_k V[node_k], node order (lut.py:233-236)
        a01 = __ffma2_rn(make_float2(w[t][k], w[t][k]), v[t][k].xy, a01);
        a2 = fmaf(w[t][k], v[t][k].z, a2);
      }
      const int j = (int)lane + 32 * (q0 + t);
      if (j < M) {
        const int jj = j + (j >= T0 ? pad : 0);
        MACT_DCHECK(jj < kP33Slice + 3);
        float* dst = B.res + 3 * jj;
        dst[0] = a01.x; dst[1] = a01.y; dst[2] = a2;
      }
    }
  }
}

template <int METHOD>
__global__ void __launch_bounds__(kP33NW * 32, 1)
    k_lut33_pair(const float4* __restrict__ lat4, const uint8_t* __restrict__ rgb, float* __restrict__ out,
                 int64_t n, int64_t nslices, int planar) {
  extern __shared__ __align__(128) uint8_t smem_p33[];
  P33Shared* S = reinterpret_cast<P33Shared*>(smem_p33);
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kP33NW; ++i) {
      mbar_init(&S->rfull[i], 1);
      mbar_init(&S->sfree[i], 1);
    }
    fence_mbar_init();
  }
  // first slice's input words in flight while the CTA stages its planes
  const uint32_t* in_w = reinterpret_cast<const uint32_t*>(rgb);
  const int64_t nbytes = 3 * n;
  auto load = [&](int64_t sl, uint32_t (&wd)[3]) {
    const int64_t w0 = sl * (kP33Slice * 3 / 4) + 3 * lane;   // word index
    if ((sl + 1) * kP33Slice <= n) {                            // a whole slice: no per-word checks
#pragma unroll
      for (int c = 0; c < 3; ++c) wd[c] = __ldg(in_w + w0 + c);
      return;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {                               // the ragged end of the buffer
      uint32_t v = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (4 * (w0 + c) + k < nbytes) v |= (uint32_t)rgb[4 * (w0 + c) + k] << (8 * k);
      wd[c] = v;
    }
  };
  int64_t sl = cl * kP33NW + warp;
  uint32_t nxt[3] = {};
  if (sl < nslices) load(sl, nxt);
  lut_quant_setup(lat4, 33 * 33 * 33, &S->q, S->red);   // ends with __syncthreads
  const LutQuant q = S->q;
  if (q.on) {
    const int first = 16 * kL33Plane * (int)rank;
    for (int i = threadIdx.x; i < kL33Planes * kL33Plane; i += blockDim.x)
      S->pk[i] = lut_quant_pack(q, __ldg(lat4 + first + i));
  }
  cluster_sync_all();   // both CTAs: barriers initialised, planes staged

  P33Warp& B = S->wb[warp];
  const uint32_t recv_peer = mapa_shared(smem_u32(B.recv), peer);
  const uint32_t rfull_peer = mapa_shared(smem_u32(&S->rfull[warp]), peer);
  const uint32_t sfree_peer = mapa_shared(smem_u32(&S->sfree[warp]), peer);
  // node index (whole lattice) -> shared address in my planes
  const uint32_t pk_base = smem_u32(S->pk) - rank * (16u * kL33Plane * 8u);
  const uint32_t lt = lanemask_lt();
  const bool merger = (lane >> 4) == rank;              // this lane's 4 pixels are in my half
  uint32_t ns = 0, nr = 0;                               // sends / receives so far (exchange phases)
  for (; sl < nslices; sl += ncl * kP33NW) {
    const uint32_t wd[3] = {nxt[0], nxt[1], nxt[2]};
    if (sl + ncl * kP33NW < nslices) load(sl + ncl * kP33NW, nxt);
    const int64_t px0 = sl * kP33Slice;
    const int64_t left = n - px0;
    const int valid = left >= kP33Slice ? kP33Slice : (int)left;
    // ---- 1. my pixels of the slice, compacted in pixel order
    uint32_t bal[4];
    int M = 0, T0 = 0, pre = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t r = byte_of(wd[(3 * k) >> 2], (3 * k) & 3);
      const bool mine = (r >> 7) == rank && (int)(4 * lane) + k < valid;
      bal[k] = __ballot_sync(0xffffffffu, mine);
      M += __popc(bal[k]);
      T0 += __popc(bal[k] & 0xFFFFu);
      pre += __popc(bal[k] & lt);
    }
    {
      int j = pre;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if ((bal[k] >> lane) & 1u) {
          const int b0 = 3 * k;   // byte offset of the pixel in the lane's 12 bytes
          const uint32_t r = byte_of(wd[b0 >> 2], b0 & 3), g = byte_of(wd[(b0 + 1) >> 2], (b0 + 1) & 3),
                         b = byte_of(wd[(b0 + 2) >> 2], (b0 + 2) & 3);
          B.list[j++] = r | g << 8 | b << 16;
        }
      }
    }
    const int T1 = M - T0, pad = (-T0) & 3;
    const int v0 = valid < kP33Half ? valid : kP33Half, v1 = valid - v0;
    const int vm = rank ? v1 : v0, Tm = rank ? T1 : T0, Tp = rank ? T0 : T1;
    const uint32_t in_bytes = (uint32_t)(12 * (vm - Tm) + 15) & ~15u;
    const uint32_t out_bytes = (uint32_t)(12 * Tp + 15) & ~15u;
    MACT_DCHECK(M <= kP33Slice && Tm <= vm && in_bytes <= sizeof(B.recv) &&
                12 * (rank ? 0 : T0 + pad) + out_bytes <= sizeof(B.res));
    // The exchange counts transfers, not slices: a slice where one rank owns
    // every pixel has a send in one direction only, and with per-slice phases
    // the rank that receives nothing could complete two phases of its
    // partner's `sfree` before the partner waits on the first (the parity wait
    // then blocks forever -- found on the R-major 2^24 cube, where whole slices
    // belong to one rank).  rfull phase k = my k-th receive; sfree phase k =
    // the partner's consumption of my k-th send.
    if (lane == 0 && in_bytes) mbar_arrive_expect_tx(&S->rfull[warp], in_bytes);
    if (ns > 0) mbar_wait(&S->sfree[warp], (ns - 1) & 1);   // my last send was consumed: res and its recv free
    __syncwarp();
    // ---- 2. interpolate my pixels
    if (q.on) p33_rounds<METHOD, true>(B, M, T0, pad, rank, lane, pk_base, lat4, q);
    else p33_rounds<METHOD, false>(B, M, T0, pad, rank, lane, pk_base, lat4, q);
    // ---- 3. the partner's part of the list to the partner
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && out_bytes)
      bulk_s2cluster(recv_peer, smem_u32(B.res + (rank ? 0 : 3 * (T0 + pad))), out_bytes, rfull_peer);
    ns += out_bytes != 0;
    // ---- 4. merge my half: ours from res, theirs from recv
    if (in_bytes) mbar_wait(&S->rfull[warp], nr & 1);
    if (merger) {
      float o[12];
      // pixel 4 lane + k of the slice: its position in my half minus the own pixels
      // before it there (list index j minus the T0 half-0 entries for rank 1)
      int j = pre;                                       // list index of this lane's next own pixel
      const int base = 4 * (int)lane - kP33Half * (int)rank + (rank ? T0 : 0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool m = (bal[k] >> lane) & 1u;
        const int theirs = base + k - j;
        const float* src = m ? B.res + 3 * (j + (rank ? pad : 0)) : B.recv + 3 * theirs;
        o[3 * k] = src[0]; o[3 * k + 1] = src[1]; o[3 * k + 2] = src[2];
        j += m;
      }
      const int64_t p = px0 + 4 * lane;
      const int lv = valid - 4 * (int)lane;              // valid pixels of this lane
      if (!planar) {
        if (lv >= 4) {
          float4* d = reinterpret_cast<float4*>(out + 3 * p);
          d[0] = make_float4(o[0], o[1], o[2], o[3]);
          d[1] = make_float4(o[4], o[5], o[6], o[7]);
          d[2] = make_float4(o[8], o[9], o[10], o[11]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < lv)
#pragma unroll
              for (int c = 0; c < 3; ++c) out[3 * (p + k) + c] = o[3 * k + c];
        }
      } else {
        if (lv >= 4 && (n & 3) == 0) {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            *reinterpret_cast<float4*>(out + c * n + p) = make_float4(o[c], o[3 + c], o[6 + c], o[9 + c]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < lv)
#pragma unroll
              for (int c = 0; c < 3; ++c) out[c * n + p + k] = o[3 * k + c];
        }
      }
    }
    // ---- 5. my recv is free for the partner's next send
    __syncwarp();
    if (in_bytes) {
      if (lane == 0) mbar_arrive_remote(sfree_peer);
      ++nr;
    }
  }
  cluster_sync_all();   // the partner may still copy into / arrive on my shared memory
}

// ------------------------------------------ 33^3: r-split INDEPENDENT CTAs
// The same r-split of the fixed-point lattice (CTA b holds planes 0..16 if
// b is even, 16..32 if odd: 148 KB), but with no exchange at all: CTA 2c and
// CTA 2c+1 both scan the same slices, each keeps only ITS pixels (r bit 7 ==
// b & 1), interpolates them from its own shared memory and writes the 12-byte
// results straight to global memory at the pixel's position.  The two CTAs
// never talk -- no cluster, no DSMEM copy, no merge, no mbarrier -- and run at
// the same pace over the same addresses, so L2 serves the second reader of a
// slice and merges the two CTAs' partial sector writes before they reach DRAM.
//
// Per warp: a ring `list` of pending own pixels (r | g << 8 | b << 16 |
// pos << 24 | slice parity << 31).  A 128-px slice appends ~64 entries in pixel
// order (ballots + prefix popcounts, branch-free: one PRMT builds an entry, a
// predicated STS appends it); the warp then interpolates FULL rounds
// of 32 entries (the 17^3 code: integer selection, LDS.64 fixed-point nodes,
// FFMA2) and carries the remainder (< 32) into the next slice, so no lane idles
// on a ragged last round; an entry never survives more than one slice boundary
// (a remainder older than that is flushed as a partial round), which is why
// one parity bit names its slice.  Results go out as three STG.32 per entry
// (routing the words through a transpose buffer so that each store covers a
// contiguous third of the round measured slower: 109 vs 128 Gpix/s).
#ifndef MACT_LUT33S_NW
#define MACT_LUT33S_NW 32
#endif
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
constexpr int kS33NW = MACT_LUT33S_NW;
constexpr int kS33Ring = 256;                  // >= 31 carried + 128 appended
struct S33Shared {
  uint32_t list[kS33NW][kS33Ring];             // first: each warp's ring is 1 KB aligned (address = base | offset)
  uint2 pk[kL33Planes * kL33Plane];
  LutQuant q;
  float red[32][6];
};
constexpr size_t kS33Smem = sizeof(S33Shared);

// One round: entries head .. head + m - 1 of the ring (lane l takes entry l).
// q0 / q1: output pointer of the first pixel of the latest slice of parity 0 / 1.
template <int METHOD, bool PK, bool PLANAR>
__device__ __forceinline__ void s33_round(uint32_t list_base, uint32_t head_b, int m, uint32_t rank, uint32_t lane,
                                          uint32_t pk_base, const float4* lat4, const LutQuant& q, float* q0,
                                          float* q1, int64_t n) {
  constexpr int K = LutK<METHOD>::K;
  const bool act = (int)lane < m;
  // padding lanes take a colour of MY half: a node outside my planes would
  // address shared memory outside the CTA's window
  uint32_t e = rank << 7;
  if (act) e = lds_u32(list_base | ((head_b + 4u * lane) & (4u * kS33Ring - 4u)));
  int idx[K];
  float w[K];
  Node2 v[K];
  Lut33Sel<METHOD>::template select<true>(byte_of(e, 0), byte_of(e, 1), byte_of(e, 2), idx, w);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    MACT_DCHECK(!PK || (uint32_t)(idx[k] - 16 * kL33Plane * (int)rank) < (uint32_t)(kL33Planes * kL33Plane));
    v[k] = p33_node<PK>(pk_base, lat4, q, idx[k]);
  }
  float2 a01 = __fmul2_rn(make_float2(w[0], w[0]), v[0].xy);
  float a2 = w[0] * v[0].z;
#pragma unroll
  for (int k = 1; k < K; ++k) {   // out += w_k V[node_k], node order (lut.py:233-236)
    a01 = __ffma2_rn(make_float2(w[k], w[k]), v[k].xy, a01);
    a2 = fmaf(w[k], v[k].z, a2);
  }
  float* d = (int32_t)e < 0 ? q1 : q0;
  const uint32_t pos = (e >> 24) & 127u;
  if (act) {
    if constexpr (PLANAR) {
      d += pos;
      d[0] = a01.x; d[n] = a01.y; d[2 * n] = a2;
    } else {
      d += 3u * pos;
      d[0] = a01.x; d[1] = a01.y; d[2] = a2;
    }
  }
}

template <int METHOD, bool PLANAR>
__global__ void __launch_bounds__(kS33NW * 32, 1)
    k_lut33_split(const float4* __restrict__ lat4, const uint8_t* __restrict__ rgb, float* __restrict__ out,
                  int64_t n, int64_t nslices) {
  extern __shared__ __align__(1024) uint8_t smem_s33[];
  S33Shared* S = reinterpret_cast<S33Shared*>(smem_s33);
  const uint32_t rank = blockIdx.x & 1u;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t list_base = smem_u32(S->list[warp]);
  if (list_base & (4u * kS33Ring - 1u)) __trap();             // ring addressing ORs the offset into the base
  // This warp's slices: sl0, sl0 + stride, ...  The loop runs on 32-bit counters
  // and running pointers (no 64-bit index arithmetic per slice): iterations
  // below `full` are whole slices, the one after (if any) is the ragged end.
  const int64_t stride = ncl * kS33NW, sl0 = cl * kS33NW + warp;
  const int iters = sl0 < nslices ? (int)((nslices - 1 - sl0) / stride) + 1 : 0;
  const int64_t nfull = n / kP33Slice;
  const int full = sl0 < nfull ? (int)((nfull - 1 - sl0) / stride) + 1 : 0;
  const uint32_t* pin = reinterpret_cast<const uint32_t*>(rgb) + sl0 * (kP33Slice * 3 / 4) + 3 * lane;
  const int64_t pin_step = stride * (kP33Slice * 3 / 4);
  // bytes past the end of the buffer read as a colour of the OTHER half, so the
  // ragged last slice needs no bounds test in the scan
  const uint32_t fill = rank ? 0u : 0x80u;
  auto load = [&](int it, const uint32_t* p, uint32_t (&wd)[3]) {
    if (it < full) {                                            // a whole slice: no per-byte checks
#pragma unroll
      for (int c = 0; c < 3; ++c) wd[c] = __ldg(p + c);
      return;
    }
    const int64_t b0 = reinterpret_cast<const uint8_t*>(p) - rgb, nbytes = 3 * n;
#pragma unroll
    for (int c = 0; c < 3; ++c) {                               // the ragged end of the buffer
      uint32_t v = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        v |= (b0 + 4 * c + k < nbytes ? (uint32_t)rgb[b0 + 4 * c + k] : fill) << (8 * k);
      wd[c] = v;
    }
  };
  uint32_t nxt[3] = {};
  if (iters > 0) load(0, pin, nxt);    // first slice in flight while the CTA stages its planes
  lut_quant_setup(lat4, 33 * 33 * 33, &S->q, S->red);   // ends with __syncthreads
  const LutQuant q = S->q;
  if (q.on) {
    const int first = 16 * kL33Plane * (int)rank;
    for (int i = threadIdx.x; i < kL33Planes * kL33Plane; i += blockDim.x)
      S->pk[i] = lut_quant_pack(q, __ldg(lat4 + first + i));
  }
  __syncthreads();
  const uint32_t pk_base = smem_u32(S->pk) - rank * (16u * kL33Plane * 8u);
  const uint32_t lt = lanemask_lt();
  const uint32_t flip = rank ? 0u : 0x80808080u;   // after the flip, bit 7 of r set <=> the pixel is mine
  // PK: fixed-point nodes from my planes, else fp32 nodes from the L2 lattice (decided once)
  auto body = [&](auto pk_tag) {
    constexpr bool PK = decltype(pk_tag)::value;
    uint32_t head_b = 0;                 // ring byte offset of the oldest pending entry
    uint32_t tag0 = (4u * lane) << 24;   // pos << 24 | slice parity << 31 of the lane's first pixel
    int cnt = 0;
    float* qs = out + (PLANAR ? 1 : 3) * (sl0 * kP33Slice);   // output of the slice's first pixel
    const int64_t qs_step = (PLANAR ? 1 : 3) * (stride * kP33Slice);
    float *q0 = out, *q1 = out;
    auto round = [&](int m) {
      s33_round<METHOD, PK, PLANAR>(list_base, head_b, m, rank, lane, pk_base, lat4, q, q0, q1, n);
      head_b += 4u * (uint32_t)m;
      cnt -= m;
    };
    for (int it = 0; it < iters; ++it, qs += qs_step) {
      const uint32_t w0 = nxt[0], w1 = nxt[1], w2 = nxt[2];
      pin += pin_step;
      if (it + 1 < iters) load(it + 1, pin, nxt);
      if ((int32_t)tag0 < 0) q1 = qs; else q0 = qs;
      const int old = cnt;
      // ---- my pixels of the slice: pixel column k = pixels 4 lane + k.  The r bytes
      // of the four pixels sit at byte 0 / 3 of w0, byte 2 of w1, byte 1 of w2.
      const uint32_t f0 = w0 ^ flip, f1 = w1 ^ flip, f2 = w2 ^ flip;
      const uint32_t e0 = __byte_perm(w0, tag0, 0x7210);
      const uint32_t e1 = (__byte_perm(w0, w1, 0x0543) & 0xFFFFFFu) | (tag0 + (1u << 24));
      const uint32_t e2 = (__byte_perm(w1, w2, 0x0432) & 0xFFFFFFu) | (tag0 + (2u << 24));
      const uint32_t e3 = __byte_perm(w2, tag0 + (3u << 24), 0x7321);
      // list order = pixel order (lane-major): a round's 32 entries then cover ~64
      // consecutive pixels, so its stores touch ~24 sectors; appending column by
      // column (a round's entries 48 B apart, one sector each) measured 116 vs 144 Gpix/s.
      // Written in PTX so that each own flag is ONE predicate feeding its ballot,
      // its predicated store and the slot increment (the C++ form compiled to two
      // or three evaluations of every flag).
      static_assert(kS33Ring == 256, "ring mask in the PTX below");
      uint32_t a_end;
      asm volatile(
          "{\n"
          ".reg .pred p0, p1, p2, p3;\n"
          ".reg .b32 t, b0, b1, b2, b3, a, ad;\n"
          "and.b32 t, %1, 0x80;\n"
          "setp.ne.u32 p0, t, 0;\n"
          "setp.lt.s32 p1, %1, 0;\n"
          "and.b32 t, %2, 0x800000;\n"
          "setp.ne.u32 p2, t, 0;\n"
          "and.b32 t, %3, 0x8000;\n"
          "setp.ne.u32 p3, t, 0;\n"
          "vote.sync.ballot.b32 b0, p0, 0xffffffff;\n"
          "vote.sync.ballot.b32 b1, p1, 0xffffffff;\n"
          "vote.sync.ballot.b32 b2, p2, 0xffffffff;\n"
          "vote.sync.ballot.b32 b3, p3, 0xffffffff;\n"
          "and.b32 b0, b0, %9;\n"
          "and.b32 b1, b1, %9;\n"
          "and.b32 b2, b2, %9;\n"
          "and.b32 b3, b3, %9;\n"
          "popc.b32 b0, b0;\n"
          "popc.b32 b1, b1;\n"
          "popc.b32 b2, b2;\n"
          "popc.b32 b3, b3;\n"
          "add.u32 b0, b0, b1;\n"
          "add.u32 b2, b2, b3;\n"
          "add.u32 b0, b0, b2;\n"
          "shl.b32 b0, b0, 2;\n"
          "add.u32 a, %8, b0;\n"
          "lop3.b32 ad, a, 0x3FC, %10, 0xEA;\n"
          "@p0 st.shared.u32 [ad], %4;\n"
          "@p0 add.u32 a, a, 4;\n"
          "lop3.b32 ad, a, 0x3FC, %10, 0xEA;\n"
          "@p1 st.shared.u32 [ad], %5;\n"
          "@p1 add.u32 a, a, 4;\n"
          "lop3.b32 ad, a, 0x3FC, %10, 0xEA;\n"
          "@p2 st.shared.u32 [ad], %6;\n"
          "@p2 add.u32 a, a, 4;\n"
          "lop3.b32 ad, a, 0x3FC, %10, 0xEA;\n"
          "@p3 st.shared.u32 [ad], %7;\n"
          "@p3 add.u32 a, a, 4;\n"
          "mov.u32 %0, a;\n"
          "}\n"
          : "=r"(a_end)
          : "r"(f0), "r"(f1), "r"(f2), "r"(e0), "r"(e1), "r"(e2), "r"(e3), "r"(head_b + 4u * (uint32_t)cnt),
            "r"(lt), "r"(list_base)
          : "memory");
      // lane 31's end of list is the new tail: one shuffle instead of four popcounts
      cnt = (int)((__shfl_sync(0xffffffffu, a_end, 31) - head_b) >> 2);
      MACT_DCHECK(cnt <= kS33Ring);
      __syncwarp();
      // ---- full rounds; a remainder from before this slice goes out now
      if (cnt >= 32) {
        do round(32); while (cnt >= 32);
      } else if (old > 0) {
        round(cnt);
      }
      tag0 ^= 0x80000000u;
    }
    if (cnt > 0) round(cnt);
  };
  if (q.on) body(std::true_type{});
  else body(std::false_type{});
}

// Per-pixel 33^3 path for unaligned buffers: the same selection and the same
// node arithmetic as the pair kernel (fixed-point nodes quantised on the fly
// from the L2 lattice with the same LutQuant), so every path is bit-identical.
template <int METHOD>
struct OpLut33Gen {
  static constexpr int NOUT = 1;
  using Params = LutParams;
  struct Shared {
    LutQuant q;
    float red[32][6];
  };
  static __device__ __forceinline__ void init(Shared* s, const Params& p) {
    lut_quant_setup(p.lat, 33 * 33 * 33, &s->q, s->red);
  }
  static __device__ __forceinline__ void px(uint32_t r, uint32_t g, uint32_t b, const Shared* s,
                                            uint32_t, const Params& p, float (*o)[3]) {
    constexpr int K = LutK<METHOD>::K;
    int idx[K];
    float w[K];
    Lut33Sel<METHOD>::template select<true>(r, g, b, idx, w);
    const LutQuant q = s->q;
    auto nd = [&](int i) {
      const float4 t = __ldg(p.lat + i);
      return q.on ? lut_quant_unpack2(q, lut_quant_pack(q, t)) : Node2{make_float2(t.x, t.y), t.z};
    };
    Node2 v = nd(idx[0]);
    float2 a01 = __fmul2_rn(make_float2(w[0], w[0]), v.xy);
    float a2 = w[0] * v.z;
#pragma unroll
    for (int k = 1; k < K; ++k) {
      v = nd(idx[k]);
      a01 = __ffma2_rn(make_float2(w[k], w[k]), v.xy, a01);
      a2 = fmaf(w[k], v.z, a2);
    }
    o[0][0] = a01.x; o[0][1] = a01.y; o[0][2] = a2;
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
template <typename TI>
__device__ __forceinline__ double px_chan(const TI* p, int64_t i) { return (double)p[i]; }

// One kernel for every fp64 LUT evaluation: angular destinations, real-valued
// pixels and the float64 fidelity mode.  Cell location and weights follow
// lut._locate / node_weights in fp64 (lut_nodes_real, bit-identical to the
// reference); linear components accumulate out += w_j V[node_j] in node order
// (lut.py:233-236), rounded like numpy, so a linear destination with fp64
// output reproduces the reference bit for bit.
//
// CACHED: the caching variant (lut._interpolate_caching, lut.py:294-331) on
// the per-cell cache arrays of mact_lut_cache_build: linear components as
// trilinear polynomial terms (sum over the 8 terms in order, lut.py:303-306)
// or base node plus weighted corner differences (lut.py:309-319), each
// operation rounded like numpy's.
template <int N, int METHOD, typename TI, typename TO, bool CACHED = false>
__global__ void k_lut_fp64(const double* __restrict__ lat, int mask, const TI* __restrict__ rgb,
                           TO* __restrict__ out, int64_t n, int planar,
                           const double* __restrict__ tri = nullptr,
                           const double* __restrict__ cdiff = nullptr) {
  constexpr int K = LutK<METHOD>::K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int idx[K];
    double w[K], d[3];
    lut_nodes_real<N, METHOD>(px_chan(rgb, 3 * i), px_chan(rgb, 3 * i + 1), px_chan(rgb, 3 * i + 2), idx, w, d);
    double res[3];
    // cell of the base corner in the (N-1)^3 cache
    const int bf = idx[0], br = bf / (N * N), bg = (bf / N) % N, bb = bf % N;
    const int64_t cell = ((int64_t)br * (N - 1) + bg) * (N - 1) + bb;
    for (int comp = 0; comp < 3; ++comp) {
      if (!((mask >> comp) & 1) && CACHED && METHOD == MACT_LUT_TRILINEAR) {   // lut.py:301-306
        const double t[8] = {1.0, d[0], d[1], d[2], __dmul_rn(d[0], d[1]), __dmul_rn(d[0], d[2]),
                             __dmul_rn(d[1], d[2]), __dmul_rn(__dmul_rn(d[0], d[1]), d[2])};
        const double* c = tri + cell * 24 + comp;
        double a = __dmul_rn(c[0], t[0]);
        for (int k = 1; k < 8; ++k) a = __dadd_rn(a, __dmul_rn(c[3 * k], t[k]));
        res[comp] = a;
      } else if (!((mask >> comp) & 1) && CACHED) {                           // lut.py:307-319
        const double* c = cdiff + cell * 24 + comp;
        double a = lat[3 * bf + comp];
        for (int j = 0; j < K; ++j) {
          const int local = idx[j] - bf;
          const int row = (local / (N * N)) << 2 | ((local % (N * N)) / N) << 1 | (local % N);
          a = __dadd_rn(a, __dmul_rn(w[j], c[3 * row]));
        }
        res[comp] = a;
      } else if (!((mask >> comp) & 1)) {
        double a = 0.0;
        for (int j = 0; j < K; ++j) a = __dadd_rn(a, __dmul_rn(w[j], lat[3 * idx[j] + comp]));
        res[comp] = a;
      } else if (METHOD == MACT_LUT_TRILINEAR) {         // lut.py:249-262
        double v[8];
        for (int j = 0; j < 8; ++j) v[j] = lat[3 * idx[j] + comp];   // corner c = r<<2|g<<1|b
        const double r00 = angular_lerp_d(v[0], v[4], d[0]), r01 = angular_lerp_d(v[1], v[5], d[0]);
        const double r10 = angular_lerp_d(v[2], v[6], d[0]), r11 = angular_lerp_d(v[3], v[7], d[0]);
        res[comp] = angular_lerp_d(angular_lerp_d(r00, r10, d[1]), angular_lerp_d(r01, r11, d[1]), d[2]);
      } else {                                            // _circular_blend, lut.py:219-228
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
      if (planar) out[comp * n + i] = (TO)res[comp];
      else out[3 * i + comp] = (TO)res[comp];
    }
  }
}

// lut.build_cache (lut.py:265-291): per cell (r-major over (n-1)^3) the 8
// trilinear polynomial coefficients and the 8 corner differences, each (8, 3)
// fp64, evaluated left to right as the numpy expressions are.
__global__ void k_lut_cache_build(const double* __restrict__ lat, int n, double* __restrict__ tri,
                                  double* __restrict__ cdiff) {
  const int m = n - 1, total = m * m * m * 3;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int comp = i % 3, cell = i / 3;
    const int br = cell / (m * m), bg = (cell / m) % m, bb = cell % m;
    double c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)   // corner k = r<<2 | g<<1 | b (_CORNER_OFFSETS, lut.py:59-60)
      c[k] = lat[3 * (((br + (k >> 2 & 1)) * n + bg + (k >> 1 & 1)) * n + bb + (k & 1)) + comp];
    double* t = tri + (int64_t)cell * 24 + comp;
    t[0] = c[0];
    t[3] = __dadd_rn(c[4], -c[0]);
    t[6] = __dadd_rn(c[2], -c[0]);
    t[9] = __dadd_rn(c[1], -c[0]);
    t[12] = __dadd_rn(__dadd_rn(__dadd_rn(c[6], -c[4]), -c[2]), c[0]);
    t[15] = __dadd_rn(__dadd_rn(__dadd_rn(c[5], -c[4]), -c[1]), c[0]);
    t[18] = __dadd_rn(__dadd_rn(__dadd_rn(c[3], -c[2]), -c[1]), c[0]);
    double s7 = __dadd_rn(__dadd_rn(__dadd_rn(c[7], -c[6]), -c[5]), -c[3]);
    s7 = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(s7, c[4]), c[2]), c[1]), -c[0]);
    t[21] = s7;
    double* dd = cdiff + (int64_t)cell * 24 + comp;
#pragma unroll
    for (int k = 0; k < 8; ++k) dd[3 * k] = __dadd_rn(c[k], -c[0]);
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

// The interpolation kernels' own selection (Op::select: the reference's cells;
// TIES = false, so a tie's zero-weight middle node may be another corner).
template <int N, int METHOD>
__global__ void k_lut_nodes_timed(const uint8_t* __restrict__ rgb, int64_t n, int32_t* __restrict__ nodes,
                                  float* __restrict__ weights) {
  constexpr int K = LutK<METHOD>::K;
  using Sel = std::conditional_t<N == 33, Lut33Sel<METHOD>, OpLut<N, METHOD>>;
  constexpr int NG = N == 33 ? 33 : OpLut<N, METHOD>::NG;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int idx[K];
    float w[K];
    Sel::template select<true>(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], idx, w);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int ir = min(idx[j] / (NG * NG), N - 1), ig = min((idx[j] / NG) % NG, N - 1), ib = min(idx[j] % NG, N - 1);
      nodes[i * K + j] = (ir * N + ig) * N + ib;
      weights[i * K + j] = w[j];
    }
  }
}

// Real-valued pixels: fp64 nodes and weights exactly as lut.node_weights
// computes them (lut.py:115-199).
template <int N, int METHOD, typename TI>
__global__ void k_lut_nodes_real(const TI* __restrict__ rgb, int64_t n, int32_t* __restrict__ nodes,
                                 double* __restrict__ weights) {
  constexpr int K = LutK<METHOD>::K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int idx[K];
    double w[K], d[3];
    lut_nodes_real<N, METHOD>((double)rgb[3 * i], (double)rgb[3 * i + 1], (double)rgb[3 * i + 2], idx, w, d);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      nodes[i * K + j] = idx[j];
      weights[i * K + j] = w[j];
    }
  }
}

// ------------------------------------------------- 33^3: component-split clusters
// The 33^3 lattice (35937 nodes) does not fit one CTA's shared memory as
// float4 nodes (575 KB), but ONE component of it does (144 KB).  A cluster of
// three CTAs (one per SM) works on the same 4096-pixel step: CTA rank c
// stages component c of the lattice and computes component c of every pixel
// of the step, gathering nodes with LDS.32 (random-gather cost per byte equal
// to the float4 path) instead of LDG.128 through L1/L2, whose per-line tag
// processing bounded the L2-resident version at ~0.25 px/clk/SM.
// Output stays interleaved and line-complete: the step's pixels are split in
// three ranges (1368/1364/1364, multiples of 4 so every range is a 16-byte
// aligned byte span).  Every CTA sends its component of range k to CTA k as a
// planar block with 16-byte st.async distributed-shared-memory stores that
// complete transaction bytes on the owner's "full" mbarrier; each owner
// interleaves its three planes into an (N,3) staging buffer and drains it
// with one bulk store.  The planar and staging buffers are double-buffered
// and handed back through per-(owner, buffer) "empty" mbarriers in the
// writers' shared memory, so the three CTAs never meet at a cluster barrier
// inside the loop (the R01 version's per-step cluster.sync cost ~25 % of its
// time in barrier/membar stalls).  (Measured alternatives: scattered STG.32
// from the three CTAs -> 2.8x DRAM traffic; 4-byte DSMEM scatter straight
// into interleaved staging -> DSMEM-bound.)
constexpr int kLut33Threads = 1024;
constexpr int kLut33Step = 4 * kLut33Threads;          // pixels per step
__host__ __device__ constexpr int lut33_range_start(int k) { return k == 0 ? 0 : k == 1 ? 1368 : 2732; }
constexpr int kLut33Rmax = 1368;                       // largest owner range (pixels)
constexpr size_t kLut33Smem =
    (((33 * 33 * 33) + 31) / 32 * 32 + 4 * kLut33Rmax * 3) * sizeof(float) + 8 * sizeof(uint64_t);

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t addr, float4 v, uint32_t mbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
      "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <int METHOD>
__global__ void __cluster_dims__(3, 1, 1) __launch_bounds__(kLut33Threads, 1)
    k_lut33_comp(const float4* __restrict__ lat4, const uint8_t* __restrict__ rgb,
                 float* __restrict__ out, int64_t nsteps) {
  namespace cg = cooperative_groups;
  constexpr int N = 33, NN = N * N * N, K = LutK<METHOD>::K;
  constexpr int PLANE = kLut33Rmax, PBUF = 3 * kLut33Rmax, SBUF = 3 * kLut33Rmax;
  extern __shared__ __align__(128) float sm33[];
  float* lat_c = sm33;                                   // NN floats
  float* planar = sm33 + ((NN + 31) / 32) * 32;          // [2][3][RMAX]: components of MY range
  float* stage = planar + 2 * PBUF;                      // [2][RMAX*3]: interleaved, bulk-stored
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + 2 * SBUF);   // [2]: my planar buffer b landed
  uint64_t* empty = full + 2;                            // [3][2]: owner k's planar buffer b is free
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t comp = cluster.block_rank();
  const int64_t cl = blockIdx.x / 3, ncl = gridDim.x / 3;
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    for (int i = 0; i < 6; ++i) mbar_init(&empty[i], 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < NN; i += blockDim.x) {
    const float4 v = __ldg(lat4 + i);
    lat_c[i] = comp == 0 ? v.x : comp == 1 ? v.y : v.z;
  }
  // Two warp groups of 512 threads alternate steps: group g owns buffer g and
  // runs steps it = g, g+2, ..., so one group's gathers overlap the other's
  // exchange wait, interleave and store (a named barrier per group, no
  // CTA-wide barrier in the loop).  Each thread handles two 4-pixel chunks
  // of a step: pixels 4*tg and 2048 + 4*tg.
  const int grp = (int)(threadIdx.x >> 9), tg = (int)(threadIdx.x & 511);
  uint32_t owner[2], dst[2], ofull[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t4 = 4 * tg + 2048 * h;
    owner[h] = t4 < 1368 ? 0 : (t4 < 2732 ? 1 : 2);
    const int off = t4 - lut33_range_start(owner[h]);
    dst[h] = mapa_u32(smem_u32(planar + grp * PBUF + comp * PLANE + off), owner[h]);
    ofull[h] = mapa_u32(smem_u32(&full[grp]), owner[h]);
  }
  const int r0 = lut33_range_start(comp);
  const int rlen = (comp == 2 ? kLut33Step : lut33_range_start(comp + 1)) - r0;
  const uint32_t full_bytes = (uint32_t)rlen * 3u * 4u;
  cluster.sync();                                        // barriers initialised, lattices staged
  const uint32_t* in_w = reinterpret_cast<const uint32_t*>(rgb);
  // input words of the group's next step are loaded one step ahead
  uint32_t nw[2][3] = {};
  auto load_words = [&](int64_t step) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t g = step * kLut33Threads + h * 512 + tg;
      nw[h][0] = __ldg(in_w + 3 * g); nw[h][1] = __ldg(in_w + 3 * g + 1); nw[h][2] = __ldg(in_w + 3 * g + 2);
    }
  };
  if (cl + grp * ncl < nsteps) load_words(cl + grp * ncl);
  for (int64_t it = grp; cl + it * ncl < nsteps; it += 2) {
    const int64_t step = cl + it * ncl;
    const uint32_t use = (uint32_t)(it >> 1);
    uint32_t cw[2][3];
#pragma unroll
    for (int h = 0; h < 2; ++h) { cw[h][0] = nw[h][0]; cw[h][1] = nw[h][1]; cw[h][2] = nw[h][2]; }
    if (step + 2 * ncl < nsteps) load_words(step + 2 * ncl);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t ch[12] = {byte_of(cw[h][0], 0), byte_of(cw[h][0], 1), byte_of(cw[h][0], 2), byte_of(cw[h][0], 3),
                               byte_of(cw[h][1], 0), byte_of(cw[h][1], 1), byte_of(cw[h][1], 2), byte_of(cw[h][1], 3),
                               byte_of(cw[h][2], 0), byte_of(cw[h][2], 1), byte_of(cw[h][2], 2), byte_of(cw[h][2], 3)};
      // all node loads of a batch in flight together; trilinear (K = 8) goes
      // 2 pixels at a time so a 1024-thread CTA stays within 64 registers
      constexpr int PB = K > 6 ? MACT_LUT33_TRI_PB : 4;
      float a[4];
#pragma unroll
      for (int q0 = 0; q0 < 4; q0 += PB) {
        int idx[PB][K];
        float w[PB][K], v[PB][K];
#pragma unroll
        for (int q = 0; q < PB; ++q)
          lut_nodes<N, METHOD, float, false>(ch[3 * (q0 + q)], ch[3 * (q0 + q) + 1], ch[3 * (q0 + q) + 2], idx[q], w[q]);
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
          for (int j = 0; j < K; ++j) {
            MACT_DCHECK(idx[q][j] >= 0 && idx[q][j] < NN);
            v[q][j] = lat_c[idx[q][j]];
          }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          a[q0 + q] = w[q][0] * v[q][0];
#pragma unroll
          for (int j = 1; j < K; ++j) a[q0 + q] = fmaf(w[q][j], v[q][j], a[q0 + q]);
        }
      }
      // the owner's buffer must have been consumed (its use - 1) before it is
      // refilled.  Plain CTA-scope-acquire waits, as CUTLASS's cluster pipelines
      // use: an .acquire.cluster wait compiles to CCTL.IVALL (L1 invalidate),
      // which cost 21 % of the stall samples; the st.async payload is made
      // visible by the mbarrier's transaction completion itself.
      if (use >= 1) mbar_wait(&empty[owner[h] * 2 + grp], (use - 1) & 1);
      st_async_v4(dst[h], make_float4(a[0], a[1], a[2], a[3]), ofull[h]);
    }
    // owner role: wait for the three components of my range, interleave, store
    if (tg == 0) mbar_arrive_expect_tx(&full[grp], full_bytes);
    mbar_wait(&full[grp], use & 1);
    const float* pl = planar + grp * PBUF;
    float* sg = stage + grp * SBUF;
    // the bulk store issued from sg at this group's previous step must have
    // finished reading it before any thread of the group overwrites it
    if (tg == 0) bulk_wait_read<0>();
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(512) : "memory");
    for (int i = tg; 4 * i < rlen; i += 512) {           // interleave 4 pixels per thread
      const float4 c0 = *reinterpret_cast<const float4*>(pl + 4 * i);
      const float4 c1 = *reinterpret_cast<const float4*>(pl + PLANE + 4 * i);
      const float4 c2 = *reinterpret_cast<const float4*>(pl + 2 * PLANE + 4 * i);
      float4* d = reinterpret_cast<float4*>(sg + 12 * i);
      d[0] = make_float4(c0.x, c1.x, c2.x, c0.y);
      d[1] = make_float4(c1.y, c2.y, c0.z, c1.z);
      d[2] = make_float4(c2.z, c0.w, c1.w, c2.w);
    }
    fence_proxy_async_smem();
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(512) : "memory");   // stage written, planar read
    if (tg == 0) {
      bulk_s2g(out + 3 * (step * kLut33Step + r0), sg, (uint32_t)rlen * 12u);
      bulk_commit();
#pragma unroll
      for (uint32_t c = 0; c < 3; ++c) mbar_arrive_cluster(mapa_u32(smem_u32(&empty[comp * 2 + grp]), c));
    }
  }
  if (tg == 0) bulk_wait<0>();
  cluster.sync();                                        // partners may still signal / write my smem
}

// Planar output (3, N) needs no exchange at all: component c of a step is a
// contiguous 16 KB run of plane c.  STRIDED: the same CTAs write interleaved
// (N, 3) output directly, component c of pixel i at 3 i + c.  Independent CTAs (no cluster), CTA b holds
// component b % 3 and streams steps b / 3, b / 3 + G/3, ...; the two warp
// groups alternate steps and each drains its staging plane with one bulk store.
template <int METHOD, bool STRIDED = false>
__global__ void __launch_bounds__(kLut33Threads, 1)
    k_lut33_planar(const float4* __restrict__ lat4, const uint8_t* __restrict__ rgb,
                   float* __restrict__ out, int64_t n, int64_t nsteps) {
  constexpr int N = 33, NN = N * N * N, K = LutK<METHOD>::K;
  extern __shared__ __align__(128) float sm33[];
  float* lat_c = sm33;                                   // NN floats
  float* stage = sm33 + ((NN + 31) / 32) * 32;           // [2][4096]: one plane run per group
  const int comp = (int)(blockIdx.x % 3);
  const int64_t cl = blockIdx.x / 3, ncl = gridDim.x / 3;
  for (int i = threadIdx.x; i < NN; i += blockDim.x) {
    const float4 v = __ldg(lat4 + i);
    lat_c[i] = comp == 0 ? v.x : comp == 1 ? v.y : v.z;
  }
  __syncthreads();
  const int grp = (int)(threadIdx.x >> 9), tg = (int)(threadIdx.x & 511);
  const uint32_t* in_w = reinterpret_cast<const uint32_t*>(rgb);
  float* sg = stage + grp * kLut33Step;
  for (int64_t it = grp; cl + it * ncl < nsteps; it += 2) {
    const int64_t step = cl + it * ncl;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t g = step * kLut33Threads + h * 512 + tg;
      const uint32_t w0 = __ldg(in_w + 3 * g), w1 = __ldg(in_w + 3 * g + 1), w2 = __ldg(in_w + 3 * g + 2);
      const uint32_t ch[12] = {byte_of(w0, 0), byte_of(w0, 1), byte_of(w0, 2), byte_of(w0, 3),
                               byte_of(w1, 0), byte_of(w1, 1), byte_of(w1, 2), byte_of(w1, 3),
                               byte_of(w2, 0), byte_of(w2, 1), byte_of(w2, 2), byte_of(w2, 3)};
      constexpr int PB = K > 6 ? MACT_LUT33_TRI_PB : 4;
      float a[4];
#pragma unroll
      for (int q0 = 0; q0 < 4; q0 += PB) {
        int idx[PB][K];
        float w[PB][K], v[PB][K];
#pragma unroll
        for (int q = 0; q < PB; ++q)
          lut_nodes<N, METHOD, float, false>(ch[3 * (q0 + q)], ch[3 * (q0 + q) + 1], ch[3 * (q0 + q) + 2], idx[q], w[q]);
#pragma unroll
        for (int q = 0; q < PB; ++q)
#pragma unroll
          for (int j = 0; j < K; ++j) {
            MACT_DCHECK(idx[q][j] >= 0 && idx[q][j] < NN);
            v[q][j] = lat_c[idx[q][j]];
          }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          a[q0 + q] = w[q][0] * v[q][0];
#pragma unroll
          for (int j = 1; j < K; ++j) a[q0 + q] = fmaf(w[q][j], v[q][j], a[q0 + q]);
        }
      }
      if constexpr (STRIDED) {   // interleaved (N, 3) output: this CTA's component of 4 pixels
        float* d = out + 3 * (4 * g) + comp;
        d[0] = a[0]; d[3] = a[1]; d[6] = a[2]; d[9] = a[3];
        continue;
      }
      if (h == 0 && tg == 0) bulk_wait_read<0>();       // this group's previous plane run drained
      if (h == 0) asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(512) : "memory");
      *reinterpret_cast<float4*>(sg + 4 * (h * 512 + tg)) = make_float4(a[0], a[1], a[2], a[3]);
    }
    if constexpr (STRIDED) continue;
    fence_proxy_async_smem();
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(512) : "memory");
    if (tg == 0) {
      bulk_s2g(out + comp * n + step * kLut33Step, sg, kLut33Step * 4u);
      bulk_commit();
    }
  }
  if (tg == 0) bulk_wait<0>();
}

// Resident clusters of `size` CTAs for a kernel, per device (smem opt-in
// checked); bounded by MACT_GRID_CAP.
static int max_clusters(const void* fn, int size, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({fn, dev});
  if (it != cache.end()) return it->second;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    set_error(MACT_ECUDA, "cudaFuncSetAttribute(%zu B smem): %s", smem, cudaGetErrorString(e));
    return -1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(size * 48);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  int mc = 0;
  if (cudaOccupancyMaxActiveClusters(&mc, fn, &cfg) != cudaSuccess || mc < 1) {   // __cluster_dims__ kernels
    cudaGetLastError();
    cudaLaunchAttribute attr;                                                       // runtime cluster size
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = size;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&mc, fn, &cfg) != cudaSuccess || mc < 1) {
      cudaGetLastError();
      mc = num_sms() / (size + 1);
    }
  }
  if (mc * size > grid_cap()) mc = grid_cap() / size > 0 ? grid_cap() / size : 1;
  cache[{fn, dev}] = mc;
  return mc;
}

template <int METHOD>
static int launch_lut33_comp(const float* lat, const uint8_t* rgb, float* out, int64_t n, int planar,
                             cudaStream_t st) {
  NvtxRange range("lut33_interp");
  constexpr size_t smem = kLut33Smem;
  const bool aligned = (uintptr_t)rgb % 16 == 0 && (uintptr_t)out % 16 == 0;
  const bool ok = !planar && aligned;
  const int64_t nsteps = aligned && (!planar || n % 4 == 0) ? n / kLut33Step : 0;
  // Interleaved trilinear: independent component CTAs writing their component
  // of every pixel with stride-12 B stores (L2 merges the three components)
  // beat the cluster exchange (82 vs 74 Gpix/s); the simplex methods, whose
  // cluster kernel is faster, keep it (strided: 62-71 vs 86-101).
  constexpr bool kStrided = METHOD == MACT_LUT_TRILINEAR;
  if ((planar || kStrided) && nsteps > 0) {   // planar: independent component CTAs, no exchange
    // the strided variant writes global memory directly: no staging runs
    const size_t psmem = (((33 * 33 * 33) + 31) / 32 * 32 + (planar ? 2 * kLut33Step : 0)) * sizeof(float);
    auto pfn = planar ? k_lut33_planar<METHOD, false> : k_lut33_planar<METHOD, true>;
    const int64_t cap = persistent_grid((const void*)pfn, kLut33Threads, psmem);
    if (cap <= 0) return MACT_ECUDA;
    int64_t groups = cap / 3;
    if (groups > nsteps) groups = nsteps;
    if (groups < 1) groups = 1;
    pfn<<<(unsigned)(3 * groups), kLut33Threads, psmem, st>>>(reinterpret_cast<const float4*>(lat), rgb,
                                                                   out, n, nsteps);
    count_launch();
    if (int rc = check_launch("lut33_planar")) return rc;
  } else if (ok && nsteps > 0) {
    auto kfn = k_lut33_comp<METHOD>;
    const int mc = max_clusters((const void*)kfn, 3, kLut33Threads, smem);
    if (mc < 0) return MACT_ECUDA;
    const int64_t clusters = mc < nsteps ? mc : nsteps;
    kfn<<<(unsigned)(3 * clusters), kLut33Threads, smem, st>>>(reinterpret_cast<const float4*>(lat),
                                                               rgb, out, nsteps);
    count_launch();
    if (int rc = check_launch("lut33_comp")) return rc;
  }
  const int64_t done = nsteps * kLut33Step;
  if (done < n) {   // tail or unaligned buffers: the L2-gather streaming kernel
    Outs outs{{out, nullptr, nullptr}};
    LutParams p{reinterpret_cast<const float4*>(lat)};
    if (done == 0)
      return launch_stream_t<OpLut<33, METHOD>, 16, 1, 3, 1>(rgb, outs, n, planar, p, st, "lut_interp");
    auto kfn = k_generic<OpLut<33, METHOD>, 256>;
    const size_t sb = sizeof(typename OpLut<33, METHOD>::Shared);
    const int64_t cap = persistent_grid((const void*)kfn, 256, sb);
    if (cap <= 0) return MACT_ECUDA;
    int64_t grid = (n - done + 255) / 256;
    if (grid > cap) grid = cap;
    kfn<<<(unsigned)grid, 256, sb, st>>>(rgb, outs, done, n, planar, p);
    count_launch();
    return check_launch("lut_interp");
  }
  return MACT_OK;
}

// 33^3 on r-split CTA pairs (k_lut33_pair); unaligned buffers take the
// per-pixel kernel with the same arithmetic.
template <int METHOD>
static int launch_lut33_pair(const float* lat, const uint8_t* rgb, float* out, int64_t n, int planar,
                             cudaStream_t st) {
  NvtxRange range("lut33_interp");
  LutParams p{reinterpret_cast<const float4*>(lat)};
  const bool aligned = (uintptr_t)rgb % 16 == 0 && (uintptr_t)out % 16 == 0;
  if (!aligned) {
    Outs outs{{out, nullptr, nullptr}};
    auto kfn = k_generic<OpLut33Gen<METHOD>, 256>;
    const size_t sb = sizeof(typename OpLut33Gen<METHOD>::Shared);
    const int64_t cap = persistent_grid((const void*)kfn, 256, sb);
    if (cap <= 0) return MACT_ECUDA;
    int64_t grid = (n + 255) / 256;
    if (grid > cap) grid = cap;
    kfn<<<(unsigned)grid, 256, sb, st>>>(rgb, outs, 0, n, planar, p);
    count_launch();
    return check_launch("lut_interp");
  }
  const int64_t nslices = (n + kP33Slice - 1) / kP33Slice;
  auto kfn = k_lut33_pair<METHOD>;
  const int mc = max_clusters((const void*)kfn, 2, kP33NW * 32, kP33Smem);
  if (mc < 0) return MACT_ECUDA;
  int64_t clusters = mc;
  const int64_t need = (nslices + kP33NW - 1) / kP33NW;   // clusters with at least one slice per warp
  if (clusters > need) clusters = need;
  if (clusters < 1) clusters = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * clusters));
  cfg.blockDim = dim3(kP33NW * 32);
  cfg.dynamicSmemBytes = kP33Smem;
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kfn, reinterpret_cast<const float4*>(lat), rgb, out, n, nslices,
                                           planar);
  if (e != cudaSuccess) return set_error(MACT_ECUDA, "lut33_pair launch: %s", cudaGetErrorString(e));
  count_launch();
  return check_launch("lut33_pair");
}

// 33^3 on r-split independent CTAs (k_lut33_split): interleaved or planar
// output, any 4-byte aligned input; other buffers take the per-pixel kernel
// with the same arithmetic.
template <int METHOD>
static int launch_lut33_split(const float* lat, const uint8_t* rgb, float* out, int64_t n, int planar,
                              cudaStream_t st) {
  NvtxRange range("lut33_interp");
  LutParams p{reinterpret_cast<const float4*>(lat)};
  if ((uintptr_t)rgb % 4 != 0) {
    Outs outs{{out, nullptr, nullptr}};
    auto kfn = k_generic<OpLut33Gen<METHOD>, 256>;
    const size_t sb = sizeof(typename OpLut33Gen<METHOD>::Shared);
    const int64_t cap = persistent_grid((const void*)kfn, 256, sb);
    if (cap <= 0) return MACT_ECUDA;
    int64_t grid = (n + 255) / 256;
    if (grid > cap) grid = cap;
    kfn<<<(unsigned)grid, 256, sb, st>>>(rgb, outs, 0, n, planar, p);
    count_launch();
    return check_launch("lut_interp");
  }
  const int64_t nslices = (n + kP33Slice - 1) / kP33Slice;
  auto kfn = planar ? k_lut33_split<METHOD, true> : k_lut33_split<METHOD, false>;
  const int64_t cap = persistent_grid((const void*)kfn, kS33NW * 32, kS33Smem);
  if (cap <= 0) return MACT_ECUDA;
  int64_t pairs = cap / 2;
  const int64_t need = (nslices + kS33NW - 1) / kS33NW;   // pairs with at least one slice per warp
  if (pairs > need) pairs = need;
  if (pairs < 1) pairs = 1;
  kfn<<<(unsigned)(2 * pairs), kS33NW * 32, kS33Smem, st>>>(reinterpret_cast<const float4*>(lat), rgb, out, n,
                                                           nslices);
  count_launch();
  return check_launch("lut33_split");
}

// 33^3 kernel selection: the r-split independent CTAs (k_lut33_split) serve
// both layouts -- measured on C3 (trilinear / prism / pyramidal / tetrahedral):
// split 117 / 135 / 142 / 156 Gpix/s interleaved and 116 / 132 / 132 / 145
// planar, against 80 / 85 / 91 / 95 for the r-split cluster pairs
// (k_lut33_pair, DSMEM exchange) and 80 / 97 / 107 / 126 planar for the
// component CTAs (k_lut33_planar).  MACT_LUT33_KERNEL=split|pair|comp forces
// one family for A/B runs and for the parity tests of the older kernels; read
// per call (a getenv is ~100 ns next to a launch), so tests can exercise all
// of them in one process.
enum { kLut33Split = 0, kLut33Pair = 1, kLut33Comp = 2 };
static int lut33_kernel(int planar) {
  const char* e = getenv("MACT_LUT33_KERNEL");
  if (e && strcmp(e, "split") == 0) return kLut33Split;
  if (e && strcmp(e, "pair") == 0) return kLut33Pair;
  if (e && strcmp(e, "comp") == 0) return kLut33Comp;
  (void)planar;
  return kLut33Split;
}

template <int N, int METHOD>
static int launch_interp(const float* lat, const uint8_t* rgb, float* out, int64_t n, int planar,
                         cudaStream_t st) {
  Outs outs{{out, nullptr, nullptr}};
  LutParams p{reinterpret_cast<const float4*>(lat)};
  // 17^3: 64-bit fixed-point nodes (trilinear: b-pair entries) or the fp32
  // planes; 9^3: 8 bank-private float4 copies; 16 compute warps per CTA.
  // 33^3: r-split CTA pairs for interleaved output, independent component
  // CTAs for planar output (lut33_comp); unaligned buffers take the per-pixel
  // kernels with the same arithmetic.
  if constexpr (N == 33) {
    if (n <= 0) return MACT_OK;
    const int k = lut33_kernel(planar);
    return k == kLut33Comp   ? launch_lut33_comp<METHOD>(lat, rgb, out, n, planar, st)
           : k == kLut33Pair ? launch_lut33_pair<METHOD>(lat, rgb, out, n, planar, st)
                             : launch_lut33_split<METHOD>(lat, rgb, out, n, planar, st);
  } else
    return launch_stream_t<OpLut<N, METHOD>, (OpLut<N, METHOD>::PAIR ? MACT_LUT_NW_TRI17 : MACT_LUT_NW),
                           (N <= 9 ? 2 : OpLut<N, METHOD>::PAIR ? MACT_LUT_G_TRI17 : MACT_LUT_G), MACT_LUT_SIN, MACT_LUT_NOB>(
        rgb, outs, n, planar, p, st, "lut_interp");
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

// tri / cdiff != nullptr: the caching variant (mact_lut_interp_cached)
template <int N, typename TI, typename TO>
static int interp_fp64(int method, int mask, const double* lat, const TI* rgb, TO* out,
                       int64_t n, int planar, cudaStream_t st, const double* tri, const double* cdiff) {
  int64_t g = (n + 255) / 256;
  if (g > 8LL * num_sms()) g = 8LL * num_sms();
  const bool c = tri != nullptr;
#define MACT_FP64_CASE(M)                                                                                   \
  case M:                                                                                                   \
    if (c) k_lut_fp64<N, M, TI, TO, true><<<(unsigned)g, 256, 0, st>>>(lat, mask, rgb, out, n, planar, tri, cdiff); \
    else k_lut_fp64<N, M, TI, TO, false><<<(unsigned)g, 256, 0, st>>>(lat, mask, rgb, out, n, planar);      \
    break;
  switch (method) {
    MACT_FP64_CASE(MACT_LUT_TRILINEAR)
    MACT_FP64_CASE(MACT_LUT_PRISM)
    MACT_FP64_CASE(MACT_LUT_PYRAMIDAL)
    MACT_FP64_CASE(MACT_LUT_TETRAHEDRAL)
    default: return set_error(MACT_EBADARG, "unknown interpolation method %d", method);
  }
#undef MACT_FP64_CASE
  count_launch();
  return check_launch("lut_interp_fp64");
}

template <typename TI, typename TO>
static int interp_fp64_grid(int grid_n, int method, int mask, const double* lat, const TI* rgb, TO* out,
                            int64_t n, int planar, cudaStream_t st, const double* tri, const double* cdiff) {
  switch (grid_n) {
    case 9: return interp_fp64<9>(method, mask, lat, rgb, out, n, planar, st, tri, cdiff);
    case 17: return interp_fp64<17>(method, mask, lat, rgb, out, n, planar, st, tri, cdiff);
    case 33: return interp_fp64<33>(method, mask, lat, rgb, out, n, planar, st, tri, cdiff);
  }
  return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
}

template <typename TI>
static int interp_fp64_out(int out_dtype, int grid_n, int method, int mask, const double* lat, const TI* rgb,
                           void* out, int64_t n, int planar, cudaStream_t st, const double* tri = nullptr,
                           const double* cdiff = nullptr) {
  if (out_dtype == MACT_DTYPE_F64)
    return interp_fp64_grid(grid_n, method, mask, lat, rgb, (double*)out, n, planar, st, tri, cdiff);
  return interp_fp64_grid(grid_n, method, mask, lat, rgb, (float*)out, n, planar, st, tri, cdiff);
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

template <int N>
static int nodes_timed_grid(int method, const uint8_t* rgb, int64_t n, int32_t* nodes, float* w,
                            cudaStream_t st) {
  int64_t g = (n + 255) / 256;
  if (g > 8LL * num_sms()) g = 8LL * num_sms();
  switch (method) {
    case MACT_LUT_TRILINEAR: k_lut_nodes_timed<N, MACT_LUT_TRILINEAR><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_PRISM: k_lut_nodes_timed<N, MACT_LUT_PRISM><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_PYRAMIDAL: k_lut_nodes_timed<N, MACT_LUT_PYRAMIDAL><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_TETRAHEDRAL: k_lut_nodes_timed<N, MACT_LUT_TETRAHEDRAL><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    default: return set_error(MACT_EBADARG, "unknown interpolation method %d", method);
  }
  count_launch();
  return check_launch("lut_nodes_timed");
}

template <int N, typename TI>
static int nodes_real_grid(int method, const TI* rgb, int64_t n, int32_t* nodes, double* w, cudaStream_t st) {
  int64_t g = (n + 255) / 256;
  if (g > 8LL * num_sms()) g = 8LL * num_sms();
  switch (method) {
    case MACT_LUT_TRILINEAR: k_lut_nodes_real<N, MACT_LUT_TRILINEAR, TI><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_PRISM: k_lut_nodes_real<N, MACT_LUT_PRISM, TI><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_PYRAMIDAL: k_lut_nodes_real<N, MACT_LUT_PYRAMIDAL, TI><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    case MACT_LUT_TETRAHEDRAL: k_lut_nodes_real<N, MACT_LUT_TETRAHEDRAL, TI><<<(unsigned)g, 256, 0, st>>>(rgb, n, nodes, w); break;
    default: return set_error(MACT_EBADARG, "unknown interpolation method %d", method);
  }
  count_launch();
  return check_launch("lut_nodes_real");
}

template <typename TI>
static int nodes_real(int grid_n, int method, const TI* rgb, int64_t n, int32_t* nodes, double* w,
                      cudaStream_t st) {
  switch (grid_n) {
    case 9: return nodes_real_grid<9>(method, rgb, n, nodes, w, st);
    case 17: return nodes_real_grid<17>(method, rgb, n, nodes, w, st);
    case 33: return nodes_real_grid<33>(method, rgb, n, nodes, w, st);
  }
  return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
}

}  // namespace mact

using namespace mact;

extern "C" int mact_lut_nodes_real(int grid_n, int method, const void* rgb, int in_dtype, int64_t n,
                                   int32_t* nodes, double* weights, void* stream) {
  if (n < 0 || (n > 0 && (!rgb || !nodes || !weights))) return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (in_dtype == MACT_DTYPE_U8) return nodes_real(grid_n, method, (const uint8_t*)rgb, n, nodes, weights, st);
  if (in_dtype == MACT_DTYPE_F32) return nodes_real(grid_n, method, (const float*)rgb, n, nodes, weights, st);
  if (in_dtype == MACT_DTYPE_F64) return nodes_real(grid_n, method, (const double*)rgb, n, nodes, weights, st);
  return set_error(MACT_EBADARG, "unsupported input dtype %d", in_dtype);
}

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
  return mact_lut_interp_real(lattice64, grid_n, method, angular_mask, rgb, MACT_DTYPE_U8, out,
                              MACT_DTYPE_F32, n, layout, stream);
}

extern "C" int mact_lut_cache_build(const double* lattice64, int grid_n, double* trilinear,
                                    double* corner_diff, void* stream) {
  if (!lattice64 || !trilinear || !corner_diff) return set_error(MACT_EBADARG, "bad argument");
  if (grid_n != 9 && grid_n != 17 && grid_n != 33) return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
  const int total = (grid_n - 1) * (grid_n - 1) * (grid_n - 1) * 3;
  k_lut_cache_build<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(lattice64, grid_n, trilinear,
                                                                          corner_diff);
  count_launch();
  return check_launch("lut_cache_build");
}

static int lut_interp_fp64_entry(const double* lattice64, const double* tri, const double* cdiff, int grid_n,
                                 int method, int angular_mask, const void* rgb, int in_dtype, void* out,
                                 int out_dtype, int64_t n, int layout, void* stream);

extern "C" int mact_lut_interp_cached(const double* lattice64, const double* trilinear,
                                      const double* corner_diff, int grid_n, int method, int angular_mask,
                                      const void* rgb, int in_dtype, void* out, int out_dtype, int64_t n,
                                      int layout, void* stream) {
  if (n > 0 && (!trilinear || !corner_diff)) return set_error(MACT_EBADARG, "caching interpolation needs the cache");
  return lut_interp_fp64_entry(lattice64, trilinear, corner_diff, grid_n, method, angular_mask, rgb, in_dtype,
                               out, out_dtype, n, layout, stream);
}

extern "C" int mact_lut_interp_real(const double* lattice64, int grid_n, int method, int angular_mask,
                                    const void* rgb, int in_dtype, void* out, int out_dtype, int64_t n,
                                    int layout, void* stream) {
  return lut_interp_fp64_entry(lattice64, nullptr, nullptr, grid_n, method, angular_mask, rgb, in_dtype, out,
                               out_dtype, n, layout, stream);
}

static int lut_interp_fp64_entry(const double* lattice64, const double* tri, const double* cdiff, int grid_n,
                                 int method, int angular_mask, const void* rgb, int in_dtype, void* out,
                                 int out_dtype, int64_t n, int layout, void* stream) {
  if (n < 0 || (n > 0 && (!lattice64 || !rgb || !out))) return set_error(MACT_EBADARG, "bad argument");
  if (angular_mask < 0 || angular_mask > 7) return set_error(MACT_EBADARG, "bad angular mask %d", angular_mask);
  if (layout != MACT_LAYOUT_INTERLEAVED && layout != MACT_LAYOUT_PLANAR)
    return set_error(MACT_EBADARG, "unknown layout %d", layout);
  if (out_dtype != MACT_DTYPE_F32 && out_dtype != MACT_DTYPE_F64)
    return set_error(MACT_EBADARG, "out_dtype must be f32 or f64 (%d)", out_dtype);
  if (grid_n != 9 && grid_n != 17 && grid_n != 33) return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
  if (method < 0 || method > 3) return set_error(MACT_EBADARG, "unknown interpolation method %d", method);
  if (n == 0) return MACT_OK;
  const int planar = layout == MACT_LAYOUT_PLANAR;
  cudaStream_t st = (cudaStream_t)stream;
  switch (in_dtype) {
    case MACT_DTYPE_U8:
      return interp_fp64_out(out_dtype, grid_n, method, angular_mask, lattice64, (const uint8_t*)rgb, out, n,
                             planar, st, tri, cdiff);
    case MACT_DTYPE_F32:
      return interp_fp64_out(out_dtype, grid_n, method, angular_mask, lattice64, (const float*)rgb, out, n,
                             planar, st, tri, cdiff);
    case MACT_DTYPE_F64:
      return interp_fp64_out(out_dtype, grid_n, method, angular_mask, lattice64, (const double*)rgb, out, n,
                             planar, st, tri, cdiff);
  }
  return set_error(MACT_EBADARG, "unsupported input dtype %d", in_dtype);
}

extern "C" int mact_lut_nodes_timed(int grid_n, int method, const uint8_t* rgb, int64_t n, int32_t* nodes,
                                    float* weights, void* stream) {
  if (n < 0 || (n > 0 && (!rgb || !nodes || !weights))) return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (grid_n) {
    case 9: return nodes_timed_grid<9>(method, rgb, n, nodes, weights, st);
    case 17: return nodes_timed_grid<17>(method, rgb, n, nodes, weights, st);
    case 33: return nodes_timed_grid<33>(method, rgb, n, nodes, weights, st);
  }
  return set_error(MACT_EBADARG, "grid_n must be one of 9, 17, 33");
}
