// mact_lut.cuh — 3D-LUT cell location and simplex selection (K4 device side).
//
// Follows mact/lut.py:98-199 with INTEGER arithmetic:
//   x = p (n-1) ; base = min(x div 255, n-2) ; rem = x - 255 base   (lut.py:98-105)
// so frac = rem/255 and every comparison between offsets (prism dg >= db,
// pyramid strict/tie rules, tetrahedral stable descending sort) is made on
// the integers rem_r, rem_g, rem_b.  Because spacing = 255/(n-1) is an exact
// binary fraction for n in {9,17,33}, the reference's fp64 frac is the
// correctly rounded rem/255 and orders identically (tests pin this on the
// full cube).  Weights are integer products / 255^k, exact until one final
// rounding.  Node order and accumulation order match the reference
// (out += w_j * V[node_j], j ascending, lut.py:233-236).
#pragma once

#include "mact_common.cuh"

namespace mact {

template <int METHOD>
struct LutK;
template <> struct LutK<MACT_LUT_TRILINEAR> { static constexpr int K = 8; };
template <> struct LutK<MACT_LUT_PRISM> { static constexpr int K = 6; };
template <> struct LutK<MACT_LUT_PYRAMIDAL> { static constexpr int K = 5; };
template <> struct LutK<MACT_LUT_TETRAHEDRAL> { static constexpr int K = 4; };

// Unsigned on purpose: a signed x / 255 compiles to a 4-instruction
// sign-corrected sequence (IMAD.HI + SHF + LEA.HI.SX32 + a zeroed
// accumulator), the unsigned one to IMAD.HI.U32 + SHF.
// x / 255 for x = p (n-1) <= 8160 is hi(x * 0x01010102): exact on that range
// (checked exhaustively), one IMAD.HI without the shift of the general
// 32-bit division sequence.
template <int N>
__device__ __forceinline__ void lut_locate(uint32_t p, int& base, int& rem) {
  static_assert(N >= 2 && N <= 33, "shift-free /255 is exact for p (n-1) <= 8160");
  if constexpr (N == 9 || N == 17 || N == 33) {
    // 256 / (n-1) = 2^S: min(p (n-1) div 255, n-2) == p >> S for every byte p,
    // the clamp of p = 255 included (255 >> S = n-2), so the cell is one shift
    // -- no IMAD.HI (not a full-rate instruction) and no clamp.  Checked
    // exhaustively in tests/test_host_logic.py.
    constexpr int S = N == 9 ? 5 : N == 17 ? 4 : 3;
    const uint32_t bse = p >> S;
    base = (int)bse;
    rem = (int)(p * (uint32_t)(N - 1) - 255u * bse);
  } else {
    // hi(p (n-1) * 0x01010102) with the factor n-1 folded into the magic (< 2^32 for n <= 33)
    uint32_t bse = __umulhi(p, 0x01010102u * (uint32_t)(N - 1));
    bse = bse > (uint32_t)(N - 2) ? (uint32_t)(N - 2) : bse;
    base = (int)bse;
    rem = (int)(p * (uint32_t)(N - 1) - 255u * bse);
  }
}

// Node flat indices and weights of one pixel.  rem values in [0,255].
// TIES = false (interpolation only): the tetrahedral order comes from
// max / min / sum instead of the stable sort.  The weights are the same
// integers; under ties the zero-weight middle node may be a different corner
// of the cell, which leaves every sum bit-identical (fmaf(0, v, a) == a).
// mact_lut_nodes reports the reference's indices and keeps TIES = true.
// lut_nodes_at: the same from the located cell (bf = flat index of its base
// corner in a lattice of N nodes per axis, rr/rg/rb = the integer offsets);
// lut_nodes locates first.
template <int N, int METHOD, typename W = float, bool TIES = true>
__device__ __forceinline__ void lut_nodes_at(int bf, int rr, int rg, int rb,
                                             int (&idx)[LutK<METHOD>::K],
                                             W (&w)[LutK<METHOD>::K]) {
  constexpr int SR = N * N, SG = N, SB = 1;
  const W fr = (W)rr, fg = (W)rg, fb = (W)rb;
  constexpr W inv1 = (W)(1.0 / 255.0);
  constexpr W inv2 = (W)(1.0 / (255.0 * 255.0));
  constexpr W inv3 = (W)(1.0 / (255.0 * 255.0 * 255.0));
  if constexpr (METHOD == MACT_LUT_TRILINEAR) {
    const W ar[2] = {(W)255 - fr, fr}, ag[2] = {(W)255 - fg, fg}, ab[2] = {(W)255 - fb, fb};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int cr = c >> 2 & 1, cg = c >> 1 & 1, cb = c & 1;
      idx[c] = bf + cr * SR + cg * SG + cb * SB;
      w[c] = (ar[cr] * ag[cg] * ab[cb]) * inv3;      // product < 2^24: exact
    }
  } else if constexpr (METHOD == MACT_LUT_PRISM) {
    const bool up = rg >= rb;                        // lut.py:146
    const W ta = up ? (W)255 - fg : (W)255 - fb;
    const W tb = (W)(up ? rg - rb : rb - rg);
    const W tc = up ? fb : fg;
    const int mid = up ? SG : SB, far = SG + SB;
    const W a0 = (W)255 - fr;
    idx[0] = bf; idx[1] = bf + mid; idx[2] = bf + far;
    idx[3] = bf + SR; idx[4] = bf + mid + SR; idx[5] = bf + far + SR;
    w[0] = ta * a0 * inv2; w[1] = tb * a0 * inv2; w[2] = tc * a0 * inv2;
    w[3] = ta * fr * inv2; w[4] = tb * fr * inv2; w[5] = tc * fr * inv2;
  } else if constexpr (METHOD == MACT_LUT_PYRAMIDAL) {
    const bool sel_r = (rg > rr) & (rb > rr);        // lut.py:166-167
    const bool sel_g = !sel_r & (rr >= rg) & (rb >= rg);
    const int m = sel_r ? rr : sel_g ? rg : rb;
    const int u = sel_r ? rg : rr;
    const int v = sel_r ? rb : sel_g ? rb : rg;
    const int nu = sel_r ? SG : SR;
    const int nv = (sel_r | sel_g) ? SB : SG;
    const W fu = (W)u, fv = (W)v;
    idx[0] = bf; idx[1] = bf + nu; idx[2] = bf + nv; idx[3] = bf + nu + nv;
    idx[4] = bf + SR + SG + SB;
    w[0] = ((W)255 - fu) * ((W)255 - fv) * inv2;
    w[1] = fu * ((W)255 - fv) * inv2;
    w[2] = fv * ((W)255 - fu) * inv2;
    w[3] = (W)(u * v - 255 * m) * inv2;
    w[4] = (W)m * inv1;
  } else if constexpr (!TIES) {
    // keys offset << 16 | stride: max3 / min3 give the largest / smallest offset
    // together with its axis (under ties any of the tied axes: the node it
    // selects carries weight 0): two 3-input min / max, two shifts and two masks
    // in place of four compares and four selects.  (Routing the shifts and field
    // extractions through IMAD.HI with multipliers ptxas cannot fold -- FMA pipe
    // instead of ALU -- measured 20 % slower on every LUT kernel: IMAD.HI is not
    // a full-rate instruction.)
    static_assert(SR < 65536, "stride field");
    const uint32_t kr = ((uint32_t)rr << 16) + (uint32_t)SR, kg = ((uint32_t)rg << 16) + (uint32_t)SG,
                   kb = ((uint32_t)rb << 16) + (uint32_t)SB;
    const uint32_t k1 = max(kr, max(kg, kb)), k3 = min(kr, min(kg, kb));
    const int d1 = (int)(k1 >> 16), d3 = (int)(k3 >> 16);
    const int s1 = (int)(k1 & 0xFFFFu), s3 = (int)(k3 & 0xFFFFu);
    const int d2 = rr + rg + rb - d1 - d3;
    idx[0] = bf; idx[1] = bf + s1; idx[2] = bf + SR + SG + SB - s3; idx[3] = bf + SR + SG + SB;
    const W f1 = (W)d1, f2 = (W)d2, f3 = (W)d3;              // integers <= 255: the differences are exact
    w[0] = ((W)255 - f1) * inv1;
    w[1] = (f1 - f2) * inv1;
    w[2] = (f2 - f3) * inv1;
    w[3] = f3 * inv1;
  } else {
    // stable argsort of -d (lut.py:185): ties keep r before g before b
    const int pos_r = (rg > rr) + (rb > rr);
    const int pos_g = (rr >= rg) + (rb > rg);
    const int s1 = pos_r == 0 ? SR : pos_g == 0 ? SG : SB;
    const int d1 = pos_r == 0 ? rr : pos_g == 0 ? rg : rb;
    const int s2 = pos_r == 1 ? SR : pos_g == 1 ? SG : SB;
    const int d2 = pos_r == 1 ? rr : pos_g == 1 ? rg : rb;
    const int d3 = pos_r == 2 ? rr : pos_g == 2 ? rg : rb;
    idx[0] = bf; idx[1] = bf + s1; idx[2] = bf + s1 + s2; idx[3] = bf + SR + SG + SB;
    w[0] = (W)(255 - d1) * inv1;
    w[1] = (W)(d1 - d2) * inv1;
    w[2] = (W)(d2 - d3) * inv1;
    w[3] = (W)d3 * inv1;
  }
}

template <int N, int METHOD, typename W = float, bool TIES = true>
__device__ __forceinline__ void lut_nodes(uint32_t pr, uint32_t pg, uint32_t pb,
                                          int (&idx)[LutK<METHOD>::K],
                                          W (&w)[LutK<METHOD>::K]) {
  int br, bg, bb, rr, rg, rb;
  lut_locate<N>(pr, br, rr);
  lut_locate<N>(pg, bg, rg);
  lut_locate<N>(pb, bb, rb);
  lut_nodes_at<N, METHOD, W, TIES>((br * N + bg) * N + bb, rr, rg, rb, idx, w);
}

// Real-valued pixels (lut.py:98-105 and :115-199 in fp64, the reference's
// evaluation order): x = p / spacing, base = clamp(floor(x), 0, n-2),
// frac = x - base (> 1 or < 0 outside [0, 255]: the reference extrapolates).
template <int N>
__device__ __forceinline__ void lut_locate_real(double p, int& base, double& frac) {
  constexpr double spacing = 255.0 / (N - 1);         // exact for n = 9, 17, 33
  const double x = __ddiv_rn(p, spacing);
  double f = floor(x);
  f = f > (double)(N - 2) ? (double)(N - 2) : f;
  f = f < 0.0 ? 0.0 : f;
  base = (int)f;
  frac = __dadd_rn(x, -f);
}

template <int N, int METHOD>
__device__ __forceinline__ void lut_nodes_real(double pr, double pg, double pb,
                                               int (&idx)[LutK<METHOD>::K], double (&w)[LutK<METHOD>::K],
                                               double (&d)[3]) {
  constexpr int SR = N * N, SG = N, SB = 1;
  int br, bg, bb;
  lut_locate_real<N>(pr, br, d[0]);
  lut_locate_real<N>(pg, bg, d[1]);
  lut_locate_real<N>(pb, bb, d[2]);
  const double dr = d[0], dg = d[1], db = d[2];
  const int bf = (br * N + bg) * N + bb;
  if constexpr (METHOD == MACT_LUT_TRILINEAR) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double wr = (c >> 2) & 1 ? dr : __dadd_rn(1.0, -dr);
      const double wg = (c >> 1) & 1 ? dg : __dadd_rn(1.0, -dg);
      const double wb = c & 1 ? db : __dadd_rn(1.0, -db);
      idx[c] = bf + ((c >> 2) & 1) * SR + ((c >> 1) & 1) * SG + (c & 1) * SB;
      w[c] = __dmul_rn(__dmul_rn(wr, wg), wb);
    }
  } else if constexpr (METHOD == MACT_LUT_PRISM) {
    const bool up = dg >= db;
    const double ta = up ? __dadd_rn(1.0, -dg) : __dadd_rn(1.0, -db);
    const double tb = up ? __dadd_rn(dg, -db) : __dadd_rn(db, -dg);
    const double tc = up ? db : dg;
    const int mid = up ? SG : SB, far = SG + SB;
    const double a0 = __dadd_rn(1.0, -dr);
    idx[0] = bf; idx[1] = bf + mid; idx[2] = bf + far;
    idx[3] = bf + SR; idx[4] = bf + mid + SR; idx[5] = bf + far + SR;
    w[0] = __dmul_rn(ta, a0); w[1] = __dmul_rn(tb, a0); w[2] = __dmul_rn(tc, a0);
    w[3] = __dmul_rn(ta, dr); w[4] = __dmul_rn(tb, dr); w[5] = __dmul_rn(tc, dr);
  } else if constexpr (METHOD == MACT_LUT_PYRAMIDAL) {
    const bool sel_r = (dg > dr) && (db > dr);
    const bool sel_g = !sel_r && (dr >= dg) && (db >= dg);
    const double dm = sel_r ? dr : sel_g ? dg : db;
    const double du = sel_r ? dg : dr;
    const double dv = sel_r ? db : sel_g ? db : dg;
    const int nu = sel_r ? SG : SR;
    const int nv = (sel_r || sel_g) ? SB : SG;
    idx[0] = bf; idx[1] = bf + nu; idx[2] = bf + nv; idx[3] = bf + nu + nv; idx[4] = bf + SR + SG + SB;
    w[0] = __dmul_rn(__dadd_rn(1.0, -du), __dadd_rn(1.0, -dv));
    w[1] = __dmul_rn(du, __dadd_rn(1.0, -dv));
    w[2] = __dmul_rn(dv, __dadd_rn(1.0, -du));
    w[3] = __dadd_rn(__dmul_rn(du, dv), -dm);
    w[4] = dm;
  } else {
    // stable argsort of -d (lut.py:185): ties keep r before g before b
    const int pos_r = (dg > dr) + (db > dr);
    const int pos_g = (dr >= dg) + (db > dg);
    const int s1 = pos_r == 0 ? SR : pos_g == 0 ? SG : SB;
    const double d1 = pos_r == 0 ? dr : pos_g == 0 ? dg : db;
    const int s2 = pos_r == 1 ? SR : pos_g == 1 ? SG : SB;
    const double d2 = pos_r == 1 ? dr : pos_g == 1 ? dg : db;
    const double d3 = pos_r == 2 ? dr : pos_g == 2 ? dg : db;
    idx[0] = bf; idx[1] = bf + s1; idx[2] = bf + s1 + s2; idx[3] = bf + SR + SG + SB;
    w[0] = __dadd_rn(1.0, -d1);
    w[1] = __dadd_rn(d1, -d2);
    w[2] = __dadd_rn(d2, -d3);
    w[3] = d3;
  }
}

// lut.angular_lerp (lut.py:202-216): circular interpolation wrapped to
// [0, 2 pi); a vanishing blended direction resolves to theta0 mod 2 pi.
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

}  // namespace mact
