/*
 * mact_cuda.h — C ABI of libmact_cuda.so, the B200 (sm_100a) implementation of
 * the MACT per-pixel colour-transform path (arXiv 1009.0854).
 *
 * The reference (`mact` 0.1.0, pure Python/numpy, /root/reference/pkg/src/mact)
 * has no native FFI; its plugin seam is a Python callable
 * `pixels (...,3) -> (...,3) float` (harness.py:71-74, :77-78).  Each entry point
 * below replaces one such reference function and is bound from the Python
 * mirror package `paper_1009_0854_b200` through ctypes (INTEGRATION.md shows
 * the binding a maintainer would add to `mact` itself).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Unless stated otherwise pointers are DEVICE
 *    pointers owned by the caller; the library allocates nothing on the hot
 *    path.  `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Calls are stream-ordered and asynchronous.
 *  - Pixels are interleaved RGB, C order, `n` pixels (the reference's (...,3)
 *    layout, harness.py:35-46).  Outputs are fp32 (the reference returns fp64,
 *    exact.py:48-49; fp32 is the documented deviation, within the north-star
 *    tolerance) — interleaved (N,3) or planar (3,N).
 *  - Return status: MACT_OK, MACT_EBADARG (-> ValueError in Python),
 *    MACT_EUNKNOWN_APPROX (-> UnknownApproximant), MACT_ECUDA (-> MactError);
 *    `mact_last_error()` returns a thread-local message for the last failure.
 */
#ifndef MACT_CUDA_H
#define MACT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MACT_OK = 0,
  MACT_EBADARG = 1,
  MACT_EUNKNOWN_APPROX = 2,
  MACT_ECUDA = 3
};

enum { MACT_SPACE_LAB = 0, MACT_SPACE_HSI = 1, MACT_SPACE_SCT = 2,
       MACT_SPACE_HSI_ARCCOS = 3 /* mact_exact only: exact.rgb_to_hsi_arccos (exact.py:104-116) */ };
enum { MACT_LAYOUT_INTERLEAVED = 0, MACT_LAYOUT_PLANAR = 1 };
enum { MACT_DTYPE_U8 = 0, MACT_DTYPE_F32 = 1, MACT_DTYPE_F64 = 2 };
enum {
  MACT_LUT_TRILINEAR = 0,
  MACT_LUT_PRISM = 1,
  MACT_LUT_PYRAMIDAL = 2,
  MACT_LUT_TETRAHEDRAL = 3
};
enum { MACT_METRIC_DISTANCE = 0, MACT_METRIC_COMPONENT = 1 };
enum { MACT_CAND_FAST = 0, MACT_CAND_LUT = 1, MACT_CAND_ARRAY = 2,
       MACT_CAND_FAST_F64 = 3 /* fast transform in the reference's fp64 arithmetic */ };

#define MACT_MAX_COEFFS 8

/* Coefficient sets resolved from a MactConfig (fast.py:46-78).  Polynomials
 * are ascending a_0..a_deg, evaluated by Horner highest-first
 * (approximants.py:55-71).  Passed BY VALUE to every kernel as a
 * __grid_constant__ parameter: no mutable device globals, so concurrent
 * configurations on different streams are safe. */
typedef struct MactCoeffs {
  int32_t cbrt_num_deg, cbrt_den_deg;  /* CIELAB rational (n, m)      approximants.py:179-213 */
  int32_t hsi_deg;                     /* atan(sqrt3 x) refit degree  fast.py:38-43          */
  int32_t asin_deg, acos_deg, atan_deg;/* SCT (n_asin, m_acos, r_atan) fast.py:67-75         */
  double cbrt_num[MACT_MAX_COEFFS];
  double cbrt_den[MACT_MAX_COEFFS];
  double atan_sqrt3[MACT_MAX_COEFFS];
  double asin_half[MACT_MAX_COEFFS];   /* approximants.py:231-238 */
  double acos_half[MACT_MAX_COEFFS];   /* approximants.py:240-247 */
  double atan_f[MACT_MAX_COEFFS];      /* approximants.py:249-256 */
  double atan_g[MACT_MAX_COEFFS];      /* approximants.py:258-265 */
} MactCoeffs;

/* Per-shard error-statistic partial (harness.py:63-74 semantics):
 * sum of the metric (fp64), number of scored pixels, max value, GLOBAL index
 * of the first pixel attaining it (index_base + local index), and the number
 * of pixels excluded because the exact component is undefined (NaN). */
typedef struct MactErrStats {
  double sum;
  double max;
  uint64_t count;
  uint64_t argmax;
  uint64_t nan_count;
  uint64_t _pad;
} MactErrStats;

/* Candidate description for the fused error reduction. */
typedef struct MactErrSpec {
  int32_t space;        /* MACT_SPACE_*                                      */
  int32_t metric;       /* MACT_METRIC_DISTANCE (harness DISTANCES) or COMPONENT */
  int32_t candidate;    /* MACT_CAND_FAST / _LUT / _ARRAY                      */
  int32_t lut_grid_n;   /* for MACT_CAND_LUT                                   */
  int32_t lut_method;   /* MACT_LUT_*                                          */
  int32_t cand_dtype;   /* MACT_CAND_ARRAY: MACT_DTYPE_F32 / _F64, interleaved */
  const float* lut_lattice;   /* (n^3, 4) fp32 device lattice, r-major          */
  const void* cand_array;     /* (n, 3) candidate outputs                      */
  const void* ref_array;      /* optional (n,3) reference outputs, NULL = exact on device */
  int32_t ref_dtype;
  int32_t _pad;
} MactErrSpec;

/* ---- MACT fast transforms (K1-K3) -------------------------------------- */
/* replaces mact.fast.rgb_to_lab_fast (fast.py:86-107); in_dtype U8 takes the
 * 256-entry gamma table path (fast.py:92-95), F32 the analytic path (:96-99). */
int mact_lab_fast(const void* rgb, int in_dtype, float* out, int64_t n,
                  const MactCoeffs* c, int layout, void* stream);
/* replaces mact.fast.rgb_to_hsi_fast (fast.py:125-148) */
int mact_hsi_fast(const void* rgb, int in_dtype, float* out, int64_t n,
                  const MactCoeffs* c, int layout, void* stream);
/* replaces mact.fast.rgb_to_sct_fast (fast.py:188-203) */
int mact_sct_fast(const void* rgb, int in_dtype, float* out, int64_t n,
                  const MactCoeffs* c, int layout, void* stream);
/* The fast transforms in the reference's own arithmetic: fp64 out, numpy's
 * operation order, every operation rounded once, the fp64 GAMMA_TABLE.
 * Bit-identical to mact.fast.rgb_to_*_fast (fast.py:86-203) for uint8 pixels
 * (and for real-valued HSI/SCT pixels).  space = MACT_SPACE_*; the fidelity
 * mode next to the fp32 throughput path above. */
int mact_fast_f64(int space, const void* rgb, int in_dtype, double* out, int64_t n,
                  const MactCoeffs* c, int layout, void* stream);
/* all three from one read of the pixels (BASELINE config 5); any output may be NULL */
int mact_all_fast(const uint8_t* rgb, float* lab, float* hsi, float* sct, int64_t n,
                  const MactCoeffs* c, int layout, void* stream);

/* ---- exact transforms, fp64 ground truth (K5) --------------------------- */
/* replaces mact.exact.rgb_to_{lab,hsi,sct}_exact (exact.py:86-92, :119-137,
 * :140-149); in_dtype U8/F32/F64, out_dtype F32/F64, interleaved. */
int mact_exact(int space, const void* rgb, int in_dtype, void* out, int out_dtype,
               int64_t n, void* stream);
/* replaces mact.exact.sct_to_rgb (exact.py:152-160), fp64 in/out */
int mact_sct_to_rgb(const double* sct, double* rgb, int64_t n, void* stream);
/* replaces mact.exact.{lab,hsi}_distance / sct_distance_indirect (exact.py:163-190);
 * x, y interleaved (n,3) of dtype F32/F64 each; out fp64 (n). */
int mact_distance(int space, const void* x, int x_dtype, const void* y, int y_dtype,
                  double* out, int64_t n, void* stream);

/* ---- 3D LUT (K4) --------------------------------------------------------- */
/* replaces mact.lut.build_lut (lut.py:82-95): lattice values at k*255/(n-1),
 * NaN -> 0; writes fp64 (n^3,3) and/or the fp32 DEVICE LATTICE (n^3,4):
 * node = (c0, c1, c2, 0), 16-byte aligned (one 16-B load per node).  Either
 * output may be NULL. */
int mact_lut_build(int space, int grid_n, double* lattice_f64, float* lattice_f32,
                   void* stream);
/* replaces mact.lut.interpolate(lut, pixels, method, "standard") (lut.py:231-246,
 * :341-350) for the linear (CIELAB) destination; `lattice` is the (n^3,4)
 * device lattice of mact_lut_build; pixels uint8. */
int mact_lut_interp(const float* lattice, int grid_n, int method, const uint8_t* rgb,
                    float* out, int64_t n, int layout, void* stream);
/* the same for angular destinations: `angular_mask` bit c marks component c as
 * an angle (lut.Lut3D.angular_mask, lut.py:44-48: hsi 1, sct 6), blended on
 * the circle as lut.py:202-262 does (trilinear: cascaded angular_lerp; simplex
 * methods: weighted circular mean); linear components use the weighted sum.
 * Evaluated in fp64 on the fp64 lattice (n^3,3) of mact_lut_build (the
 * circular mean is ill-conditioned near the gray axis). */
int mact_lut_interp_angular(const double* lattice64, int grid_n, int method, int angular_mask,
                            const uint8_t* rgb, float* out, int64_t n, int layout, void* stream);
/* mact.lut.interpolate on any pixel dtype (MACT_DTYPE_U8/F32/F64) and any
 * destination, evaluated in fp64 on the fp64 (n^3,3) lattice: cell location
 * and weights follow lut._locate / node_weights in fp64 (lut.py:98-199;
 * pixels outside [0, 255] extrapolate like the reference), linear
 * components accumulate in the reference's order, angular ones blend on the
 * circle (lut.py:202-262).  out_dtype MACT_DTYPE_F64 on a linear destination
 * is bit-identical to the reference.  mact_lut_interp_angular is its uint8 /
 * fp32-out case. */
int mact_lut_interp_real(const double* lattice64, int grid_n, int method, int angular_mask,
                         const void* rgb, int in_dtype, void* out, int out_dtype, int64_t n, int layout,
                         void* stream);
/* Test/debug entry (no reference counterpart): the node indices and fp32
 * weights exactly as the uint8 INTERPOLATION kernels of mact_lut_interp select
 * them (their own device function: the reference's cells; tetrahedral order
 * from max / min keys, so a tie's zero-weight node may be another corner).  The
 * parity tests check that the nonzero-weight nodes equal lut.node_weights' (lut.py:115-199). */
int mact_lut_nodes_timed(int grid_n, int method, const uint8_t* rgb, int64_t n, int32_t* nodes,
                         float* weights, void* stream);
/* replaces mact.lut.build_cache (lut.py:265-291): per cell of the (n-1)^3
 * cells (r-major) the trilinear polynomial coefficients `trilinear` and the
 * corner differences `corner_diff`, both (n-1)^3 x 8 x 3 fp64 (device),
 * evaluated in the reference's operation order (bit-identical). */
int mact_lut_cache_build(const double* lattice64, int grid_n, double* trilinear, double* corner_diff,
                         void* stream);
/* replaces mact.lut._interpolate_caching (lut.py:294-331), i.e. interpolate(...,
 * variant="caching"): mact_lut_interp_real's contract, with linear components
 * evaluated from the cache arrays in the reference's order (bit-identical with
 * out_dtype MACT_DTYPE_F64). */
int mact_lut_interp_cached(const double* lattice64, const double* trilinear, const double* corner_diff,
                           int grid_n, int method, int angular_mask, const void* rgb, int in_dtype, void* out,
                           int out_dtype, int64_t n, int layout, void* stream);
/* replaces mact.lut.node_weights (lut.py:115-199): flat node indices (n,k)
 * and weights (n,k), k = 8/6/5/4; indices bit-exact with the reference. */
int mact_lut_nodes(int grid_n, int method, const uint8_t* rgb, int64_t n,
                   int32_t* nodes, float* weights, void* stream);
/* the same for any pixel dtype (MACT_DTYPE_U8/F32/F64) with fp64 weights,
 * computed exactly as lut.node_weights does (lut.py:98-199): bit-identical
 * indices and weights */
int mact_lut_nodes_real(int grid_n, int method, const void* rgb, int in_dtype, int64_t n,
                        int32_t* nodes, double* weights, void* stream);

/* ---- error reduction (K6) ------------------------------------------------ */
/* Fused candidate + exact + metric + reduction over pixels rgb[0..n)
 * (harness.measure_error semantics, harness.py:71-122; per-component abs error
 * of SURVEY A21).  Writes 1 (DISTANCE) or 3 (COMPONENT) MactErrStats to
 * `out` (device).  `workspace` must hold mact_err_workspace_bytes() bytes.
 * `rgb` may be NULL with `cube_start` >= 0: pixels are then generated on
 * device as the R-major cube enumeration index cube_start + i (harness.py:35-46). */
size_t mact_err_workspace_bytes(void);
int mact_err_reduce(const MactErrSpec* spec, const MactCoeffs* c, const uint8_t* rgb,
                    int64_t cube_start, int64_t n, int64_t index_base, MactErrStats* out,
                    void* workspace, void* stream);

/* exact.rgb_to_{lab,hsi,sct}_exact formulas (exact.py:60-149) in fp32 with
 * libdevice cbrtf/atanf/acosf/atan2f/sqrtf, uint8 in, fp32 out, on the
 * streaming skeleton: the comparator of the paper's Table 4 gain on B200
 * (SURVEY.md §8(f) item 2).  Not a parity path (fp32 rounding). */
int mact_exact_f32(int space, const uint8_t* rgb, float* out, int64_t n, int layout, void* stream);

/* ---- elementwise building blocks (fp64 device arrays) --------------------- */
/* The reference's scalar approximant functions, bit-identical to numpy:
 *   MACT_FN_FORM        out = a(x) (b_deg < 0) or a(x)/b(x)       fast.cbrt_fast, fast.py:81-83
 *                       (approximants.py:55-82; *degenerate = 1 if any |b(x)| < 1e-300)
 *   MACT_FN_ATAN_SQRT3  out = sign(x) a(|x|)                      fast.atan_sqrt3_fast, fast.py:118-122
 *   MACT_FN_ACOS        out = x < 0.5 ? a(x) : b(sqrt(max(1-x,0)))  fast.acos_fast, fast.py:151-162
 *                       (a = ACOS_HALF, b = ASIN_HALF)
 *   MACT_FN_ATAN_UNIT   out = atan(x/y) split fits, x = g, y = r;   fast.atan_unit_fast, fast.py:165-185
 *                       NaN at g = r = 0 (a = ATAN_F, b = ATAN_G)
 * a[i], b[i] are ascending coefficients; degrees <= 7. */
enum { MACT_FN_FORM = 0, MACT_FN_ATAN_SQRT3 = 1, MACT_FN_ACOS = 2, MACT_FN_ATAN_UNIT = 3 };
typedef struct MactApproxSpec {
  int32_t fn, a_deg, b_deg, _pad;
  double a[8], b[8];
} MactApproxSpec;
int mact_approx_eval(const MactApproxSpec* spec, const double* x, const double* y, double* out,
                     int64_t n, int32_t* degenerate /* device, may be NULL */, void* stream);

/* approximants.eval_poly / eval_rational (approximants.py:55-82), replaces
 * Polynomial.__call__ / Rational.__call__ for any degree < MACT_POLY_MAX:
 * out = num(x) (den_deg < 0) or num(x)/den(x), numpy's Horner order and
 * rounding (bit-identical); *degenerate = 1 if any |den(x)| < 1e-300. */
#define MACT_POLY_MAX 32
typedef struct MactPolySpec {
  int32_t num_deg, den_deg;
  double num[MACT_POLY_MAX], den[MACT_POLY_MAX];
} MactPolySpec;
int mact_poly_eval(const MactPolySpec* spec, const double* x, double* out, int64_t n,
                   int32_t* degenerate /* device, may be NULL */, void* stream);

/* exact.py:52-83 elementwise, fp64:
 *   MACT_ELEM_INVERSE_GAMMA  out0 = inverse_gamma(in0)               (exact.py:52-57)
 *   MACT_ELEM_RGB_TO_XYZ     (out0, out1, out2) = rgb_to_xyz(in0..2)  (exact.py:60-66)
 *   MACT_ELEM_LAB_F          out0 = lab_f(in0)                       (exact.py:69-72)
 *   MACT_ELEM_XYZ_TO_LAB     out0 (n,3) = xyz_to_lab(in0..2)         (exact.py:75-83)
 *   MACT_ELEM_ANGULAR_LERP   out0 = lut.angular_lerp(in0, in1, in2)  (lut.py:202-216) */
enum { MACT_ELEM_INVERSE_GAMMA = 0, MACT_ELEM_RGB_TO_XYZ = 1, MACT_ELEM_LAB_F = 2,
       MACT_ELEM_XYZ_TO_LAB = 3, MACT_ELEM_ANGULAR_LERP = 4,
       /* TargetFn.exact (approximants.py:101-115), out0 = f(in0):
        * cbrt, arctan(sqrt(3) x), 2 arcsin(x / sqrt(2)), arccos, arctan, pi/2 - arctan */
       MACT_ELEM_TARGET_CBRT = 5, MACT_ELEM_TARGET_ATAN_SQRT3 = 6, MACT_ELEM_TARGET_ASIN_HALF = 7,
       MACT_ELEM_TARGET_ACOS_HALF = 8, MACT_ELEM_TARGET_ATAN_F = 9, MACT_ELEM_TARGET_ATAN_G = 10 };
int mact_exact_elem(int op, const double* in0, const double* in1, const double* in2,
                    double* out0, double* out1, double* out2, int64_t n, void* stream);

/* ---- pixel generators ---------------------------------------------------- */
/* harness.cube_chunk (harness.py:35-46) on device: rgb[i] = cube pixel start+i */
int mact_cube_fill(uint8_t* rgb, int64_t start, int64_t n, void* stream);

/* harness.call_probabilities (harness.py:137-175) as exact full-cube counts:
 * counts (device, 6 x u64) = {cbrt_x, cbrt_y, cbrt_z, arcsin, arccos, arctan}
 * call-site hits over all 2^24 colours; probability = count / 2^24. */
int mact_call_counts(unsigned long long* counts, void* stream);

/* ---- host streaming executor (end-to-end, HOST buffers) ------------------ */
/* Runs a fast transform over HOST buffers: chunked H2D -> kernel -> D2H on
 * `nstreams` CUDA streams so both copy engines and the SMs overlap.  Host
 * buffers should be pinned (cudaHostAlloc / registered); pageable buffers are
 * staged through pinned bounce buffers.  op = MACT_SPACE_* (fast transform).
 * Calls on one context are serialised internally (thread-safe). */
typedef struct MactHostCtx MactHostCtx;
int mact_host_ctx_create(int device, int64_t chunk_px, int nstreams, MactHostCtx** ctx);
int mact_host_ctx_destroy(MactHostCtx* ctx);
int mact_transform_host(MactHostCtx* ctx, int op, const uint8_t* host_rgb, float* host_out,
                        int64_t n, const MactCoeffs* c, int layout);
/* The same with fp64 results in the reference's own arithmetic (mact_fast_f64):
 * what mact.fast.rgb_to_*_fast returns for 8-bit pixels, bit for bit
 * (fast.py:86-107, :125-148, :188-203). */
int mact_transform_host_f64(MactHostCtx* ctx, int op, const uint8_t* host_rgb, double* host_out,
                            int64_t n, const MactCoeffs* c, int layout);
/* mact.lut.interpolate over HOST buffers (lut.py:341-350) through the same
 * chunk pipeline; `lattice` is the device (n^3,4) lattice, linear destination. */
int mact_lut_interp_host(MactHostCtx* ctx, const float* lattice, int grid_n, int method,
                         const uint8_t* host_rgb, float* host_out, int64_t n, int layout);

/* ---- calibration ---------------------------------------------------------- */
/* out = (r, g, b) as fp32 through the same streaming kernel: the achievable
 * bandwidth of the 3 B in / 12 B out pattern with no arithmetic (not a
 * reference function; bench.py reports it next to the HBM roofline). */
int mact_probe_expand(const uint8_t* rgb, float* out, int64_t n, void* stream);

/* ---- misc ----------------------------------------------------------------- */
/* How the uint8 fast CIELAB kernels evaluate this configuration's rational
 * (fast.py:110-115): MACT_LAB_PATH_SEG = segmented fp32 cubic (the default
 * when the host-side fit check passes), MACT_LAB_PATH_MONIC = fp64 monic
 * (4,4) quotient, MACT_LAB_PATH_PQ = fp64 P/Q; negative = error status.
 * The environment variable MACT_LAB_EVAL=fp64 (read per call) forces the fp64
 * evaluation.  Host-only (no device work). */
#define MACT_LAB_PATH_SEG 1
#define MACT_LAB_PATH_MONIC 2
#define MACT_LAB_PATH_PQ 3
int mact_lab_eval_path(const MactCoeffs* c);
const char* mact_last_error(void);
int mact_version(void);
/* number of kernel launches issued by this thread since the last reset */
uint64_t mact_launch_count(void);
void mact_launch_count_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* MACT_CUDA_H */
