// mact_runtime.cu — host-side runtime of libmact_cuda: error reporting,
// coefficient packing (MactConfig -> kernel parameter block), persistent-grid
// sizing, launch accounting.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include <nvtx3/nvToolsExt.h>

#include "mact_common.cuh"

namespace mact {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

void count_launch(int k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(MACT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return MACT_OK;
}

int num_sms() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  cache[dev] = sms;
  return sms;
}

int persistent_grid(const void* fn, int threads, size_t smem_bytes) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(fn, threads, smem_bytes, dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_bytes);
  if (e != cudaSuccess) {
    set_error(MACT_ECUDA, "cudaFuncSetAttribute(%zu B smem): %s", smem_bytes,
              cudaGetErrorString(e));
    return -1;
  }
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem_bytes);
  if (e != cudaSuccess) {
    set_error(MACT_ECUDA, "occupancy query: %s", cudaGetErrorString(e));
    return -1;
  }
  if (occ < 1) occ = 1;
  const int grid = occ * num_sms();
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = grid;
  return grid;
}

// MactConfig -> kernel coefficient block.  Degree bounds follow the bundled
// registry (approximants.py:168-265): CIELAB rationals n,m in 2..4, the HSI
// refit 2..5, SCT polynomials 4..5.  Anything else is UnknownApproximant.
int make_kcoeffs(const MactCoeffs* c, KCoeffs* k) {
  if (c == nullptr) return set_error(MACT_EBADARG, "null coefficient block");
  auto bad = [](int d, int lo, int hi) { return d < lo || d > hi; };
  if (bad(c->cbrt_num_deg, 2, kCbrtDeg) || bad(c->cbrt_den_deg, 2, kCbrtDeg))
    return set_error(MACT_EUNKNOWN_APPROX, "no CIELAB rational with degrees (%d,%d)",
                     c->cbrt_num_deg, c->cbrt_den_deg);
  if (bad(c->hsi_deg, 2, kPolyDeg))
    return set_error(MACT_EUNKNOWN_APPROX, "no atan_sqrt3 polynomial of degree %d", c->hsi_deg);
  if (bad(c->asin_deg, 4, kPolyDeg) || bad(c->acos_deg, 4, kPolyDeg) ||
      bad(c->atan_deg, 4, kPolyDeg))
    return set_error(MACT_EUNKNOWN_APPROX, "no SCT polynomials with degrees (%d,%d,%d)",
                     c->asin_deg, c->acos_deg, c->atan_deg);
  auto fill_d = [](double* dst, const double* src, int deg, int cap) {
    for (int i = 0; i <= cap; ++i) dst[i] = i <= deg ? src[i] : 0.0;
  };
  fill_d(k->cbrt_num, c->cbrt_num, c->cbrt_num_deg, kCbrtDeg);
  fill_d(k->cbrt_den, c->cbrt_den, c->cbrt_den_deg, kCbrtDeg);
  fill_d(k->hsi_d, c->atan_sqrt3, c->hsi_deg, kPolyDeg);
  fill_d(k->asin_d, c->asin_half, c->asin_deg, kPolyDeg);
  fill_d(k->acos_d, c->acos_half, c->acos_deg, kPolyDeg);
  fill_d(k->atanf_d, c->atan_f, c->atan_deg, kPolyDeg);
  fill_d(k->atang_d, c->atan_g, c->atan_deg, kPolyDeg);
  for (int i = 0; i <= kPolyDeg; ++i) {
    k->hsi[i] = (float)k->hsi_d[i];
    k->asin[i] = (float)k->asin_d[i];
    k->acos[i] = (float)k->acos_d[i];
    k->atanf[i] = (float)k->atanf_d[i];
    k->atang[i] = (float)k->atang_d[i];
  }
  const double white[3] = {kWhiteX, kWhiteY, kWhiteZ};
  for (int r = 0; r < 3; ++r)
    for (int col = 0; col < 3; ++col) k->mxyz[r * 3 + col] = (float)(rgb2xyz(r, col) / white[r]);
  k->monic44 = (c->cbrt_num_deg == 4 && c->cbrt_den_deg == 4 && c->cbrt_num[4] != 0.0 &&
                c->cbrt_den[4] != 0.0) ? 1 : 0;
  if (k->monic44) {
    const double p4 = c->cbrt_num[4], q4 = c->cbrt_den[4], kk = p4 / q4;
    double pm[4];
    for (int i = 0; i < 4; ++i) {
      pm[i] = c->cbrt_num[i] / p4;
      k->qm[i] = c->cbrt_den[i] / q4;
    }
    const double e3 = pm[3] - k->qm[3];          // leading coefficient of P' - Q'
    if (e3 == 0.0) {
      k->monic44 = 0;
    } else {
      for (int i = 0; i < 3; ++i) k->dm[i] = (pm[i] - k->qm[i]) / e3;
      const double sc = kk * e3;
      k->lin_s = kLabSlope / sc;
      k->lin_o = (kLabOffset - kk) / sc;
      k->l_s = 116.0 * sc;
      k->l_o = 116.0 * kk - 16.0;
      k->a_s = (float)(500.0 * sc);
      k->b_s = (float)(200.0 * sc);
    }
  }
  return MACT_OK;
}

}  // namespace mact

extern "C" const char* mact_last_error(void) { return mact::g_last_error.c_str(); }
extern "C" int mact_version(void) { return 100; }
extern "C" uint64_t mact_launch_count(void) { return mact::g_launches.load(); }
extern "C" void mact_launch_count_reset(void) { mact::g_launches.store(0); }
