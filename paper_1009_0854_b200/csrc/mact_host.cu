// mact_host.cu — host streaming executor: the end-to-end path over HOST buffers.
//
// The reference's transforms take and return host numpy arrays
// (fast.py:86, :125, :188).  A drop-in therefore pays host<->device
// transfers; this executor hides them behind each other and behind compute:
// the pixel stream is cut into chunks, chunk k runs H2D -> kernel -> D2H on
// stream k % nstreams, so the H2D engine, the SMs and the D2H engine work on
// three different chunks at once.  Pinned host buffers are DMA'd directly;
// pageable buffers are staged through pinned bounce buffers, with the CPU
// memcpy of chunk k overlapping the DMA of chunk k-1.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "mact_common.cuh"

struct MactHostCtx {
  int device = 0;
  int64_t chunk = 0;
  int nstreams = 0;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> done;        // per stream: last D2H of that slot finished
  std::vector<uint8_t*> d_in;
  std::vector<char*> d_out;             // chunk x 24 B: fp32 (12 B/px) or fp64 (24 B/px) results
  std::vector<uint8_t*> h_in;           // pinned bounce buffers (pageable callers)
  std::vector<char*> h_out;
  std::mutex mu;                        // one call at a time owns the streams and staging buffers
};

using namespace mact;

static constexpr size_t kMaxOutPx = 24;   // bytes per pixel of a staging slot (fp64 (N,3))

// Parallel memcpy for the pageable staging path: one host thread moves ~5-10
// GB/s (less while first-touch page faults land in a fresh numpy array), so
// large copies are split across hardware threads.
static void par_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t kMinPerThread = 4u << 20;
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  size_t nt = std::min<size_t>(std::min<size_t>(hw, 16), std::max<size_t>(1, bytes / kMinPerThread));
  if (nt <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t part = (bytes + nt - 1) / nt;
  for (size_t i = 0; i < nt; ++i) {
    const size_t lo = i * part, hi = std::min(bytes, lo + part);
    if (lo >= hi) break;
    th.emplace_back([=] { memcpy((char*)dst + lo, (const char*)src + lo, hi - lo); });
  }
  for (auto& t : th) t.join();
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

extern "C" int mact_host_ctx_create(int device, int64_t chunk_px, int nstreams, MactHostCtx** out) {
  if (!out || chunk_px <= 0 || nstreams <= 0 || nstreams > 16)
    return set_error(MACT_EBADARG, "bad host-context arguments");
  chunk_px = (chunk_px + 2047) / 2048 * 2048;
  auto* c = new MactHostCtx();
  c->device = device;
  c->chunk = chunk_px;
  c->nstreams = nstreams;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  for (int s = 0; s < nstreams && e == cudaSuccess; ++s) {
    cudaStream_t st;
    cudaEvent_t ev;
    uint8_t* di = nullptr;
    char* dout = nullptr;
    if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) break;
    c->streams.push_back(st);
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) break;
    c->done.push_back(ev);
    if ((e = cudaMalloc(&di, (size_t)chunk_px * 3)) != cudaSuccess) break;
    c->d_in.push_back(di);
    if ((e = cudaMalloc(&dout, (size_t)chunk_px * kMaxOutPx)) != cudaSuccess) break;
    c->d_out.push_back(dout);
  }
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    mact_host_ctx_destroy(c);
    return set_error(MACT_ECUDA, "host context: %s", cudaGetErrorString(e));
  }
  *out = c;
  return MACT_OK;
}

extern "C" int mact_host_ctx_destroy(MactHostCtx* c) {
  if (!c) return MACT_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  for (auto s : c->streams) cudaStreamSynchronize(s);
  for (auto p : c->d_in) cudaFree(p);
  for (auto p : c->d_out) cudaFree(p);
  for (auto p : c->h_in) cudaFreeHost(p);
  for (auto p : c->h_out) cudaFreeHost(p);
  for (auto e : c->done) cudaEventDestroy(e);
  for (auto s : c->streams) cudaStreamDestroy(s);
  cudaSetDevice(prev);
  delete c;
  return MACT_OK;
}

static int ensure_bounce(MactHostCtx* c) {
  if (!c->h_in.empty()) return MACT_OK;
  for (int s = 0; s < c->nstreams; ++s) {
    uint8_t* hi = nullptr;
    char* ho = nullptr;
    cudaError_t e = cudaHostAlloc(&hi, (size_t)c->chunk * 3, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&ho, (size_t)c->chunk * kMaxOutPx, cudaHostAllocDefault);
    if (e != cudaSuccess) return set_error(MACT_ECUDA, "pinned bounce buffers: %s", cudaGetErrorString(e));
    c->h_in.push_back(hi);
    c->h_out.push_back(ho);
  }
  return MACT_OK;
}

static int run_kernel(int op, const uint8_t* din, float* dout, int64_t n, const MactCoeffs* cf,
                      int layout, cudaStream_t st) {
  switch (op) {
    case MACT_SPACE_LAB: return mact_lab_fast(din, MACT_DTYPE_U8, dout, n, cf, layout, st);
    case MACT_SPACE_HSI: return mact_hsi_fast(din, MACT_DTYPE_U8, dout, n, cf, layout, st);
    case MACT_SPACE_SCT: return mact_sct_fast(din, MACT_DTYPE_U8, dout, n, cf, layout, st);
  }
  return set_error(MACT_EBADARG, "unknown transform %d", op);
}

// D2H of one chunk's result (es = 4 or 8 bytes per component); planar output
// lands in 3 strided host planes.
static cudaError_t copy_out(char* host_out, const char* dout, int64_t off, int64_t m, int64_t n,
                            int layout, size_t es, cudaStream_t st) {
  if (layout == MACT_LAYOUT_INTERLEAVED)
    return cudaMemcpyAsync(host_out + 3 * off * es, dout, (size_t)m * 3 * es, cudaMemcpyDeviceToHost, st);
  return cudaMemcpy2DAsync(host_out + off * es, (size_t)n * es, dout, (size_t)m * es, (size_t)m * es, 3,
                           cudaMemcpyDeviceToHost, st);
}

// The chunk pipeline shared by every host entry point; `launch` runs the
// kernel of one chunk (device in, device out, pixels, stream); es = bytes per
// output component (4: fp32, 8: the fp64 fidelity mode).
template <class Launch>
static int stream_host(MactHostCtx* c, const uint8_t* host_rgb, void* host_out_v, int64_t n,
                       int layout, size_t es, Launch&& launch) {
  char* host_out = static_cast<char*>(host_out_v);
  std::lock_guard<std::mutex> guard(c->mu);
  NvtxRange range("mact_host_stream");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  const bool direct = is_pinned(host_rgb) && is_pinned(host_out);
  int rc = MACT_OK;
  if (!direct) rc = ensure_bounce(c);
  // Small inputs are cut into at least 2 x nstreams chunks (>= 64 Ki px, multiple
  // of 2048) so their H2D, kernel and D2H still overlap; large ones use the
  // context's chunk size.
  int64_t chunk = c->chunk;
  if (n < c->chunk * 2 * c->nstreams) {
    chunk = (n + 2 * c->nstreams - 1) / (2 * c->nstreams);
    chunk = std::max<int64_t>(65536, (chunk + 2047) / 2048 * 2048);
    chunk = std::min<int64_t>(chunk, c->chunk);
  }
  const int64_t nchunks = (n + chunk - 1) / chunk;
  // slot bookkeeping for pageable callers: chunk that last used each slot
  std::vector<int64_t> pending(c->nstreams, -1);
  auto drain = [&](int s) -> int {
    const int64_t k = pending[s];
    if (k < 0) return MACT_OK;
    cudaError_t e = cudaEventSynchronize(c->done[s]);
    if (e != cudaSuccess) return set_error(MACT_ECUDA, "d2h: %s", cudaGetErrorString(e));
    const int64_t off = k * chunk, m = std::min<int64_t>(chunk, n - off);
    if (layout == MACT_LAYOUT_INTERLEAVED) {
      par_memcpy(host_out + 3 * off * es, c->h_out[s], (size_t)m * 3 * es);
    } else {
      for (int p = 0; p < 3; ++p)
        par_memcpy(host_out + (p * n + off) * es, c->h_out[s] + p * m * es, (size_t)m * es);
    }
    pending[s] = -1;
    return MACT_OK;
  };
  for (int64_t k = 0; k < nchunks && rc == MACT_OK; ++k) {
    const int s = (int)(k % c->nstreams);
    cudaStream_t st = c->streams[s];
    const int64_t off = k * chunk, m = std::min<int64_t>(chunk, n - off);
    cudaError_t e;
    if (direct) {
      e = cudaMemcpyAsync(c->d_in[s], host_rgb + 3 * off, (size_t)m * 3, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) rc = launch(c->d_in[s], c->d_out[s], m, st);
      if (rc == MACT_OK && e == cudaSuccess) e = copy_out(host_out, c->d_out[s], off, m, n, layout, es, st);
    } else {
      if ((rc = drain(s)) != MACT_OK) break;
      par_memcpy(c->h_in[s], host_rgb + 3 * off, (size_t)m * 3);
      e = cudaMemcpyAsync(c->d_in[s], c->h_in[s], (size_t)m * 3, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) rc = launch(c->d_in[s], c->d_out[s], m, st);
      if (rc == MACT_OK && e == cudaSuccess)
        e = cudaMemcpyAsync(c->h_out[s], c->d_out[s], (size_t)m * 3 * es, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaEventRecord(c->done[s], st);
      pending[s] = k;
    }
    if (e != cudaSuccess) rc = set_error(MACT_ECUDA, "host stream: %s", cudaGetErrorString(e));
  }
  if (!direct)
    for (int s = 0; s < c->nstreams && rc == MACT_OK; ++s) rc = drain(s);
  for (auto st : c->streams) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess && rc == MACT_OK) rc = set_error(MACT_ECUDA, "sync: %s", cudaGetErrorString(e));
  }
  cudaSetDevice(prev);
  return rc;
}

extern "C" int mact_transform_host(MactHostCtx* c, int op, const uint8_t* host_rgb, float* host_out,
                                   int64_t n, const MactCoeffs* cf, int layout) {
  if (!c || n < 0 || (n > 0 && (!host_rgb || !host_out)) || !cf)
    return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  if (op < 0 || op > 2) return set_error(MACT_EBADARG, "unknown transform %d", op);
  return stream_host(c, host_rgb, host_out, n, layout, 4,
                     [&](const uint8_t* din, char* dout, int64_t m, cudaStream_t st) {
                       return run_kernel(op, din, reinterpret_cast<float*>(dout), m, cf, layout, st);
                     });
}

extern "C" int mact_transform_host_f64(MactHostCtx* c, int op, const uint8_t* host_rgb, double* host_out,
                                       int64_t n, const MactCoeffs* cf, int layout) {
  if (!c || n < 0 || (n > 0 && (!host_rgb || !host_out)) || !cf)
    return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  if (op < 0 || op > 2) return set_error(MACT_EBADARG, "unknown transform %d", op);
  return stream_host(c, host_rgb, host_out, n, layout, 8,
                     [&](const uint8_t* din, char* dout, int64_t m, cudaStream_t st) {
                       return mact_fast_f64(op, din, MACT_DTYPE_U8, reinterpret_cast<double*>(dout), m, cf,
                                            layout, st);
                     });
}

extern "C" int mact_lut_interp_host(MactHostCtx* c, const float* lattice, int grid_n, int method,
                                    const uint8_t* host_rgb, float* host_out, int64_t n, int layout) {
  if (!c || !lattice || n < 0 || (n > 0 && (!host_rgb || !host_out)))
    return set_error(MACT_EBADARG, "bad argument");
  if (n == 0) return MACT_OK;
  return stream_host(c, host_rgb, host_out, n, layout, 4,
                     [&](const uint8_t* din, char* dout, int64_t m, cudaStream_t st) {
                       return mact_lut_interp(lattice, grid_n, method, din, reinterpret_cast<float*>(dout), m,
                                              layout, st);
                     });
}
