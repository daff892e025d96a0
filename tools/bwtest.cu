// bwtest.cu — memory-engine calibration for the 3 B in / 12 B out pattern on B200.
// Standalone (not part of libmact_cuda); build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// 1) plain: thread = 4 px, 3 x LDG.32 in (coalesced), 3 x STG.128 out (48 B stride)
__global__ void k_plain(const uint32_t* __restrict__ in, float4* __restrict__ out, int64_t ngrp) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngrp; g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w0 = __ldg(in + 3 * g), w1 = __ldg(in + 3 * g + 1), w2 = __ldg(in + 3 * g + 2);
    float f[12];
    for (int k = 0; k < 4; ++k) { f[k] = (float)((w0 >> (8 * k)) & 255); f[4 + k] = (float)((w1 >> (8 * k)) & 255); f[8 + k] = (float)((w2 >> (8 * k)) & 255); }
    out[3 * g] = make_float4(f[0], f[1], f[2], f[3]);
    out[3 * g + 1] = make_float4(f[4], f[5], f[6], f[7]);
    out[3 * g + 2] = make_float4(f[8], f[9], f[10], f[11]);
  }
}
// 2) same with streaming stores
__global__ void k_plain_cs(const uint32_t* __restrict__ in, float4* __restrict__ out, int64_t ngrp) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ngrp; g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w0 = __ldg(in + 3 * g), w1 = __ldg(in + 3 * g + 1), w2 = __ldg(in + 3 * g + 2);
    float f[12];
    for (int k = 0; k < 4; ++k) { f[k] = (float)((w0 >> (8 * k)) & 255); f[4 + k] = (float)((w1 >> (8 * k)) & 255); f[8 + k] = (float)((w2 >> (8 * k)) & 255); }
    __stcs(out + 3 * g, make_float4(f[0], f[1], f[2], f[3]));
    __stcs(out + 3 * g + 1, make_float4(f[4], f[5], f[6], f[7]));
    __stcs(out + 3 * g + 2, make_float4(f[8], f[9], f[10], f[11]));
  }
}
// 3) coalesced write-only: float4 per thread, contiguous
__global__ void k_write(float4* __restrict__ out, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = make_float4(1.f, 2.f, 3.f, (float)i);
}
// 4) coalesced copy float4
__global__ void k_copy(const float4* __restrict__ in, float4* __restrict__ out, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __ldg(in + i);
}
// 5) 1:4 expand, coalesced: read uint32 (4 B), write float4 (16 B) — same byte ratio as 3:12
__global__ void k_expand(const uint32_t* __restrict__ in, float4* __restrict__ out, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = __ldg(in + i);
    out[i] = make_float4((float)(w & 255), (float)((w >> 8) & 255), (float)((w >> 16) & 255), (float)(w >> 24));
  }
}
__global__ void k_expand_cs(const uint32_t* __restrict__ in, float4* __restrict__ out, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = __ldg(in + i);
    __stcs(out + i, make_float4((float)(w & 255), (float)((w >> 8) & 255), (float)((w >> 16) & 255), (float)(w >> 24)));
  }
}

template <class F>
float timeit(F f, int iters = 10) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f(); cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / iters;
}

int main() {
  const int64_t npx = 1LL << 27;                 // 134M px: 402 MB in, 1.6 GB out
  uint8_t* in; float* out;
  CK(cudaMalloc(&in, npx * 3 + 64)); CK(cudaMalloc(&out, npx * 12 + 64));
  CK(cudaMemset(in, 7, npx * 3)); CK(cudaMemset(out, 0, npx * 12));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t ngrp = npx / 4;
  for (int bpsm : {4, 8, 16, 32}) {
    int grid = sms * bpsm;
    float ms = timeit([&] { k_plain<<<grid, 256>>>((uint32_t*)in, (float4*)out, ngrp); });
    printf("plain     grid=%5d  %.3f ms  %.1f GB/s  %.1f Gpix/s\n", grid, ms, npx * 15 / ms / 1e6, npx / ms / 1e6);
    ms = timeit([&] { k_plain_cs<<<grid, 256>>>((uint32_t*)in, (float4*)out, ngrp); });
    printf("plain_cs  grid=%5d  %.3f ms  %.1f GB/s  %.1f Gpix/s\n", grid, ms, npx * 15 / ms / 1e6, npx / ms / 1e6);
    ms = timeit([&] { k_expand<<<grid, 256>>>((uint32_t*)in, (float4*)out, npx * 3 / 4); });
    printf("expand    grid=%5d  %.3f ms  %.1f GB/s\n", grid, ms, npx * 15 / ms / 1e6);
    ms = timeit([&] { k_expand_cs<<<grid, 256>>>((uint32_t*)in, (float4*)out, npx * 3 / 4); });
    printf("expand_cs grid=%5d  %.3f ms  %.1f GB/s\n", grid, ms, npx * 15 / ms / 1e6);
    ms = timeit([&] { k_write<<<grid, 256>>>((float4*)out, npx * 12 / 16); });
    printf("write     grid=%5d  %.3f ms  %.1f GB/s\n", grid, ms, npx * 12 / ms / 1e6);
    ms = timeit([&] { k_copy<<<grid, 256>>>((float4*)out, (float4*)out + npx * 6 / 16, npx * 6 / 16); });
    printf("copy      grid=%5d  %.3f ms  %.1f GB/s (r+w)\n", grid, ms, npx * 12 / ms / 1e6);
  }
  float ms = timeit([&] { cudaMemsetAsync(out, 0, npx * 12); });
  printf("memset    %.3f ms  %.1f GB/s\n", ms, npx * 12 / ms / 1e6);
  ms = timeit([&] { cudaMemcpyAsync(out + npx * 3 / 2, out, npx * 6, cudaMemcpyDeviceToDevice); });
  printf("memcpy    %.3f ms  %.1f GB/s (r+w)\n", ms, npx * 12 / ms / 1e6);
  return 0;
}
