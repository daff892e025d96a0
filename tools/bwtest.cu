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

// 6) the same expand with the input wrapped onto a 32 MB window (L2-resident after the first pass): DRAM sees
//    writes only, the SMs still issue every load -- separates the DRAM read/write mix from SM-side limits
__global__ void k_expand_l2(const uint32_t* __restrict__ in, float4* __restrict__ out, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = __ldg(in + (i & ((8LL << 20) - 1)));
    out[i] = make_float4((float)(w & 255), (float)((w >> 8) & 255), (float)((w >> 16) & 255), (float)(w >> 24));
  }
}
// 7) read-only: sum of uint4 (checks the pure read rate)
__global__ void k_read(const uint4* __restrict__ in, uint32_t* __restrict__ sink, int64_t nv) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(in + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}
// 8) mixes r : w = 1 : k by bytes, coalesced float4 both ways (k = 1 is the copy, k = 4 the expand ratio)
template <int K>
__global__ void k_mix(const float4* __restrict__ in, float4* __restrict__ out, int64_t nv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(in + i);
#pragma unroll
    for (int k = 0; k < K; ++k) out[(int64_t)k * nv + i] = make_float4(v.x + k, v.y, v.z, v.w);
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
  {
    const int grid = sms * 16;
    float ms = timeit([&] { k_expand_l2<<<grid, 256>>>((uint32_t*)in, (float4*)out, npx * 3 / 4); });
    printf("expand_l2 (input L2-resident)  %.3f ms  %.1f GB/s algorithmic, %.1f GB/s of writes\n", ms,
           npx * 15 / ms / 1e6, npx * 12 / ms / 1e6);
    uint32_t* sink; CK(cudaMalloc(&sink, 4));
    ms = timeit([&] { k_read<<<grid, 256>>>((uint4*)out, sink, npx * 12 / 16); });
    printf("read      %.3f ms  %.1f GB/s\n", ms, npx * 12 / ms / 1e6);
    const int64_t nv = npx * 12 / 16 / 5;    // in: nv float4, out: K nv float4, inside the 1.6 GB buffer
    ms = timeit([&] { k_mix<1><<<grid, 256>>>((float4*)out, (float4*)out + nv, nv); });
    printf("mix 1:1   %.3f ms  %.1f GB/s (r+w)\n", ms, nv * 16.0 * 2 / ms / 1e6);
    ms = timeit([&] { k_mix<2><<<grid, 256>>>((float4*)out, (float4*)out + nv, nv); });
    printf("mix 1:2   %.3f ms  %.1f GB/s (r+w)\n", ms, nv * 16.0 * 3 / ms / 1e6);
    ms = timeit([&] { k_mix<4><<<grid, 256>>>((float4*)out, (float4*)out + nv, nv); });
    printf("mix 1:4   %.3f ms  %.1f GB/s (r+w)\n", ms, nv * 16.0 * 5 / ms / 1e6);
  }
  float ms = timeit([&] { cudaMemsetAsync(out, 0, npx * 12); });
  printf("memset    %.3f ms  %.1f GB/s\n", ms, npx * 12 / ms / 1e6);
  ms = timeit([&] { cudaMemcpyAsync(out + npx * 3 / 2, out, npx * 6, cudaMemcpyDeviceToDevice); });
  printf("memcpy    %.3f ms  %.1f GB/s (r+w)\n", ms, npx * 12 / ms / 1e6);
  return 0;
}
