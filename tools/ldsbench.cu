// Random shared-memory gather cost per warp instruction for 4/8/16-byte
// loads (sizes the LUT lattice node format).  Prints cycles per warp-load
// per SM (== wavefronts when smem-bound).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int W>
__global__ void k(float* out, int iters, int entries) {
  extern __shared__ __align__(16) unsigned char sm[];
  for (int i = threadIdx.x; i < entries * W / 4; i += blockDim.x) ((float*)sm)[i] = (float)i;
  __syncthreads();
  uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      const uint32_t idx = (s >> 8) & (entries - 1);
      if (W == 4) acc += ((const float*)sm)[idx];
      else if (W == 8) { float2 v = ((const float2*)sm)[idx]; acc += v.x + v.y; }
      else { float4 v = ((const float4*)sm)[idx]; acc += v.x + v.y + v.z + v.w; }
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

template <int W>
void run(int bytes, int threads, int bps) {
  int entries = bytes / W;
  float* o; cudaMalloc(&o, 4);
  cudaFuncSetAttribute(k<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  int iters = 2048;
  dim3 grid(148 * bps);
  k<W><<<grid, threads, bytes>>>(o, 16, entries);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<W><<<grid, threads, bytes>>>(o, iters, entries);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cycles = ms * 1e-3 * clk * 1e3;
  double warp_loads_per_sm = (double)bps * threads / 32 * iters * 8;
  printf("W=%2d table=%6d B threads=%d x %d/SM: %.2f cyc per warp-load/SM  (%s)\n", W, bytes, threads, bps,
         cycles / warp_loads_per_sm, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}

int main() {
  for (int bytes : {65536, 131072}) {
    run<4>(bytes, 512, 2);
    run<8>(bytes, 512, 2);
    run<16>(bytes, 512, 2);
  }
  return 0;
}
