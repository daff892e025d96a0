// fp64 pipe throughput by operand form (B200)
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 2048
struct C8 { double c[8]; };
template <int OP>
__global__ void k(float* out, const __grid_constant__ C8 cc) {
  double d[8], e[8];
  for (int i = 0; i < 8; ++i) { d[i] = 1.0 + i + threadIdx.x * 1e-3; e[i] = 0.5 + i; }
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) d[i] = fma(d[i], cc.c[i], cc.c[(i + 1) & 7]);      // reg * const + const
      if (OP == 1) d[i] = fma(d[i], e[i], cc.c[i]);                    // reg * reg + const
      if (OP == 2) d[i] = fma(d[i], e[i], e[(i + 3) & 7]);            // 3 regs
      if (OP == 3) d[i] = d[i] + cc.c[i];                              // DADD reg + const
      if (OP == 4) d[i] = d[i] * e[i];                                 // DMUL reg * reg
      if (OP == 5) { d[i] = fma(d[i], e[i], cc.c[i]); e[i] = e[i] * 1.0000001f; }  // DFMA + FMUL mix
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += d[i] + e[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  C8 cc; for (int i = 0; i < 8; ++i) cc.c[i] = 0.999999 - i * 1e-7;
  const char* names[] = {"DFMA r*c+c", "DFMA r*r+c", "DFMA r*r+r", "DADD r+c", "DMUL r*r", "DFMA r*r+c + FMUL"};
  auto run = [&](auto kern, const char* name) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<sms * 8, 256>>>(out, cc); cudaDeviceSynchronize();
    cudaEventRecord(a); kern<<<sms * 8, 256>>>(out, cc); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 8 * 256 * N_ITER * 8;
    printf("%-22s %8.3f ms  %6.1f fp64 lane-ops/clk/SM @1965MHz\n", name, ms, ops / (ms * 1e-3) / sms / 1.965e9);
  };
  run(k<0>, names[0]); run(k<1>, names[1]); run(k<2>, names[2]); run(k<3>, names[3]); run(k<4>, names[4]); run(k<5>, names[5]);
  return 0;
}
