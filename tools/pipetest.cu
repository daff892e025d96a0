// pipetest.cu — per-SM instruction throughput of the ops the CIELAB kernel uses (B200).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N_ITER 4096
template <int OP>
__global__ void k(float* out, float seed) {
  double d[8]; float f[8]; uint32_t u[8];
  for (int i = 0; i < 8; ++i) { d[i] = seed + i + threadIdx.x; f[i] = seed * i + threadIdx.x; u[i] = threadIdx.x * 7 + i; }
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) d[i] = fma(d[i], 1.0000001, 0.5);                 // DFMA
      if (OP == 1) f[i] = fmaf(f[i], 1.0000001f, 0.5f);              // FFMA imm
      if (OP == 2) f[i] = fmaf(f[i], f[(i + 1) & 7], f[(i + 2) & 7]);  // FFMA reg
      if (OP == 3) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[i])); f[i] = r; }
      if (OP == 4) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d[i])); d[i] = r; }
      if (OP == 5) { d[i] = (double)f[i]; f[i] = (float)d[i] + 1.0f; }  // F2F both ways (+FADD)
      if (OP == 6) u[i] = (u[i] >> 3) + 0x38000000u + u[(i + 1) & 7];  // ALU
      if (OP == 7) d[i] = d[i] * 1.0000001;                              // DMUL
      if (OP == 8) d[i] = d[i] + 0.5;                                    // DADD
    }
  }
  double s = 0; float t = 0; uint32_t w = 0;
  for (int i = 0; i < 8; ++i) { s += d[i]; t += f[i]; w += u[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s + t + (float)w;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"DFMA", "FFMA imm", "FFMA reg", "MUFU.RCP f32", "MUFU.RCP64H", "F2F f32->f64->f32 (+FADD)", "ALU shift/add", "DMUL", "DADD"};
  auto run = [&](auto kern, const char* name) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<sms * 8, 256>>>(out, 1.0f); cudaDeviceSynchronize();
    cudaEventRecord(a); kern<<<sms * 8, 256>>>(out, 1.0f); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 8 * 256 * N_ITER * 8;
    printf("%-28s %8.3f ms  %7.1f lane-ops/clk/SM (at %.0f MHz nominal)\n", name, ms, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
  };
  run(k<0>, names[0]); run(k<1>, names[1]); run(k<2>, names[2]); run(k<3>, names[3]); run(k<4>, names[4]);
  run(k<5>, names[5]); run(k<6>, names[6]); run(k<7>, names[7]); run(k<8>, names[8]);
  return 0;
}
