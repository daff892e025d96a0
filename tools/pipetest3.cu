// Which instruction classes share issue/pipe capacity with fp64 on B200?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N_ITER 2048
struct C8 { double c[8]; };
template <int OP>
__global__ void k(float* out, const __grid_constant__ C8 cc, uint32_t m) {
  double d[8], e[8]; float f[8]; uint32_t u[8];
  for (int i = 0; i < 8; ++i) { d[i] = 1.0 + i + threadIdx.x * 1e-3; e[i] = 0.5 + i; f[i] = i + threadIdx.x; u[i] = threadIdx.x * 13 + i; }
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      d[i] = fma(d[i], e[i], cc.c[i]);                                    // 1 DFMA
      if (OP == 1) f[i] = fmaf(f[i], 1.0001f, 0.5f);                       // + FFMA imm
      if (OP == 2) f[i] = fmaf(f[i], f[(i + 1) & 7], f[(i + 2) & 7]);      // + FFMA reg
      if (OP == 3) asm volatile("shf.l.wrap.b32 %0, %0, %0, 3;" : "+r"(u[i]));            // + SHF
      if (OP == 4) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(u[i]) : "r"(m));     // + IMAD
      if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(u[i]) : "r"(m));           // + IADD
      if (OP == 6) f[i] = f[i] + 1.0001f;                                   // + FADD
      if (OP == 7) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[i])); f[i] = r + 1.0f; }  // + MUFU (+FADD)
      if (OP == 8) asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(u[i]) : "r"(m));  // + LOP3
    }
  }
  double s = 0; float t = 0; uint32_t w = 0;
  for (int i = 0; i < 8; ++i) { s += d[i] + e[i]; t += f[i]; w += u[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s + t + (float)w;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  C8 cc; for (int i = 0; i < 8; ++i) cc.c[i] = 0.999999 - i * 1e-7;
  const char* names[] = {"DFMA alone", "DFMA + FFMA imm", "DFMA + FFMA reg", "DFMA + SHF", "DFMA + IMAD", "DFMA + IADD", "DFMA + FADD", "DFMA + MUFU.RCP+FADD", "DFMA + LOP3"};
  auto run = [&](auto kern, const char* name) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<sms * 8, 256>>>(out, cc, 3u); cudaDeviceSynchronize();
    cudaEventRecord(a); kern<<<sms * 8, 256>>>(out, cc, 3u); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 8 * 256 * N_ITER * 8;
    printf("%-24s %8.3f ms  %6.1f DFMA lanes/clk/SM\n", name, ms, ops / (ms * 1e-3) / sms / 1.965e9);
  };
  run(k<0>, names[0]); run(k<1>, names[1]); run(k<2>, names[2]); run(k<3>, names[3]); run(k<4>, names[4]);
  run(k<5>, names[5]); run(k<6>, names[6]); run(k<7>, names[7]); run(k<8>, names[8]);
  return 0;
}
