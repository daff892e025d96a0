// opbench.cu — issue-rate probe of the integer instructions the LUT kernels are made of (B200).
// Each kernel runs a long unrolled chain of ONE instruction kind on 8 independent registers per thread,
// 1024 threads per SM; prints warp-instructions per clock per SM (peak issue is 4).
// Standalone; build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/opbench tools/opbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define REP 64
template <int OP>
__global__ void k_op(uint32_t* out, uint32_t a0, uint32_t b0, int iters) {
  uint32_t r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = a0 + threadIdx.x * (i + 1);
  uint32_t b = b0 + threadIdx.x, c = b0 * 3 + 1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < REP / 8; ++k) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));          // IMAD
        if (OP == 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));          // IMAD.HI
        if (OP == 2) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(b), "r"(c));      // LOP3
        if (OP == 3) asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));      // SHF
        if (OP == 4) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));            // PRMT
        if (OP == 5) asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(b), "r"(c));        // IDP4A
        if (OP == 6) asm volatile("popc.b32 %0, %0;" : "+r"(r[i]));                                      // POPC
        if (OP == 7) asm volatile("max.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(b));                         // VIMNMX
        if (OP == 8) asm volatile("{.reg .f32 f; cvt.rn.f32.u32 f, %0; mov.b32 %0, f;}" : "+r"(r[i]));  // I2F
        if (OP == 9) asm volatile("add.u32 %0, %0, %1;" : "+r"(r[i]) : "r"(b));                         // IADD
        if (OP == 10) asm volatile("{.reg .f32 f, g; mov.b32 f, %0; mov.b32 g, %1; fma.rn.f32 f, f, g, g; mov.b32 %0, f;}" : "+r"(r[i]) : "r"(b));  // FFMA
        if (OP == 11) asm volatile("shl.b32 %0, %0, 3;" : "+r"(r[i]));                                   // SHL imm
        if (OP == 12) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; selp.u32 %0, %1, %2, p;}" : "+r"(r[i]) : "r"(b), "r"(c));  // ISETP+SEL
        // pairs on alternating registers: the rate says whether the two kinds share a pipe (2 / clk / SM) or not (4)
#define LOP3_ "lop3.b32 %0, %0, %1, %2, 0x96;"
#define IMAD_ "mad.lo.u32 %0, %0, %1, %2;"
#define DP4A_ "dp4a.u32.u32 %0, %0, %1, %2;"
#define PRMT_ "prmt.b32 %0, %0, %1, %2;"
#define SHF_ "shf.r.wrap.b32 %0, %0, %1, %2;"
#define I2F_ "{.reg .f32 f; cvt.rn.f32.u32 f, %0; mov.b32 %0, f;}"
#define FFMA_ "{.reg .f32 f, g; mov.b32 f, %0; mov.b32 g, %1; fma.rn.f32 f, f, g, g; mov.b32 %0, f;}"
#define LEA_ "{.reg .u32 t; shl.b32 t, %0, 5; add.u32 %0, t, %1;}"
#define MNMX_ "{.reg .u32 t; max.u32 t, %0, %1; min.u32 %0, t, %2;}"
#define PAIR(A, B) if (i & 1) asm volatile(A : "+r"(r[i]) : "r"(b), "r"(c)); else asm volatile(B : "+r"(r[i]) : "r"(b), "r"(c));
        if (OP == 20) { PAIR(LOP3_, IMAD_) }
        if (OP == 21) { PAIR(LOP3_, DP4A_) }
        if (OP == 22) { PAIR(IMAD_, DP4A_) }
        if (OP == 23) { PAIR(LOP3_, PRMT_) }
        if (OP == 24) { PAIR(LOP3_, I2F_) }
        if (OP == 25) { PAIR(LOP3_, FFMA_) }
        if (OP == 26) { PAIR(IMAD_, FFMA_) }
        if (OP == 27) { PAIR(LOP3_, SHF_) }
        if (OP == 28) asm volatile(LEA_ : "+r"(r[i]) : "r"(b), "r"(c));
        if (OP == 29) asm volatile(MNMX_ : "+r"(r[i]) : "r"(b), "r"(c));
        if (OP == 30) { PAIR(IMAD_, I2F_) }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= r[i];
  if (s == 0x12345u) out[0] = s;
}

template <int OP>
void run(const char* name, uint32_t* out, int sms) {
  const int iters = 2000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_op<OP><<<sms, 1024>>>(out, 7, 13, iters);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  k_op<OP><<<sms, 1024>>>(out, 7, 13, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double winst = (double)iters * REP * 32 * (OP == 12 || OP == 29 ? 2 : 1);   // warp-instructions per SM
  printf("%-10s %.3f ms  %.2f warp-inst/clk/SM (at the %d MHz max clock)\n", name, ms, winst / (ms * 1e-3 * khz * 1e3), khz / 1000);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 64);
  run<0>("IMAD", out, sms); run<1>("IMAD.HI", out, sms); run<2>("LOP3", out, sms); run<3>("SHF", out, sms);
  run<4>("PRMT", out, sms); run<5>("IDP4A", out, sms); run<6>("POPC", out, sms); run<7>("VIMNMX", out, sms);
  run<8>("I2F", out, sms); run<9>("IADD", out, sms); run<10>("FFMA", out, sms); run<11>("SHL", out, sms);
  run<12>("ISETP+SEL", out, sms);
  run<20>("LOP3|IMAD", out, sms); run<21>("LOP3|DP4A", out, sms); run<22>("IMAD|DP4A", out, sms);
  run<23>("LOP3|PRMT", out, sms); run<24>("LOP3|I2F", out, sms); run<25>("LOP3|FFMA", out, sms);
  run<26>("IMAD|FFMA", out, sms); run<27>("LOP3|SHF", out, sms); run<28>("LEA", out, sms); run<29>("MAX;MIN", out, sms);
  run<30>("IMAD|I2F", out, sms);
  return 0;
}
