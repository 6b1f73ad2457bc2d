// Developer microbenchmark (not product code): issue throughput of the
// instruction forms the ADC epilogue uses, on one B200.  Each thread runs
// 8 independent dependency chains; reports warp-instructions / clock / SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2i(uint64_t a) {
  uint64_t d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(0x3f8000003f800000ull));
  return d;
}

template <int OP>
__global__ void k(float* out, float s0, float s1) {
  float v[8];
  uint64_t w[8];
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) {
    v[i] = threadIdx.x * 0.001f + i;
    w[i] = (uint64_t(__float_as_uint(v[i])) << 32) | __float_as_uint(v[i] + 1);
    u[i] = threadIdx.x + i;
  }
  const uint64_t s2 = (uint64_t(__float_as_uint(s0)) << 32) | __float_as_uint(s1);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) v[i] = __fmaf_rn(v[i], s0, s1);            // FFMA reg
      if (OP == 1) v[i] = __fadd_rn(v[i], 12582912.f);        // FADD imm
      if (OP == 2) w[i] = ffma2(w[i], s2, s2);                 // FFMA2
      if (OP == 3) w[i] = fadd2i(w[i]);                        // FADD2 imm
      if (OP == 4) u[i] = (u[i] | 0x4B000000u) ^ (u[i] >> 3);  // LOP3-ish ALU
      if (OP == 5) v[i] = fminf(v[i], s0);                     // FMNMX
      if (OP == 6) v[i] = __fmaf_rn(v[i], 1.0001f, 0.5f);      // FFMA imm
    }
  }
  float acc = 0;
  for (int i = 0; i < 8; ++i) acc += v[i] + __uint_as_float(uint32_t(w[i])) + __uint_as_float(u[i]);
  if (acc == 12345.f) out[0] = acc;
}

template <int OP>
void run(const char* name, int warps) {
  float* d;
  cudaMalloc(&d, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  k<OP><<<sms, 32 * warps>>>(d, 1.0001f, 0.5f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<sms, 32 * warps>>>(d, 1.0001f, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double instr = double(sms) * warps * ITERS * 8;  // warp instructions
  const double cycles = ms * 1e-3 * 1.965e9;               // assume max clock
  printf("%-12s warps/SM=%2d  %.3f ms  %.2f warp-instr/clk/SM\n", name, warps, ms, instr / sms / cycles);
  cudaFree(d);
}

int main_pipes() {
  for (int w : {8, 16, 32}) {
    run<0>("FFMA reg", w);
    run<6>("FFMA imm", w);
    run<1>("FADD imm", w);
    run<2>("FFMA2", w);
    run<3>("FADD2 imm", w);
    run<4>("ALU LOP/SHF", w);
    run<5>("FMNMX", w);
  }
  return 0;
}
// (appended) I2F throughput probe
__global__ void k_i2f(float* out, int s0) {
  int u[8]; float v[8];
  for (int i = 0; i < 8; ++i) { u[i] = threadIdx.x * 7 + i; v[i] = 0.f; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { v[i] += __int2float_rn(u[i]); u[i] += s0; }
  }
  float acc = 0; for (int i = 0; i < 8; ++i) acc += v[i];
  if (acc == 12345.f) out[0] = acc;
}
int main2() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {16, 32}) {
    k_i2f<<<sms, 32 * warps>>>(d, 3);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k_i2f<<<sms, 32 * warps>>>(d, 3); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double instr = double(warps) * ITERS * 8;  // I2F per SM (plus same count of FADD and IADD)
    printf("I2F(+FADD+IADD) warps/SM=%d %.3f ms  %.2f I2F/clk/SM\n", warps, ms, instr / (ms * 1e-3 * 1.965e9));
  }
  return 0;
}
int main() { main_pipes(); return main2(); }
