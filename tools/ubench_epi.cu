// Developer microbenchmark (not product code): throughput of the ADC
// epilogue instruction sequence alone (register inputs, no TMEM), in
// conversions per clock per SM, for the packed f32x2 and scalar forms.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_epi tools/ubench_epi.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

struct K {
  uint64_t c_lo2, c_hi2, rint2;
  float c_lo, c_hi, maxc, rint;
};

__device__ __forceinline__ void pair2(uint32_t lo0, uint32_t lo1, uint32_t hi0, uint32_t hi1, const K& k, uint64_t w2,
                                      float& p0, float& p1, float& mr) {
  asm("{\n\t.reg .b64 L, H, T, X, Y, TT, RR, PP;\n\t.reg .f32 x0, x1, r0, r1;\n\t"
      "mov.b64 L, {%3, %4};\n\tmov.b64 H, {%5, %6};\n\t"
      "mul.rn.f32x2 T, L, %7;\n\tfma.rn.f32x2 X, H, %8, T;\n\t"
      "mov.b64 {x0, x1}, X;\n\tmin.f32 x0, x0, %9;\n\tmin.f32 x1, x1, %9;\n\tmov.b64 X, {x0, x1};\n\t"
      "add.rn.f32x2 Y, X, %10;\n\tsub.rn.f32x2 TT, Y, %10;\n\tsub.rn.f32x2 RR, X, TT;\n\t"
      "mov.b64 {r0, r1}, RR;\n\tabs.f32 r0, r0;\n\tabs.f32 r1, r1;\n\tmax.f32 r0, r0, r1;\n\tmax.f32 %2, %2, r0;\n\t"
      "mov.b64 PP, {%0, %1};\n\tfma.rn.f32x2 PP, TT, %11, PP;\n\tmov.b64 {%0, %1}, PP;\n\t}"
      : "+f"(p0), "+f"(p1), "+f"(mr)
      : "r"(lo0), "r"(lo1), "r"(hi0), "r"(hi1), "l"(k.c_lo2), "l"(k.c_hi2), "f"(k.maxc), "l"(k.rint2), "l"(w2));
}

__device__ __forceinline__ void one1(uint32_t lo, uint32_t hi, const K& k, float w, float& p, float& mr) {
  const float x = fminf(__fmaf_rn(__uint_as_float(hi), k.c_hi, __fmul_rn(__uint_as_float(lo), k.c_lo)), k.maxc);
  const float t = __fsub_rn(__fadd_rn(x, k.rint), k.rint);
  mr = fmaxf(mr, fabsf(__fsub_rn(x, t)));
  p = __fmaf_rn(t, w, p);
}

template <int MODE>
__global__ void kern(const K k, float w, float* out, uint32_t seed) {
  uint32_t lo[16], hi[16];
  float P[16];
  for (int i = 0; i < 16; ++i) {
    lo[i] = (threadIdx.x * 2654435761u + i * 40503u + seed) & 0x7fffff;
    hi[i] = (threadIdx.x * 97u + i * 13u) & 0xffff;
    P[i] = 0.f;
  }
  const uint64_t w2 = (uint64_t(__float_as_uint(w)) << 32) | __float_as_uint(w);
  float vote = 0.f;
  for (int it = 0; it < ITERS; ++it) {
    float mr = 0.f;
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      if (MODE == 0) pair2(lo[j], lo[j + 1], hi[j], hi[j + 1], k, w2, P[j], P[j + 1], mr);
      else {
        one1(lo[j], hi[j], k, w, P[j], mr);
        one1(lo[j + 1], hi[j + 1], k, w, P[j + 1], mr);
      }
      if (MODE == 2 && j == 6) {  // vote per 8 like the kernels
        if (__any_sync(0xffffffffu, mr > 1e30f)) vote += 1.f;
        mr = 0.f;
      }
    }
    if (__any_sync(0xffffffffu, mr > 1e30f)) vote += 1.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) lo[j] += 1;  // new data each iteration (IADD on ALU)
  }
  float acc = vote;
  for (int i = 0; i < 16; ++i) acc += P[i];
  if (acc == 1234.5f) out[0] = acc;
}

template <int MODE>
void run(const char* name, int warps, const K& k) {
  float* d;
  cudaMalloc(&d, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  kern<MODE><<<sms, 32 * warps>>>(k, 4.0f, d, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE><<<sms, 32 * warps>>>(k, 4.0f, d, 2);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double conv = double(warps) * ITERS * 16;  // warp-conversions per SM
  const double cycles = ms * 1e-3 * 1.965e9;
  printf("%-10s warps/SM=%2d %.3f ms  %.3f warp-conv/clk/SM  (%.2f clk per warp-conv per SMSP)\n", name, warps, ms,
         conv / cycles, 4.0 * cycles / conv);
  cudaFree(d);
}

int main() {
  K k;
  float c_lo = 1.0f / 65536.0f * 0x1p100f, c_hi = 65025.0f / 65536.0f * 0x1p100f;
  k.c_lo = c_lo;
  k.c_hi = c_hi;
  k.maxc = 127.0f / 1024;
  k.rint = 1.5f * 8192;
  auto pk = [](float v) {
    uint32_t u = *reinterpret_cast<uint32_t*>(&v);
    return (uint64_t(u) << 32) | u;
  };
  k.c_lo2 = pk(k.c_lo);
  k.c_hi2 = pk(k.c_hi);
  k.rint2 = pk(k.rint);
  for (int w : {4, 8, 16, 32}) {
    run<0>("f32x2", w, k);
    run<1>("scalar", w, k);
    run<2>("scalar+v8", w, k);
  }
  return 0;
}
