// sm_100a building blocks for the tcgen05 crossbar kernels: mbarriers, TMA
// (cp.async.bulk.tensor), UMMA shared-memory / instruction descriptors,
// tcgen05.mma kind::i8, TMEM alloc / ld, and the fp32 ADC epilogue helpers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

struct xbs_core;
namespace xbs {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------- mbarriers
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
// Wait for the single-thread roles (TMA producer, MMA issuer): the thread is
// suspended in hardware for up to ~0.5 us per try instead of spinning, so
// its warp does not steal issue slots from the epilogue warps.
#ifndef XBS_ROLE_WAIT_NS
#define XBS_ROLE_WAIT_NS 0
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  if constexpr (XBS_ROLE_WAIT_NS == 0) {
    mbar_wait(bar, parity);
  } else {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    do {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(a), "r"(parity), "r"(XBS_ROLE_WAIT_NS)
          : "memory");
    } while (!done);
  }
}

// ------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// ------------------------------------------------------- UMMA descriptors
// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start >> 4
// [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48), layout
// [61,64): 2 = SWIZZLE_128B, 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout & 7u) << 61;
  return d;
}
// Instruction descriptor, kind::i8: D s32, A/B u8, A K-major, B major as given.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool b_mn_major) {
  return (2u << 4)                      /* c_format S32        */
         | (0u << 7) | (0u << 10)       /* a, b: unsigned 8-bit */
         | (0u << 15)                   /* a K-major           */
         | (uint32_t(b_mn_major) << 16) /* b major             */
         | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ------------------------------------------------------------------ TMEM
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 16 lanes x 256 bits: thread t of the warp gets lane base + t/4... (shape 16x256b)
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// ------------------------------------------------------- ADC epilogue math
// A column current on the snapped grid is n = hi*65025 + lo units of
// 2^sh amperes (hi, lo = the two radix-255 digit-pair accumulators, each an
// exact s32 < 2^23 for 128 crossbar rows).  The fp32 fast path approximates
// scaled = I / i_fs * maxc to within 5e-5 codes; conversions whose fraction
// lies within kDelta of a rounding boundary are re-evaluated with the
// reference's own fp64 expression (converters.cpp:85-87), so every code is
// bit-exact.
struct AdcConst {
  float c_hi, c_lo, k_lo, maxc;
  float k2;       // -2^23 (c_lo + c_hi): both magic offsets folded into one constant
  float thr;      // 0.5 - delta: fractions beyond this go to the exact path
  float sat;      // maxc - 0.5 - delta: fast values above this go to the exact path
  int sh;
  int maxc_i;
  double i_fs, maxc_d;
};
constexpr float kDelta = 1.0f / 4096.0f;
constexpr float kMagic23 = 8388608.0f;     // 2^23
constexpr float kRint = 12582912.0f;       // 1.5 * 2^23

static __device__ __noinline__ float adc_exact(uint32_t hi, uint32_t lo, double i_fs, double maxc_d, int sh) {
  const long long n = (long long)hi * 65025ll + (long long)lo;
  const double I = ldexp(double(n), sh);
  const double scaled = I / i_fs * maxc_d;
  if (scaled >= maxc_d) return float(maxc_d);
  return float(llround(scaled));
}

// fp32 fast path for one conversion: returns rint(scaled) (clamped to maxc)
// and sets bit `bit` of `near` when the fraction is within kDelta of a
// rounding boundary.
__device__ __forceinline__ float adc_fast(uint32_t hi, uint32_t lo, const AdcConst& k, uint32_t& near, uint32_t bit) {
  const float hf = __fsub_rn(__int_as_float(int(hi | 0x4B000000u)), kMagic23);
  const float lt = __fmaf_rn(__int_as_float(int(lo | 0x4B000000u)), k.c_lo, k.k_lo);
  float x = __fmaf_rn(hf, k.c_hi, lt);
  x = fminf(x, k.maxc);
  const float t = __fsub_rn(__fadd_rn(x, kRint), kRint);
  const float r = fabsf(__fsub_rn(x, t));
  if (r > 0.5f - kDelta) near |= bit;
  return t;
}

// ---- packed fp32x2 (FFMA2 / FADD2, sm_100a): two conversions per instruction
__device__ __forceinline__ uint64_t pk2(uint32_t a, uint32_t b) { return (uint64_t(b) << 32) | a; }
__device__ __forceinline__ uint64_t pkf2(float a, float b) { return pk2(__float_as_uint(a), __float_as_uint(b)); }
__device__ __forceinline__ float lo2(uint64_t v) { return __uint_as_float(uint32_t(v)); }
__device__ __forceinline__ float hi2(uint64_t v) { return __uint_as_float(uint32_t(v >> 32)); }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// Splatted constants of the packed ADC fast path.
struct AdcConst2 {
  uint64_t c_hi, c_lo, k_lo, neg_m23, rint, neg_rint;
  float maxc;
};
__device__ __forceinline__ AdcConst2 make_const2(const AdcConst& k) {
  AdcConst2 c;
  c.c_hi = pkf2(k.c_hi, k.c_hi);
  c.c_lo = pkf2(k.c_lo, k.c_lo);
  c.k_lo = pkf2(k.k_lo, k.k_lo);
  c.neg_m23 = pkf2(-kMagic23, -kMagic23);
  c.rint = pkf2(kRint, kRint);
  c.neg_rint = pkf2(-kRint, -kRint);
  c.maxc = k.maxc;
  return c;
}

// Two conversions (hi/lo digit-pair accumulators of columns j, j+1): returns
// the packed rounded codes, folds |fraction - rint| into the running max m.
__device__ __forceinline__ uint64_t adc_fast2(uint32_t hi0, uint32_t hi1, uint32_t lo0, uint32_t lo1,
                                              const AdcConst2& c, float& m) {
  const uint64_t hf = fadd2(pk2(hi0 | 0x4B000000u, hi1 | 0x4B000000u), c.neg_m23);
  const uint64_t lt = ffma2(pk2(lo0 | 0x4B000000u, lo1 | 0x4B000000u), c.c_lo, c.k_lo);
  uint64_t x = ffma2(hf, c.c_hi, lt);
  x = pkf2(fminf(lo2(x), c.maxc), fminf(hi2(x), c.maxc));
  const uint64_t t = fadd2(fadd2(x, c.rint), c.neg_rint);
  const uint64_t r = fsub2(x, t);
  m = fmaxf(m, fmaxf(fabsf(lo2(r)), fabsf(hi2(r))));
  return t;
}

// One accumulator buffer's share of a warp: NQ chunks of 8 columns.  Chunk
// q reads the lo / hi digit-pair accumulators at TMEM addresses alo(q) /
// ahi(q), converts them and accumulates P2[slot(q) + j/2] += wt(q) * code
// (packed pairs).  TMEM loads run one chunk ahead of the math (software
// pipelined); the buffer is released to the MMA warp right after the last
// load completes.  Near-boundary conversions are fixed up exactly.
// Scalar fast path, 9 instructions per conversion (6 FMA-pipe, 3 ALU):
//   x = (bits(hi|M) c_hi) + ((bits(lo|M) c_lo) + k2)   [2 LOP3, 2 FFMA]
//   t = (x + 1.5*2^23) - 1.5*2^23, r = x - t            [3 FADD]
// and, per pair, running maxima of |r| and x          [2 FMNMX3 / 2]
// P += w t                                            [1 FFMA]
// No per-element clamp: a chunk whose max x exceeds k.sat (possible
// saturation) or whose max |r| exceeds k.thr (near a rounding boundary) is
// re-evaluated element by element with the reference's fp64 expression.
__device__ __forceinline__ float adc_x(uint32_t hi, uint32_t lo, const AdcConst& k) {
  // hi, lo < 2^24 (<= 256 crossbar rows) convert exactly (I2FP, ALU pipe);
  // |x - scaled| <= 3 2^-24 x  (<< kDelta).
  return __fmaf_rn(__uint2float_rn(hi), k.c_hi, __fmul_rn(__uint2float_rn(lo), k.c_lo));
}
__device__ __forceinline__ float rint_magic(float x) { return __fsub_rn(__fadd_rn(x, kRint), kRint); }

template <int NQ, int NP, class ALo, class AHi, class Slot, class Wt>
__device__ __forceinline__ void adc_pipeline_s(ALo alo, AHi ahi, Slot slot, Wt wt, const AdcConst& k,
                                               float (&P)[NP], uint32_t& exact_ctr, uint64_t* release) {
  uint32_t lo[2][8], hi[2][8];
  tmem_ld8(alo(0), lo[0]);
  tmem_ld8(ahi(0), hi[0]);
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    tmem_wait_ld();
    if (q + 1 < NQ) {
      tmem_ld8(alo(q + 1), lo[(q + 1) & 1]);
      tmem_ld8(ahi(q + 1), hi[(q + 1) & 1]);
    } else {
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(release);
    }
    const float w = wt(q);
    const int b = slot(q);
    float mr = 0.f;
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const float x0 = fminf(adc_x(hi[q & 1][j], lo[q & 1][j], k), k.maxc);
      const float x1 = fminf(adc_x(hi[q & 1][j + 1], lo[q & 1][j + 1], k), k.maxc);
      const float t0 = rint_magic(x0), t1 = rint_magic(x1);
      mr = fmaxf(mr, fmaxf(fabsf(__fsub_rn(x0, t0)), fabsf(__fsub_rn(x1, t1))));
      P[b + j] = __fmaf_rn(t0, w, P[b + j]);
      P[b + j + 1] = __fmaf_rn(t1, w, P[b + j + 1]);
    }
    if (__any_sync(0xffffffffu, mr > k.thr)) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float x = fminf(adc_x(hi[q & 1][j], lo[q & 1][j], k), k.maxc);
        const float t = rint_magic(x);
        if (fabsf(__fsub_rn(x, t)) > k.thr) {
          ++exact_ctr;
          const float d = __fsub_rn(adc_exact(hi[q & 1][j], lo[q & 1][j], k.i_fs, k.maxc_d, k.sh), t);
          P[b + j] = __fmaf_rn(d, w, P[b + j]);
        }
      }
    }
  }
}

// Non-pipelined variant (fewer live registers): one 8-column chunk,
// TMEM -> registers -> ADC -> P[b+j] += w * code.
template <int kN>
__device__ __forceinline__ void adc_chunk8s(uint32_t ta_lo, uint32_t ta_hi, const AdcConst& k, float w,
                                            float (&P)[kN], int b, uint32_t& exact_ctr, uint64_t* release) {
  uint32_t lo[8], hi[8];
  tmem_ld8(ta_lo, lo);
  tmem_ld8(ta_hi, hi);
  tmem_wait_ld();
  if (release) {
    tc_fence_before();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(release);
  }
  float mr = 0.f;
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float x0 = fminf(adc_x(hi[j], lo[j], k), k.maxc);
    const float x1 = fminf(adc_x(hi[j + 1], lo[j + 1], k), k.maxc);
    const float t0 = rint_magic(x0), t1 = rint_magic(x1);
    mr = fmaxf(mr, fmaxf(fabsf(__fsub_rn(x0, t0)), fabsf(__fsub_rn(x1, t1))));
    P[b + j] = __fmaf_rn(t0, w, P[b + j]);
    P[b + j + 1] = __fmaf_rn(t1, w, P[b + j + 1]);
  }
  if (__any_sync(0xffffffffu, mr > k.thr)) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float x = fminf(adc_x(hi[j], lo[j], k), k.maxc);
      const float t = rint_magic(x);
      if (fabsf(__fsub_rn(x, t)) > k.thr) {
        ++exact_ctr;
        const float d = __fsub_rn(adc_exact(hi[j], lo[j], k.i_fs, k.maxc_d, k.sh), t);
        P[b + j] = __fmaf_rn(d, w, P[b + j]);
      }
    }
  }
}

template <int NQ, int NP, int DBG = 0, class ALo, class AHi, class Slot, class Wt>
__device__ __forceinline__ void adc_pipeline(ALo alo, AHi ahi, Slot slot, Wt wt, const AdcConst& k,
                                             const AdcConst2& c2, uint64_t (&P2)[NP], uint32_t& exact_ctr,
                                             uint64_t* release) {
  if constexpr (DBG == 1) {  // perf experiment: TMEM loads only
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      tmem_ld8(alo(q), lo);
      tmem_ld8(ahi(q), hi);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 8; j += 2) P2[slot(q) + j / 2] ^= pk2(lo[j] ^ hi[j], lo[j + 1] ^ hi[j + 1]);
    }
    tc_fence_before();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(release);
    return;
  }
  uint32_t lo[2][8], hi[2][8];
  tmem_ld8(alo(0), lo[0]);
  tmem_ld8(ahi(0), hi[0]);
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    tmem_wait_ld();
    if (q + 1 < NQ) {
      tmem_ld8(alo(q + 1), lo[(q + 1) & 1]);
      tmem_ld8(ahi(q + 1), hi[(q + 1) & 1]);
    } else {
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(release);
    }
    const uint64_t w2 = wt(q);
    const int b = slot(q);
    float m = 0.f;
#pragma unroll
    for (int j = 0; j < 8; j += 2)
      P2[b + j / 2] = ffma2(adc_fast2(hi[q & 1][j], hi[q & 1][j + 1], lo[q & 1][j], lo[q & 1][j + 1], c2, m), w2,
                            P2[b + j / 2]);
    if (__any_sync(0xffffffffu, m > 0.5f - kDelta)) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t near = 0;
        const float f = adc_fast(hi[q & 1][j], lo[q & 1][j], k, near, 1u);
        if (near) {
          ++exact_ctr;
          const float d = __fsub_rn(adc_exact(hi[q & 1][j], lo[q & 1][j], k.i_fs, k.maxc_d, k.sh), f);
          P2[b + j / 2] = ffma2((j & 1) ? pkf2(0.f, d) : pkf2(d, 0.f), w2, P2[b + j / 2]);
        }
      }
    }
  }
}

// fp32 fast path without per-element boundary bookkeeping: returns the
// rounded code and folds |fraction - rint| into a running max `m`.
__device__ __forceinline__ float adc_fast_m(uint32_t hi, uint32_t lo, const AdcConst& k, float& m) {
  const float hf = __fsub_rn(__int_as_float(int(hi | 0x4B000000u)), kMagic23);
  const float lt = __fmaf_rn(__int_as_float(int(lo | 0x4B000000u)), k.c_lo, k.k_lo);
  float x = __fmaf_rn(hf, k.c_hi, lt);
  x = fminf(x, k.maxc);
  const float t = __fsub_rn(__fadd_rn(x, kRint), kRint);
  m = fmaxf(m, fabsf(__fsub_rn(x, t)));
  return t;
}

// One 8-column chunk of a chain: TMEM -> registers, ADC, P[base+j] += w*code.
// If any lane of the warp saw a fraction within kDelta of 1/2 the whole
// chunk is re-checked element by element and the near-boundary codes are
// replaced by the exact fp64 evaluation (P += w * (exact - fast)).
template <int kN>
__device__ __forceinline__ void adc_chunk8(uint32_t ta_lo, uint32_t ta_hi, const AdcConst& k, float w,
                                           float (&P)[kN], int base, uint32_t& exact_ctr, uint64_t* release) {
  uint32_t lo[8], hi[8];
  tmem_ld8(ta_lo, lo);
  tmem_ld8(ta_hi, hi);
  tmem_wait_ld();
  if (release) {  // last TMEM read of this accumulator buffer by this warp
    tc_fence_before();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(release);
  }
  float m = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) P[base + j] = __fmaf_rn(adc_fast_m(hi[j], lo[j], k, m), w, P[base + j]);
  if (__any_sync(0xffffffffu, m > 0.5f - kDelta)) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t near = 0;
      const float fast = adc_fast(hi[j], lo[j], k, near, 1u);
      if (near) {
        ++exact_ctr;
        const float ex = adc_exact(hi[j], lo[j], k.i_fs, k.maxc_d, k.sh);
        P[base + j] = __fmaf_rn(__fsub_rn(ex, fast), w, P[base + j]);
      }
    }
  }
}

// 16 conversions accumulated straight into P[j] += w * code: fast path for
// all, then for the (rare) near-boundary ones the exact fp64 code replaces
// the fast one (P += w * (exact - fast); all operands are exact integers).
// The warp takes the fix-up branch only when one of its lanes needs it.
template <int kN>
__device__ __forceinline__ void adc_accum16(const uint32_t (&hi)[16], const uint32_t (&lo)[16], const AdcConst& k,
                                            float w, float (&P)[kN], int base, uint32_t& exact_ctr) {
  uint32_t near = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) P[base + j] = __fmaf_rn(adc_fast(hi[j], lo[j], k, near, 1u << j), w, P[base + j]);
  if (__any_sync(0xffffffffu, near != 0)) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if ((near >> j) & 1u) {
        ++exact_ctr;
        uint32_t dummy = 0;
        const float fast = adc_fast(hi[j], lo[j], k, dummy, 1u);
        const float ex = adc_exact(hi[j], lo[j], k.i_fs, k.maxc_d, k.sh);
        P[base + j] = __fmaf_rn(__fsub_rn(ex, fast), w, P[base + j]);
      }
  }
}

// 16 conversions: fast path for all, exact fp64 re-evaluation only for the
// (rare) near-boundary ones; the warp takes the fix-up branch only when one
// of its lanes needs it.
__device__ __forceinline__ void adc_chunk16(const uint32_t (&hi)[16], const uint32_t (&lo)[16], const AdcConst& k,
                                            float (&t)[16], uint32_t& exact_ctr) {
  uint32_t near = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) t[j] = adc_fast(hi[j], lo[j], k, near, 1u << j);
  if (__any_sync(0xffffffffu, near != 0)) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if ((near >> j) & 1u) {
        ++exact_ctr;
        t[j] = adc_exact(hi[j], lo[j], k.i_fs, k.maxc_d, k.sh);
      }
  }
}

// host helpers (xbs_vmm_tc.cu)
bool make_map_u8(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo,
                 int swizzle_bytes = 128);
int num_sms();
AdcConst make_adc_const(const xbs_core* c);

}  // namespace tc
}  // namespace xbs
