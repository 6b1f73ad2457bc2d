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
// Wait with a suspend-time hint: the thread sleeps in hardware until the
// phase completes (or the hint expires) instead of spinning on try_wait, so
// a waiting warp does not take issue slots from the warps that have work.
__device__ __forceinline__ void mbar_wait_hint(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(0x100000)
        : "memory");
  } while (!done);
}
// Non-blocking probe: true if the phase with this parity has completed.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
// One lane of a converged warp (the others skip the guarded issue).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
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
// Descriptor of the tile `bytes` (a multiple of 16) past the one `d`
// describes: only the start-address field moves.  Shared-memory addresses
// are < 2^18, so start >> 4 + bytes >> 4 stays inside the 14-bit field and
// a 32-bit add on the low word is exact (no per-MMA re-encoding).
__device__ __forceinline__ uint64_t sdesc_add(uint64_t d, uint32_t bytes) {
  const uint32_t lo = uint32_t(d) + (bytes >> 4), hi = uint32_t(d >> 32);
  return (uint64_t(hi) << 32) | lo;
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

// Wave alignment of the persistent VMM producers (performance only, never a
// correctness dependency: the wait is bounded).  The CTA pairs that share a
// unit column of digit tiles read it through L2 only while they sweep it
// within a few crossbar tiles of each other (at 2-3 TB/s of operand traffic
// L2 turns over in ~50 us); nothing else keeps persistent CTAs in step, so
// each producer arrives on a global counter at the start of a round of units
// and waits (at most ~30 us) for the others.
// Returns false when the wait timed out (the caller then stops waiting: the
// CTA pairs are not all resident, e.g. another kernel shares the GPU).
__device__ __forceinline__ bool wave_align(unsigned int* ctr, unsigned int target, bool wait) {
  atomicAdd(ctr, 1u);
  if (!wait) return false;
  const long long t0 = clock64();
  while (*reinterpret_cast<volatile unsigned int*>(ctr) < target) {
    if (clock64() - t0 > 60000) return false;
    __nanosleep(64);
  }
  return true;
}

// ------------------------------------------------- CTA pairs (cta_group::2)
// Clusters of two CTAs on one TPC: the leader (rank 0) issues the M = 256
// MMAs for both; the peer's TMA loads complete on the leader's barriers and
// its epilogue warps release the leader's TMEM-empty barriers remotely.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (a shared::cta address of this CTA) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Arrival that orders nothing (the caller's TMEM reads already completed at
// tcgen05.wait::ld): no cluster-scope release fence per arrival.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-D TMA load into this CTA's smem, completing bytes on a barrier that may
// live in the peer CTA (cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
// ... with an L2 eviction-priority hint (createpolicy): operands a kernel
// re-reads (the digit tiles of a unit column) stay, streamed ones go first
__device__ __forceinline__ void tma_load_2d_pair_hint(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int x,
                                                      int y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2.L2::cache_hint "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void umma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive (once the issued MMAs complete) on the barrier at this smem offset in both CTAs
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot) {  // one warp in each CTA
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

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
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

// ------------------------------------------------------- ADC epilogue math
// A column current on the snapped grid is n = hi*65025 + lo units of 2^sh
// amperes (hi, lo = the two radix-255 digit-pair accumulators, exact s32
// < 2^24 for <= 256 crossbar rows).  The reference's code
// (converters.cpp:79-87: scaled = I / i_fs * maxc; scaled >= maxc ? maxc :
// llround(scaled)) is monotone in n, so it is fully described by the integer
// thresholds T[k] = min{n : code(n) >= k} (computed on the host with that
// exact fp64 expression, xbs_core.cu).
//
// Fast path (every conversion): x = hi c_hi + lo c_lo in fp32 with
// |x - scaled| <= ~3 2^-24 (maxc + 1) on the unsaturated range; t = rint(x)
// clamped to maxc.  Whenever |x - t| > 0.5 - delta (delta = 3.5 2^-24 (maxc + 1))
// the fast code may be off by one and the conversion is decided exactly by
// the thresholds (adc_fix).  So every code equals the reference's.
//
// No int->float conversion: an accumulator value n < 2^24, read as fp32 bits,
// is exactly n 2^-149 (subnormal below 2^23; exponent field 1 up to 2^24 is
// the same linear map).  The FMAs take subnormal inputs at full rate, so with
// constants pre-scaled by 2^(149 - s) the kernel computes x' = x 2^-s
// exactly (every step is the unscaled one times a power of two; s is chosen
// on the host so that no constant overflows and no x' is subnormal).  The
// rounding magic, clamp and threshold are scaled alike, and the shift-add
// weights by 2^s, so P still sums true codes.
// Unsigned division by a runtime divisor fixed per launch (unit decode in
// the persistent VMM loops): q = (umulhi(n, m) + n) >> s with
// s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1, exact for n < 2^31.
// Three instructions instead of the ~25 of a signed runtime division.
struct FDiv {
  uint32_t d, m, s;
};
inline FDiv make_fdiv(uint32_t d) {
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  const uint32_t m = uint32_t(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  return FDiv{d, m, s};
}
__device__ __forceinline__ int fdiv(int n, const FDiv& f) {
  return int((__umulhi(uint32_t(n), f.m) + uint32_t(n)) >> f.s);
}

// n / d through the FDiv (FAST) or the plain runtime division: the narrow-
// layer instantiations (many short units) take the former; full-width
// layers keep the division, whose code layout their hot loops were tuned on.
template <bool FAST>
__device__ __forceinline__ int udiv(int n, int d, const FDiv& f) {
  if constexpr (FAST) return fdiv(n, f);
  else return n / d;
}

struct AdcConst {
  float c_hi, c_lo, maxc;  // scaled: c * 2^(149 - s), maxc * 2^-s
  float thr;               // (0.5 - delta) * 2^-s
  float rint;              // 1.5 * 2^(23 - s): x' + rint - rint = rint(x) 2^-s for 0 <= x < 2^22
  float unscale, scale;    // 2^s, 2^-s
  uint64_t c_lo2, c_hi2, rint2;  // (c_lo, c_lo), (c_hi, c_hi), (rint, rint) for the f32x2 path
  int maxc_i;
  const unsigned long long* tab;  // T[0..maxc], T[0] = 0
};

__device__ __forceinline__ float adc_x(uint32_t hi, uint32_t lo, const AdcConst& k) {
  return __fmaf_rn(__uint_as_float(hi), k.c_hi, __fmul_rn(__uint_as_float(lo), k.c_lo));
}
__device__ __forceinline__ float rint_magic(float x, const AdcConst& k) {
  return __fsub_rn(__fadd_rn(x, k.rint), k.rint);
}

// Exact code of the current n = hi*65025 + lo given a fast candidate t that
// is off by at most one.
static __device__ __noinline__ float adc_fix(uint32_t hi, uint32_t lo, float t, const unsigned long long* tab,
                                             int maxc) {
  const unsigned long long n = (unsigned long long)hi * 65025ull + lo;
  int c = int(t);
  if (c < maxc && n >= __ldg(tab + c + 1)) ++c;
  else if (c > 0 && n < __ldg(tab + c)) --c;
  return float(c);
}

// Two conversions with packed f32x2 arithmetic (one issue slot per pair):
// the same operations, in the same order and rounding, as adc_x / fminf /
// rint_magic / x - t / P += t w on each element.
__device__ __forceinline__ void adc_pair(uint32_t lo0, uint32_t lo1, uint32_t hi0, uint32_t hi1, const AdcConst& k,
                                         uint64_t w2, float& p0, float& p1, float& mr, float& t0, float& t1,
                                         float& r0, float& r1) {
  // outputs: %0 %1 P pair, %2 running max |x - t|, %3 %4 t pair, %5 %6 x - t pair
  asm("{\n\t.reg .b64 L, H, T, X, Y, TT, RR, PP;\n\t.reg .f32 x0, x1, a0, a1;\n\t"
      "mov.b64 L, {%7, %8};\n\tmov.b64 H, {%9, %10};\n\t"
      "mul.rn.f32x2 T, L, %11;\n\tfma.rn.f32x2 X, H, %12, T;\n\t"
      "mov.b64 {x0, x1}, X;\n\tmin.f32 x0, x0, %13;\n\tmin.f32 x1, x1, %13;\n\tmov.b64 X, {x0, x1};\n\t"
      "add.rn.f32x2 Y, X, %14;\n\tsub.rn.f32x2 TT, Y, %14;\n\tsub.rn.f32x2 RR, X, TT;\n\t"
      "mov.b64 {%5, %6}, RR;\n\tabs.f32 a0, %5;\n\tabs.f32 a1, %6;\n\tmax.f32 a0, a0, a1;\n\tmax.f32 %2, %2, a0;\n\t"
      "mov.b64 PP, {%0, %1};\n\tfma.rn.f32x2 PP, TT, %15, PP;\n\tmov.b64 {%0, %1}, PP;\n\tmov.b64 {%3, %4}, TT;\n\t}"
      : "+f"(p0), "+f"(p1), "+f"(mr), "=f"(t0), "=f"(t1), "=f"(r0), "=f"(r1)
      : "r"(lo0), "r"(lo1), "r"(hi0), "r"(hi1), "l"(k.c_lo2), "l"(k.c_hi2), "f"(k.maxc), "l"(k.rint2), "l"(w2));
}

// Eight conversions lo/hi[OFF .. OFF+8) -> P[b+j] += w * code (w: the
// shift-add weight times k.unscale).  The rounded codes and residuals stay
// in registers; if any lane saw a residual beyond thr, the warp visits the
// eight and replaces the flagged codes (P += w * (exact - fast); all
// operands exact).
template <int OFF, int NL, int kN, int G = 8>
__device__ __forceinline__ void adc_conv8(const uint32_t (&lo)[NL], const uint32_t (&hi)[NL], const AdcConst& k,
                                          float w, float (&P)[kN], int b, uint32_t& exact_ctr) {
  float mr = 0.f, t[G], r[G];
  const uint64_t w2 = (uint64_t(__float_as_uint(w)) << 32) | __float_as_uint(w);
#pragma unroll
  for (int j = 0; j < G; j += 2)
    adc_pair(lo[OFF + j], lo[OFF + j + 1], hi[OFF + j], hi[OFF + j + 1], k, w2, P[b + j], P[b + j + 1], mr, t[j],
             t[j + 1], r[j], r[j + 1]);
  if (__any_sync(0xffffffffu, mr > k.thr)) {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (fabsf(r[j]) > k.thr) {
        ++exact_ctr;
        const float code = adc_fix(hi[OFF + j], lo[OFF + j], __fmul_rn(t[j], k.unscale), k.tab, k.maxc_i);
        const float d = __fsub_rn(__fmul_rn(code, k.scale), t[j]);
        P[b + j] = __fmaf_rn(d, w, P[b + j]);
      }
    }
  }
}

// Transpose-reduce of 16 int32 values over groups of G consecutive lanes
// (the bit-plane / phase lanes of one batch row): at each butterfly step a
// lane sends half of its values to its partner and keeps the other half, so
// after log2(G) steps lane q (= lane % G) holds the totals of rows
// q * (16 / G) + i (G <= 16; for G = 32, lanes q and q ^ 1 share row q >> 1).
// 15 shuffles for 16 rows instead of 16 x log2(G) for a full butterfly.
template <int O, int N, class T>
__device__ __forceinline__ void tr_step(T (&v)[16], int q) {
  if constexpr (O >= 1) {
    if constexpr (N > 1) {
      const bool up = (q & O) != 0;
#pragma unroll
      for (int i = 0; i < N / 2; ++i) {
        const T a = v[i], b = v[i + N / 2];
        const T keep = up ? b : a;
        v[i] = keep + __shfl_xor_sync(0xffffffffu, up ? a : b, O);
      }
      tr_step<O / 2, N / 2, T>(v, q);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], O);
      tr_step<O / 2, 1, T>(v, q);
    }
  }
}
template <class T>  // int, or long long where a combined total can pass 2^31
__device__ __forceinline__ void group_reduce16(T (&v)[16], int q, int G) {
  switch (G) {
    case 2: tr_step<1, 16, T>(v, q); break;
    case 4: tr_step<2, 16, T>(v, q); break;
    case 8: tr_step<4, 16, T>(v, q); break;
    case 16: tr_step<8, 16, T>(v, q); break;
    case 32: tr_step<16, 16, T>(v, q); break;
    default: break;  // G == 1
  }
}

// host helpers (xbs_vmm_tc.cu)
bool make_map_u8(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo,
                 int swizzle_bytes = 128);
int num_sms();
AdcConst make_adc_const(const AdcP& a, const unsigned long long* tab);
void* acc32(xbs_core* c, size_t bytes, cudaStream_t st);  // split-K int32 / int64 totals (xbs_fwd_tc.cu)

}  // namespace tc
}  // namespace xbs
