// K1: tcgen05 forward crossbar VMM (layers.cpp:246-283) for sm_100a, on CTA
// pairs (cta_group::2).
//
// Unit = (two 128-row M-blocks of input bit-plane rows [b * TPi + k], one per
//         CTA of the pair; 64 device output columns of one tile column).
// For every crossbar row tile tr and slice s the leader CTA issues, per
// 128-row k-block, tcgen05.mma.cta_group::2.kind::i8 (M = 256 = both
// M-blocks, K = 32) in two phases into one 256-column TMEM accumulator
// holding both polarities:
//     A_bits phase, N = 256:  D[:, 0:64 | 64:128 | 128:192 | 192:256]
//                               = A_bits . [d0_pos | d0_neg | d2_pos | d2_neg]
//     A_255 phase,  N = 128:  D[:, 0:64 | 64:128] += A_255 . [d1_pos | d1_neg]
// so lo_p = A_bits . d0 + A_255 . d1 sits at 64 p and hi_p = A_bits . d2 at
// 128 + 64 p: the exact column current of every (row, bit plane, column)
// as hi * 65025 + lo with q = d0 + 255 d1 + 65025 d2 (three u8 limbs, a
// 24-bit snapped grid) in s32 (each CTA holds its 128 rows).  That is
// 3 R int8 MACs per (row, device) instead of the 4 R of a two-pair split.
// The B operand is split along N across the pair: the leader stages d0 of
// both polarities and d1_pos, the peer d2 of both polarities and d1_neg
// (24 KB per k-block each).  The accumulation K-extent is exactly one crossbar
// (R = 128 or 256 rows, one or two k-blocks); the epilogue then applies the
// ADC (fp32 fast path + exact threshold fix-up, xbs_tc_common.cuh) and the
// signed shift-add P += +-2^(s db) * code.  After the last tile the TPi
// bit-plane lanes of each batch row are combined in int64 as
// sum_k 2^k P_k and scaled once by k_out (layers.cpp:272-283).
//
// Roles per CTA (576 threads, 1 CTA / SM): warp 0 TMA producer, warp 1 TMEM
// allocator + (leader only) MMA issuer, warps 2..17 epilogue: warp w reads
// TMEM lanes 32 (w % 4).. and device columns 16 ((w-2)/4)... (an 8-warp
// variant with 32 columns per warp and software-pipelined TMEM reads is
// kept behind XBS_FWD_EW=8 for A/B runs)
// Pipelines per CTA: A (own M-block: {bits, 255 bits} x KB k-blocks, 32 KB
// per k-block) x 3 stages (2 for 256-row crossbars), B (24 KB per k-block:
// three 64-column SW64 digit boxes) x 4, TMEM accumulators 2 x 256
// columns.  Column blocks made only of tile padding are never scheduled.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "xbs_internal.cuh"
#include "xbs_tc_common.cuh"

namespace xbs {
namespace tc {

namespace fw {
// EW epilogue warps per CTA: 8 (32 unit columns each, software-pipelined TMEM
// reads) or 16 (16 columns each, four warps per sub-partition as in the
// backward kernel)
template <int EW> constexpr int kThreadsFor = 64 + 32 * EW;
constexpr int kCW = 64;             // device columns per unit
constexpr int kABox = 128 * 128;    // 128 rows x 128 B (one k-block), SW128
constexpr int kBBox = 128 * kCW;    // 128 crossbar rows x 64 columns, SW64
constexpr int kBStage = 3 * kBBox;  // this CTA's boxes of one k-block: two A_bits-phase boxes + one A_255 box
constexpr int kTBufs = 2;           // TMEM accumulators of 256 columns (one (tr, s), both polarities)
template <int KB> constexpr int kAStage = 2 * KB * kABox;  // [dh][kb]
template <int KB> constexpr int kAStages = KB == 1 ? 3 : 2;
template <int KB> constexpr int kBStages = 4;
template <int KB>
constexpr int kSmem = kAStages<KB> * kAStage<KB> + kBStages<KB> * kBStage + 1024 + 256;
}  // namespace fw

struct FwdArgs {
  int GR, GC, S, db, TPi, tile_cols, C, R, N;
  int live, live_last;  // 64-column units holding logical columns per tile column / in the last one
  int n_nb;              // scheduled column units
  int mfast;             // unit order: 1 = M-block pairs fastest (digits streamed once), 0 = column units fastest
  int grp;               // > 1: column units per group of the grouped order (with mfast)
  int hinta;             // the input planes' evict-first hint (off: plane tiles shared inside a group)
  int hint;              // TMA L2 hints: digit tiles evict-last, input planes evict-first
  int64_t M, rowsF;
  int num_mbp, num_units;  // num_units = base units (M-block pair x column unit) x ksplit
  int nbase, ksplit, trs;   // split-K (small layers): crossbar row tiles [sp * trs, +trs) per unit
  FDiv f_nbase, f_mbp, f_nnb, f_live;  // divisions of the unit decode
  int lg_tpi;                          // log2(TPi) (a power of two)
  int* acc;                 // ksplit > 1: int32 totals [N][M] (atomics), scaled by k_out in k_fwd_finalize
  unsigned long long* acc64;  // ... int64 (two's complement) when the layer total can pass 2^31
  int wide;                   // bit-plane combine in int64 (a unit's total can pass 2^31)
  double k_out;
  AdcConst adc;
  double* y;
  int64_t ldy;  // column stride of y (M, or the caller's ld for a mapped host buffer)
  unsigned long long* ctr;
  unsigned int* wsync;  // wave alignment counter (zeroed before the launch), or null
};

// Column unit index -> (tile column, 64-column unit); units made only of
// padding are not scheduled.
template <bool FAST>
__device__ __forceinline__ void col_unit(int nb, const FwdArgs& a, int& tc, int& h) {
  tc = udiv<FAST>(nb, a.live, a.f_live);
  if (tc >= a.GC - 1) {
    tc = a.GC - 1;
    h = nb - (a.GC - 1) * a.live;
  } else {
    h = nb - tc * a.live;
  }
}

// Unit index -> (M-block pair, column unit, row-tile range).
template <bool FAST>
__device__ __forceinline__ void fwd_unit(int u, const FwdArgs& a, int& mbp, int& nb, int& tr0, int& tr1) {
  const int sp = udiv<FAST>(u, a.nbase, a.f_nbase), ub = u - sp * a.nbase;
  if (!FAST && a.grp > 1) {  // (full-width instantiations only: the narrow ones keep their short decode)
    // groups of grp column units: inside a group the column unit runs
    // fastest, then the M-block pair, so a round of CTA pairs covers
    // (pairs / grp) M-block pairs x grp column units -- each bit-plane tile
    // is read by grp pairs and each digit tile by pairs / grp of them
    const int per = a.grp * a.num_mbp, gi = ub / per, r = ub - gi * per;
    const int gl = min(a.grp, a.n_nb - gi * a.grp);  // the last group may be short
    mbp = r / gl;
    nb = gi * a.grp + (r - mbp * gl);
  } else if (a.mfast) {
    nb = udiv<FAST>(ub, a.num_mbp, a.f_mbp);
    mbp = ub - nb * a.num_mbp;
  } else {
    mbp = udiv<FAST>(ub, a.n_nb, a.f_nnb);
    nb = ub - mbp * a.n_nb;
  }
  tr0 = sp * a.trs;
  tr1 = min(a.GR, tr0 + a.trs);
}

// NARROW: some 64-column units hold fewer than 64 logical columns (N or the
// tile width not a multiple of 64), so epilogue warps skip the conversions
// of padded columns; full-width layers keep the plain pipelined loop.
template <int KB, bool NARROW, bool WIDE, int EW = 8>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(fw::kThreadsFor<EW>, 1)
    k_fwd_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, const FwdArgs a) {
  using namespace fw;
  constexpr int kEpiWarps = EW;
  constexpr int kCPW = 64 / (kEpiWarps / 4);  // unit columns per epilogue warp (32 or 16)
  constexpr int kAStage = fw::kAStage<KB>, kAStages = fw::kAStages<KB>, kBStages = fw::kBStages<KB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kAStages * kAStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kBStages * kBStage);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kAStages;
  uint64_t* b_full = a_empty + kAStages;
  uint64_t* b_empty = b_full + kBStages;
  uint64_t* t_full = b_empty + kBStages;
  uint64_t* t_empty = t_full + kTBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + kTBufs);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < kTBufs; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 2 * kEpiWarps);  // epilogue warps of both CTAs
    }
    mbar_fence_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    {  // ------------------------------- TMA producer (converged warp, one lane issues)
      uint32_t as = 0, aph = 0, bs = 0, bph = 0;
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
      int round = 0;
      bool wwait = true;  // (lane 0) cleared by a timed-out alignment wait
      for (int u = cid; u < a.num_units; u += ncl, ++round) {
        if (!NARROW && a.wsync) {  // all producers start a round of units together (xbs_tc_common.cuh)
          if (lane == 0) wwait = wave_align(a.wsync, 2u * uint32_t(min(a.num_units, (round + 1) * ncl)), wwait);
          __syncwarp();
        }
        int mbp, nb, tr0, tr1;
        fwd_unit<NARROW>(u, a, mbp, nb, tr0, tr1);
        int tc, h;
        col_unit<NARROW>(nb, a, tc, h);
        const int mrow = (2 * mbp + int(rank)) * 128;
        for (int tr = tr0; tr < tr1; ++tr) {
          mbar_wait(&a_empty[as], aph ^ 1);
          if (elect_one()) {
            if (rank == 0) mbar_expect_tx(&a_full[as], 2 * kAStage);
            const uint32_t fa = mapa(smem_u32(&a_full[as]), 0);
#pragma unroll
            for (int dh = 0; dh < 2; ++dh)
#pragma unroll
              for (int kb = 0; kb < KB; ++kb) {
                uint8_t* dst = sA + as * kAStage + (dh * KB + kb) * kABox;
                if (a.hinta) tma_load_2d_pair_hint(dst, &mapA, fa, tr * a.R + kb * 128, int(dh * a.rowsF) + mrow, pol_a);
                else tma_load_2d_pair(dst, &mapA, fa, tr * a.R + kb * 128, int(dh * a.rowsF) + mrow);
              }
          }
          __syncwarp();
          if (++as == kAStages) { as = 0; aph ^= 1; }
          for (int s = 0; s < a.S; ++s)
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              mbar_wait(&b_empty[bs], bph ^ 1);
              if (elect_one()) {
                if (rank == 0) mbar_expect_tx(&b_full[bs], 2 * kBStage);
                const uint32_t fb = mapa(smem_u32(&b_full[bs]), 0);
                // digit plane d of polarity p: row ((((s 2 + p) GR + tr) GC + tc) L + d) R
                auto row = [&](int p, int d) { return ((((s * 2 + p) * a.GR + tr) * a.GC + tc) * kLimbs + d) * a.R + kb * 128; };
                // leader: d0_pos, d0_neg, d1_pos; peer: d2_pos, d2_neg, d1_neg
                const int dpair = rank == 0 ? 0 : 2;
                if (a.hint) {
                  tma_load_2d_pair_hint(sB + bs * kBStage, &mapB, fb, h * kCW, row(0, dpair), pol_b);
                  tma_load_2d_pair_hint(sB + bs * kBStage + kBBox, &mapB, fb, h * kCW, row(1, dpair), pol_b);
                  tma_load_2d_pair_hint(sB + bs * kBStage + 2 * kBBox, &mapB, fb, h * kCW, row(int(rank), 1), pol_b);
                } else {
                  tma_load_2d_pair(sB + bs * kBStage, &mapB, fb, h * kCW, row(0, dpair));
                  tma_load_2d_pair(sB + bs * kBStage + kBBox, &mapB, fb, h * kCW, row(1, dpair));
                  tma_load_2d_pair(sB + bs * kBStage + 2 * kBBox, &mapB, fb, h * kCW, row(int(rank), 1));
                }
              }
              __syncwarp();
              if (++bs == kBStages) { bs = 0; bph ^= 1; }
            }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // ------ MMA issuer (leader CTA; converged warp, one lane issues)
      constexpr uint32_t idesc_a = idesc_i8(256, 4 * kCW, /*b_mn_major=*/true);  // A_bits phase, N = 256
      constexpr uint32_t idesc_b = idesc_i8(256, 2 * kCW, /*b_mn_major=*/true);  // A_255 phase, N = 128
      uint32_t as = 0, aph = 0, bs = 0, bph = 0, ab = 0, abph = 0;
      for (int u = cid; u < a.num_units; u += ncl) {
        const int usp = udiv<NARROW>(u, a.nbase, a.f_nbase);
        const int ntr = min(a.GR, (usp + 1) * a.trs) - usp * a.trs;
        for (int tr = 0; tr < ntr; ++tr) {
          mbar_wait(&a_full[as], aph);
          tc_fence_after();
          const uint64_t a0d = sdesc(smem_u32(sA + as * kAStage), 16, 1024, 2);
          for (int s = 0; s < a.S; ++s) {
            mbar_wait(&t_empty[ab], abph ^ 1);
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              mbar_wait(&b_full[bs], bph);
              tc_fence_after();
              // B: each CTA's boxes MN-major SW64 (8-row K groups 512 B apart,
              // 32 K rows per MMA = 2 KB; the A_bits phase spans two 64-column
              // boxes, LBO = one box)
              const uint64_t b0d = sdesc(smem_u32(sB + bs * kBStage), kBBox, 512, 4);
              if (elect_one()) {
#pragma unroll
                for (int dh = 0; dh < 2; ++dh)
#pragma unroll
                  for (int ks = 0; ks < 4; ++ks) {
                    // A: K-major SW128 (LBO 16, SBO 1024)
                    const uint64_t ad = sdesc_add(a0d, (dh * KB + kb) * kABox + 32 * ks);
                    const uint64_t bd = sdesc_add(b0d, dh * 2 * kBBox + 2048 * ks);
#ifndef XBS_STUB_MMA  // perf experiment hook (tools/build_variant.sh): no tensor work
                    umma_i8_pair(tmem + ab * 256, ad, bd, dh ? idesc_b : idesc_a, (kb | dh | ks) != 0);
#else
                    (void)ad; (void)bd;
#endif
                  }
                umma_commit_pair(&b_empty[bs]);
                if (kb == KB - 1) umma_commit_pair(&t_full[ab]);
              }
              __syncwarp();
              if (++bs == kBStages) { bs = 0; bph ^= 1; }
            }
            if (++ab == kTBufs) { ab = 0; abph ^= 1; }
          }
          if (elect_one()) umma_commit_pair(&a_empty[as]);
          __syncwarp();
          if (++as == kAStages) { as = 0; aph ^= 1; }
        }
      }
    }
  } else {  // ---------------------------------------------------- epilogue
    // warp -> (TMEM lane quarter lg, kCPW-column slice q of the unit's 64)
    const int lg = warp & 3, q = (warp - 2) >> 2;
    const int ml = 32 * lg + lane;
    const uint32_t tl = tmem + (uint32_t(32 * lg) << 16) + kCPW * q;  // + 256 ab + 64 p (+ 128: hi)
    const uint32_t te0 = mapa(smem_u32(&t_empty[0]), 0);  // leader's barriers, 8 B apart
    uint32_t ab = 0, abph = 0, exact = 0;
    const AdcConst k = a.adc;
    for (int u = cid; u < a.num_units; u += ncl) {
      int mbp, nb, tr0, tr1;
      fwd_unit<NARROW>(u, a, mbp, nb, tr0, tr1);
      const int npair = (tr1 - tr0) * a.S;  // one TMEM buffer per (tr, s): both polarities
      float P[kCPW];
#pragma unroll
      for (int j = 0; j < kCPW; ++j) P[j] = 0.f;
      // (tr, s) buffers run tr-major, then slice: weight 2^(s db) k.unscale,
      // + for the positive and - for the negative polarity, stepped without
      // integer division
      const float wstep = float(1 << a.db);
      float wmag = k.unscale;
      int sl = 0;
      // software-pipelined TMEM reads: one 16-column half is in flight while
      // the other is converted (A: columns 0-15, B: 16-31 of this warp);
      // polarity p's lo sits at +64 p, its hi at +128 + 64 p
      static_assert(kCPW == 32 || kCPW == 16, "epilogue warps of 32 (pipelined) or 16 columns");
      uint32_t alo[16], ahi[16], blo[16], bhi[16];  // the 32-column loops' TMEM registers
      // logical columns in this warp's 32 (narrow layers: N or the tile
      // width below the unit's 64 device columns); padded columns are
      // discarded (layers.cpp:283), so their conversions are skipped
      int nv = kCPW;
      if constexpr (NARROW) {
        int tcu, hu;
        col_unit<NARROW>(nb, a, tcu, hu);
        nv = min(a.tile_cols, a.N - tcu * a.tile_cols) - hu * kCW - kCPW * q;
      }
      if constexpr (kCPW == 16) {
        // 16 columns per warp (the backward kernel's loop): both accumulator
        // halves of a polarity are read, the buffer goes back to the MMA
        // issuer after the second polarity's read, conversions follow
        for (int c = 0; c < npair; ++c) {
          const float w = wmag;
          if (++sl == a.S) {
            sl = 0;
            wmag = k.unscale;
          } else {
            wmag = __fmul_rn(wmag, wstep);
          }
          uint32_t lo[16], hi[16];
          mbar_wait_hint(&t_full[ab], abph);
          tc_fence_after();
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            if (!NARROW || nv > 0) {
              tmem_ld16(tl + ab * 256 + 64 * p, lo);
              tmem_ld16(tl + ab * 256 + 64 * p + 128, hi);
              tmem_wait_ld();
            }
            if (p == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster_relaxed(te0 + 8 * ab);
              if (++ab == kTBufs) { ab = 0; abph ^= 1; }
            }
            if (NARROW && nv <= 0) continue;
            const float wp = p == 0 ? w : -w;
#ifdef XBS_STUB_EPI
            if (lo[0] == 0xdeadbeef && hi[15] == 0x12345) P[p] += wp;
#else
            adc_conv8<0, 16, kCPW>(lo, hi, k, wp, P, 0, exact);
            if (!NARROW || nv > 8) adc_conv8<8, 16, kCPW>(lo, hi, k, wp, P, 8, exact);
#endif
          }
        }
        if (NARROW && nv <= 0) continue;  // no logical output columns: nothing to combine
      } else if (NARROW && nv <= 16) {
        // at most the first 16 columns: one TMEM read per polarity and buffer
        // (none when the warp holds only padding); barrier protocol unchanged
        for (int c = 0; c < npair; ++c) {
          const float w = wmag;
          if (++sl == a.S) {
            sl = 0;
            wmag = k.unscale;
          } else {
            wmag = __fmul_rn(wmag, wstep);
          }
          mbar_wait_hint(&t_full[ab], abph);
          tc_fence_after();
          if (nv > 0) {
            tmem_ld16(tl + ab * 256, alo);
            tmem_ld16(tl + ab * 256 + 128, ahi);
            tmem_ld16(tl + ab * 256 + 64, blo);
            tmem_ld16(tl + ab * 256 + 192, bhi);
            tmem_wait_ld();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster_relaxed(te0 + 8 * ab);
          if (++ab == kTBufs) { ab = 0; abph ^= 1; }
          if (nv > 0) {
            adc_conv8<0, 16, kCPW, 16>(alo, ahi, k, w, P, 0, exact);
            adc_conv8<0, 16, kCPW, 16>(blo, bhi, k, -w, P, 0, exact);
          }
        }
        if (nv <= 0) continue;  // no logical output columns: nothing to combine
      } else {
        mbar_wait_hint(&t_full[ab], abph);
        tc_fence_after();
        tmem_ld16(tl + ab * 256, alo);
        tmem_ld16(tl + ab * 256 + 128, ahi);
        tmem_wait_ld();
        for (int c = 0; c < npair; ++c) {
          const float w = wmag;
          if (++sl == a.S) {
            sl = 0;
            wmag = k.unscale;
          } else {
            wmag = __fmul_rn(wmag, wstep);
          }
          const uint32_t tb = tl + ab * 256;
          // positive polarity: columns 0-15 in A, 16-31 loading into B
          tmem_ld16(tb + 16, blo);
          tmem_ld16(tb + 128 + 16, bhi);
#ifdef XBS_STUB_EPI  // perf experiment hook: TMEM loads and barriers only
          if (alo[0] == 0xdeadbeef && ahi[15] == 0x12345) P[0] += w;
#else
          adc_conv8<0, 16, kCPW, 16>(alo, ahi, k, w, P, 0, exact);
#endif
          tmem_wait_ld();
          tmem_ld16(tb + 64, alo);
          tmem_ld16(tb + 192, ahi);
#ifdef XBS_STUB_EPI
          if (blo[0] == 0xdeadbeef && bhi[15] == 0x12345) P[1] += w;
#else
          adc_conv8<0, 16, kCPW, 16>(blo, bhi, k, w, P, 16, exact);
#endif
          tmem_wait_ld();
          // negative polarity
          tmem_ld16(tb + 64 + 16, blo);
          tmem_ld16(tb + 192 + 16, bhi);
#ifdef XBS_STUB_EPI
          if (alo[0] == 0xdeadbeef && ahi[15] == 0x12345) P[2] += w;
#else
          adc_conv8<0, 16, kCPW, 16>(alo, ahi, k, -w, P, 0, exact);
#endif
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster_relaxed(te0 + 8 * ab);
          if (++ab == kTBufs) { ab = 0; abph ^= 1; }
          if (c + 1 < npair) {
            mbar_wait_hint(&t_full[ab], abph);
            tc_fence_after();
            tmem_ld16(tl + ab * 256, alo);
            tmem_ld16(tl + ab * 256 + 128, ahi);
          }
#ifdef XBS_STUB_EPI
          if (blo[0] == 0xdeadbeef && bhi[15] == 0x12345) P[3] += w;
#else
          adc_conv8<0, 16, kCPW, 16>(blo, bhi, k, -w, P, 16, exact);
#endif
          tmem_wait_ld();
        }
      }
      // combine the TPi bit-plane lanes of each batch row: total = sum 2^k P_k
      // (exact in int32, or in int64 when the host bound says a total can
      // pass 2^31); per 16 columns, lane q ends with the totals of columns
      // q * (16 / TPi) + i
      const int kk = NARROW ? ml & (a.TPi - 1) : ml % a.TPi;
      const int64_t b = NARROW ? (int64_t(2 * mbp + int(rank)) * 128 + ml) >> a.lg_tpi
                               : (int64_t(2 * mbp + int(rank)) * 128 + ml) / a.TPi;
      int tc, hcol;
      col_unit<NARROW>(nb, a, tc, hcol);
      const int per = NARROW ? 16 >> a.lg_tpi : 16 / a.TPi;
      auto emit = [&](auto zero) {
        using T = decltype(zero);
#pragma unroll
        for (int h = 0; h < kCPW / 16; ++h) {
          T v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = T(__float2int_rn(P[16 * h + j])) * (T(1) << kk);
          group_reduce16(v, kk, a.TPi);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i >= per) break;
            const int cc = hcol * kCW + kCPW * q + 16 * h + kk * per + i;
            const int jg = tc * a.tile_cols + cc;
            if (b < a.M && cc < a.tile_cols && jg < a.N) {
              if (a.acc) atomicAdd(&a.acc[int64_t(jg) * a.M + b], int(v[i]));  // split-K partial (exact)
              else if (a.acc64) atomicAdd(&a.acc64[int64_t(jg) * a.M + b], (unsigned long long)(long long)v[i]);
              else a.y[int64_t(jg) * a.ldy + b] = double(v[i]) * a.k_out;
            }
          }
        }
      };
      if constexpr (WIDE) emit((long long)0);
      else emit(0);
    }
    if (a.ctr) atomicAdd(&a.ctr[0], (unsigned long long)exact);
  }
  tc_fence_before();
  cluster_sync();  // both CTAs done with the pair's TMEM and barriers
  if (warp == 1) tmem_dealloc_pair<512>(tmem);
}

// Split-K: y = total * k_out (the single fp64 rounding of layers.cpp:283);
// the partial buffer is left zero for the next call.
template <class T>
__global__ void k_fwd_finalize(int64_t M, int N, double k_out, T* __restrict__ acc, double* __restrict__ y,
                               int64_t ldy) {
  const int64_t n = M * N;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = t / M, b = t - j * M;
    y[j * ldy + b] = double(static_cast<long long>(acc[t])) * k_out;  // |total| < 2^53: exact
    acc[t] = 0;
  }
}

// int32 split-K buffer of at least `bytes` (kept zero between calls)
void* acc32(xbs_core* c, size_t bytes, cudaStream_t st) {
  if (c->acc32_bytes < bytes) {
    cudaFree(c->d_acc32);
    c->d_acc32 = nullptr;
    c->acc32_bytes = 0;
    if (cudaMalloc(&c->d_acc32, bytes) != cudaSuccess) {
      c->d_acc32 = nullptr;
      (void)cudaGetLastError();
      return nullptr;
    }
    cudaMemsetAsync(c->d_acc32, 0, bytes, st);
    c->acc32_bytes = bytes;
    ++c->gen;
  }
  return c->d_acc32;
}

}  // namespace tc

bool launch_fwd_tc(xbs_core* c, int64_t M, double* d_y, int64_t ldy, cudaStream_t st) {
  using namespace tc;
  const Geo& g = c->g;
  if ((g.R != 128 && g.R != 256) || g.TPi > 16 || c->adc.passthrough) return false;
  // Exactness bounds, per crossbar row tile a unit sums: the fp32 P
  // accumulators hold |sum| <= tiles * maxc * sum_s 2^(s db) < 2^24 (a
  // layer with more row tiles is split into row-tile ranges, split-K, whose
  // exact integer partials are added with atomics), and the bit-plane
  // combine |sum_k 2^k P_k| runs in int32, or in int64 (with int64 totals:
  // the WIDE instantiation) when it can pass 2^31 -- so any K and any
  // activation width stay on the tensor cores.
  const double sw = (std::pow(2.0, g.wb) - 1) / (std::pow(2.0, g.db) - 1);
  const double per_tile = double(c->adc.maxc) * sw;
  const int trs_cap = int(16777215.0 / per_tile);
  if (trs_cap < 1) return false;
  const bool wide = double(g.GR) * per_tile * (std::pow(2.0, g.Ti) - 1) >= 2147483648.0;
  const int64_t rowsF = rows_fwd(M, g.TPi);
  CUtensorMap mA, mB;
  if (!make_map_u8(&mA, c->d_Af, uint64_t(g.KI), uint64_t(2 * rowsF), 128, 128, 128)) return false;
  if (!make_map_u8(&mB, c->d_digits, uint64_t(g.C), uint64_t(g.digits_bytes() / g.C), fw::kCW, 128, 64))
    return false;
  FwdArgs a{};
  a.wide = wide ? 1 : 0;
  a.GR = g.GR;
  a.GC = g.GC;
  a.S = g.S;
  a.db = g.db;
  a.TPi = g.TPi;
  a.lg_tpi = 0;
  while ((1 << a.lg_tpi) < g.TPi) ++a.lg_tpi;
  a.tile_cols = g.tile_cols;
  a.C = g.C;
  a.R = g.R;
  a.N = g.N;
  a.live = (g.tile_cols + fw::kCW - 1) / fw::kCW;
  a.M = M;
  a.rowsF = rowsF;
  a.num_mbp = int(rowsF / 256);
  a.live_last = (g.N - (g.GC - 1) * g.tile_cols + fw::kCW - 1) / fw::kCW;
  a.n_nb = (g.GC - 1) * a.live + a.live_last;
  a.nbase = a.num_mbp * a.n_nb;
  // small layers: too few units for the 74 CTA pairs, so the crossbar row
  // tiles of a unit are split across pairs and the exact integer totals
  // summed with int32 atomics (the host-checked bound covers any partial)
  const int pairs = num_sms() / 2;
  a.ksplit = 1;
  if (2 * a.nbase <= pairs && g.GR > 1) a.ksplit = std::min(g.GR, pairs / a.nbase);
  a.ksplit = std::max(a.ksplit, (g.GR + trs_cap - 1) / trs_cap);
  a.trs = (g.GR + a.ksplit - 1) / a.ksplit;
  a.ksplit = (g.GR + a.trs - 1) / a.trs;
  if (int64_t(a.nbase) * a.ksplit >= (int64_t{1} << 31)) return false;
  a.num_units = a.nbase * a.ksplit;
  a.f_nbase = make_fdiv(uint32_t(a.nbase));
  a.f_mbp = make_fdiv(uint32_t(a.num_mbp));
  a.f_nnb = make_fdiv(uint32_t(a.n_nb));
  a.f_live = make_fdiv(uint32_t(a.live));
  a.acc = nullptr;
  a.acc64 = nullptr;
  if (a.ksplit > 1) {
    void* buf = acc32(c, size_t(M) * g.N * (wide ? 8 : 4), st);
    if (!buf) return false;
    if (wide) a.acc64 = static_cast<unsigned long long*>(buf);
    else a.acc = static_cast<int*>(buf);
  }
  {  // sweep the larger operand once: A (input planes) vs the conductance digits
    const double bytesA = 2.0 * double(rowsF) * g.KI, bytesB = double(g.digits_bytes()) * a.n_nb / (g.GC * (g.C / fw::kCW));
    // an operand that fits in L2 (126 MB; use half) is re-read for free
    const double l2 = 64.0 * 1024 * 1024;
    const double costM = (bytesA <= l2 ? bytesA : bytesA * a.n_nb) + bytesB;  // M-blocks fastest
    const double costO = bytesA + (bytesB <= l2 ? bytesB : bytesB * a.num_mbp);        // other index fastest
    a.mfast = costM <= costO ? 1 : 0;
    // input planes larger than L2 stream past the digit tiles of the
    // current column unit: keep the digits resident (evict-last) and let the
    // planes go first (C5: forward DRAM reads 202 -> 142 GB, -4.6 % time;
    // grouping column units pays only once the rounds are kept in step, below)
    a.hint = a.mfast && bytesA > l2 ? 1 : 0;
    if (std::getenv("XBS_NO_L2_HINTS")) a.hint = 0;  // A/B switch (perf experiments only)
  }
  a.k_out = c->k_out_fwd;
  a.adc = make_adc_const(c->adc, c->d_adc_tab);
  if (a.adc.unscale == 0.0f) return false;
  a.y = d_y;
  a.ldy = ldy;
  a.ctr = &c->d_sc->exact_path;
  // Both operands larger than L2 (C5): the CTA pairs of a round are kept in
  // step (wave_align, xbs_tc_common.cuh) and a round covers 4 column units x
  // pairs / 4 M-block pairs, so each digit tile is read through L2 by ~18
  // pairs and each plane tile by 4 (the planes then take no evict-first
  // hint).  C5 forward: DRAM reads 202 -> 43 GB per launch, 77.8 -> 75.4 ms
  // (interleaved A/B, profiles/r02/wave_ab.md).  XBS_NO_WAVE_SYNC: A/B switch.
  // Not when the epilogues store into a mapped host buffer: pairs in step
  // finish their units together, and the 32-byte PCIe writes of all 148 CTAs
  // then collide instead of hiding behind the other pairs' MMAs (C5 e2e
  // 226 -> 244 ms with the alignment, profiles/r02/wave_ab.md).
  a.wsync = nullptr;
  a.grp = 1;
  a.hinta = a.hint;
  const bool narrow_cols = (g.tile_cols % fw::kCW) != 0 || ((g.N - (g.GC - 1) * g.tile_cols) % fw::kCW) != 0;
  if (a.hint && !narrow_cols && !c->out_host && !std::getenv("XBS_NO_WAVE_SYNC")) {
    a.grp = std::getenv("XBS_WAVE_GROUP") ? std::max(1, std::atoi(std::getenv("XBS_WAVE_GROUP"))) : 4;
    a.hinta = a.grp > 1 && !std::getenv("XBS_WAVE_AHINT") ? 0 : 1;
    a.wsync = &c->d_sc->wave_sync[0];
    cudaMemsetAsync(a.wsync, 0, sizeof(unsigned int), st);
  }
  const int grid_ = 2 * std::min(a.num_units, num_sms() / 2);  // CTA pairs
  auto launch = [&](auto kern, int smem, int threads) {
    static const void* done[16];
    static int ndone = 0;
    bool seen = false;
    for (int k = 0; k < ndone; ++k) seen |= done[k] == reinterpret_cast<const void*>(kern);
    if (!seen) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (ndone < 16) done[ndone++] = reinterpret_cast<const void*>(kern);
    }
    kern<<<grid_, threads, smem, st>>>(mA, mB, a);
  };
  const bool narrow = (g.tile_cols % fw::kCW) != 0 || ((g.N - (g.GC - 1) * g.tile_cols) % fw::kCW) != 0;
  const int sel = (g.R == 256 ? 4 : 0) + (narrow ? 2 : 0) + (wide ? 1 : 0);
  // Epilogue warps per CTA (fw::kThreadsFor): 16 warps of 16 columns hand an
  // accumulator back to the MMA issuer half way through its conversions
  // (after the second polarity's TMEM read), the 8-warp software-pipelined
  // loop only after three quarters, and with two accumulators per CTA that
  // slack decides whether the next chain's MMAs are done when the epilogue
  // asks for them: C5 forward 76.0 -> 65.8 ms, C2-4096 0.841 -> 0.770 ms, C3
  // (all layers) 3.85 -> 3.36 ms, C4 12.89 -> 12.27 ms (interleaved A/B,
  // profiles/r02/ew_ab.md).  Narrow layers (most of a unit's columns are
  // padding: a few warps hold all the work) and layers too small to fill the
  // pairs (split-K, or a short chain sequence: each chain's latency shows)
  // keep the 8-warp loop, which reads a whole buffer out before converting
  // (C3 forward 3.06-3.26 vs 3.36 ms, C1 0.055 vs 0.077 ms; profiles/r02/ew_ab.md).  XBS_FWD_EW=8 | 16 forces one for A/B runs.
  static const int ew_env = std::getenv("XBS_FWD_EW") ? std::atoi(std::getenv("XBS_FWD_EW")) : 0;
  // chains a pair runs back to back: short sequences are latency-, not throughput-paced (C2-512: 16 chains,
  // 0.045 vs 0.066 ms; C2-1024: 64 chains, 0.086 vs 0.099 ms; C2-2048: 256 chains, 0.259 vs 0.246 ms)
  const int64_t chains = int64_t((a.num_units + pairs - 1) / pairs) * a.trs * g.S;
  const int ew = ew_env == 8 || ew_env == 16 ? ew_env : ((narrow || a.ksplit > 1 || chains < 128) ? 8 : 16);
  constexpr int T8 = fw::kThreadsFor<8>, T16 = fw::kThreadsFor<16>;
  switch (sel + (ew == 16 ? 8 : 0)) {
    case 0: launch(k_fwd_tc<1, false, false>, fw::kSmem<1>, T8); break;
    case 1: launch(k_fwd_tc<1, false, true>, fw::kSmem<1>, T8); break;
    case 2: launch(k_fwd_tc<1, true, false>, fw::kSmem<1>, T8); break;
    case 3: launch(k_fwd_tc<1, true, true>, fw::kSmem<1>, T8); break;
    case 4: launch(k_fwd_tc<2, false, false>, fw::kSmem<2>, T8); break;
    case 5: launch(k_fwd_tc<2, false, true>, fw::kSmem<2>, T8); break;
    case 6: launch(k_fwd_tc<2, true, false>, fw::kSmem<2>, T8); break;
    case 7: launch(k_fwd_tc<2, true, true>, fw::kSmem<2>, T8); break;
    case 8: launch(k_fwd_tc<1, false, false, 16>, fw::kSmem<1>, T16); break;
    case 9: launch(k_fwd_tc<1, false, true, 16>, fw::kSmem<1>, T16); break;
    case 10: launch(k_fwd_tc<1, true, false, 16>, fw::kSmem<1>, T16); break;
    case 11: launch(k_fwd_tc<1, true, true, 16>, fw::kSmem<1>, T16); break;
    case 12: launch(k_fwd_tc<2, false, false, 16>, fw::kSmem<2>, T16); break;
    case 13: launch(k_fwd_tc<2, false, true, 16>, fw::kSmem<2>, T16); break;
    case 14: launch(k_fwd_tc<2, true, false, 16>, fw::kSmem<2>, T16); break;
    default: launch(k_fwd_tc<2, true, true, 16>, fw::kSmem<2>, T16); break;
  }
  if (a.acc || a.acc64) {
    const int64_t n = M * g.N;
    const int fb = int(std::min<int64_t>((n + 255) / 256, 4 * num_sms()));
    if (a.acc) k_fwd_finalize<<<fb, 256, 0, st>>>(M, g.N, a.k_out, a.acc, d_y, ldy);
    else k_fwd_finalize<<<fb, 256, 0, st>>>(M, g.N, a.k_out, a.acc64, d_y, ldy);
    c->launches += 1;
  }
  return cudaPeekAtLastError() == cudaSuccess;
}

}  // namespace xbs
