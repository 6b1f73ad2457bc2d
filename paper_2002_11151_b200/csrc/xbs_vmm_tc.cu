// K2: tcgen05 backward crossbar VMM for sm_100a, plus the tensor-map / ADC
// constant helpers shared with K1 (xbs_fwd_tc.cu) and K3a (xbs_dw_tc.cu).
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "xbs_internal.cuh"
#include "xbs_tc_common.cuh"

namespace xbs {
namespace tc {

#ifndef XBS_BWD_EPI_WARPS
#define XBS_BWD_EPI_WARPS 16
#endif
constexpr int kEpiWarps = XBS_BWD_EPI_WARPS;  // 2 or 4 per SM sub-partition
constexpr int kThreads = 64 + 32 * kEpiWarps;  // + TMA producer, MMA issuer
constexpr int kPlane = 128 * 128;          // one 128x128 u8 box

// ------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D u8 tensor [outer][inner], box box_inner x box_outer, 128B (default)
// or 64B swizzle.
static bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                     uint32_t box_outer, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

bool make_map_u8(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo,
                 int swizzle_bytes) {
  return make_map(m, base, inner, outer, bi, bo,
                  swizzle_bytes == 32   ? CU_TENSOR_MAP_SWIZZLE_32B
                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                        : CU_TENSOR_MAP_SWIZZLE_128B);
}
int num_sms() { return sm_count(); }

AdcConst make_adc_const(const AdcP& a, const unsigned long long* tab) {
  AdcConst k{};
  const double cn = std::ldexp(1.0, a.sh) / a.i_fs * a.maxc_d;  // codes per current unit
  const float c_lo = float(cn), c_hi = float(65025.0 * cn);
  // x_fast = (hi c_hi (1+e2) + lo c_lo (1+e1)(1+e3))(1+e4), |e| <= u = 2^-24
  // (constants' rounding, FMUL, FFMA), so |x_fast - x| <= ((1+u)^3 - 1) x
  // with x <= maxc + 1 wherever the code is not saturated.  delta = 3.5 u
  // (maxc + 1) covers that, the fp64 host constants (~2^-52 relative) and
  // the rounding of thr to fp32 (<= 2^-25).
  const double maxc = double(a.maxc);
  const double delta = 3.5 * 0x1p-24 * (maxc + 1.0);
  // scale 2^-s (xbs_tc_common.cuh): c_hi 2^(149 - s) <= 2^126, and the
  // smallest nonzero term lo c_lo 2^-s >= 2^-100 stays normal
  int e_hi;
  (void)std::frexp(double(c_hi), &e_hi);  // c_hi < 2^e_hi
  const int s = e_hi + 23;
  if (!(c_lo > 0.0f) || std::ldexp(double(c_lo), -s) < 0x1p-100 || s > 110 || s < -100)
    return AdcConst{};  // out of the scaled range: caller falls back
  k.c_lo = std::ldexp(c_lo, 149 - s);
  k.c_hi = std::ldexp(c_hi, 149 - s);
  k.thr = std::ldexp(float(0.5 - delta), -s);
  k.maxc = std::ldexp(float(a.maxc), -s);
  k.rint = std::ldexp(1.5f, 23 - s);
  k.unscale = std::ldexp(1.0f, s);
  k.scale = std::ldexp(1.0f, -s);
  auto pk = [](float v) {
    uint32_t u;
    std::memcpy(&u, &v, 4);
    return (uint64_t(u) << 32) | u;
  };
  k.c_lo2 = pk(k.c_lo);
  k.c_hi2 = pk(k.c_hi);
  k.rint2 = pk(k.rint);
  k.maxc_i = a.maxc;
  k.tab = tab;
  return k;
}

}  // namespace tc

// ---------------------------------------------------------------------------
// K2 backward (layers.cpp:339-379) on CTA pairs (cta_group::2).  Unit =
// (two 128-row blocks of error bit-plane rows [(b * TPe + k) * 2 + phase], one
// per CTA of the pair; 64 device rows of one crossbar row tile).  For each
// crossbar column tile tc and slice s the leader issues, per 128-column
// k-block, tcgen05.mma.cta_group::2.kind::i8 (M = 256, K = 32) with the
// transposed tiles read K-major straight from the same digit planes, in two
// phases into one 256-column accumulator holding both polarities:
//     A_bits phase, N = 256: D[:, 64 p + r]       = v_phi . d0_p,
//                            D[:, 128 + 64 p + r] = v_phi . d2_p
//     A_255 phase,  N = 128: D[:, 64 p + r]      += 255 v_phi . d1_p
// i.e. lo / hi of the products vp.gp and vm.gp (p = 0) or vp.gn and vm.gn
// (p = 1) of the reference (phase in M), q = d0 + 255 d1 + 65025 d2.  B is
// split along N across the pair: the leader stages d0 of both polarities and
// d1_pos, the peer d2 of both polarities and d1_neg.  Two 256-column TMEM
// accumulators let the MMAs run one (tc, s) ahead of the epilogue.  The epilogue
// converts every product through the ADC and accumulates +-2^(s db) * code
// with sign +1 when phase == polarity (acc_pos) and -1 otherwise (acc_neg).
namespace tc {

namespace bw {
constexpr int kBHalf = 64 * 128;     // one [64 rows][128 cols] digit box
constexpr int kBStage = 3 * kBHalf;  // this CTA's boxes: two A_bits-phase boxes (pos, neg) + one A_255 box
constexpr int kTBufs = 2;            // TMEM accumulators of 256 columns (one (tc, s), both polarities)
template <int KB> constexpr int kAStage = 2 * KB * kPlane;  // [dh][kb]
template <int KB> constexpr int kAStages = 2;
template <int KB> constexpr int kBStages = KB == 1 ? 5 : 4;
template <int KB>
constexpr int kSmem = kAStages<KB> * kAStage<KB> + kBStages<KB> * kBStage + 1024 + 256;
}  // namespace bw

struct BwdArgs {
  int GR, GC, S, db, TPe, tile_rows, tile_cols, R, C, K, N;
  int live, live_last;  // 64-row blocks holding logical rows per row tile / in the last row tile
  int n_rb;              // scheduled row blocks
  int mfast;             // unit order: 1 = M-block pairs fastest (digits streamed once), 0 = row blocks fastest
  int grp;               // > 1: row blocks per group of the grouped order (with mfast)
  int hinta;             // the error planes' evict-first hint (off: plane tiles shared inside a group)
  int hint;              // TMA L2 hints: digit tiles evict-last, error planes evict-first
  int64_t M, rowsB;
  int num_mbp, num_units;  // num_units = base units (M-block pair x row block) x ksplit
  int nbase, ksplit, tcs;   // split-K (small layers): crossbar column tiles [sp * tcs, +tcs) per unit
  FDiv f_nbase, f_mbp, f_nrb, f_live;  // divisions of the unit decode
  int lg_grp;                          // log2(2 TPe) (TPe a power of two)
  int abox;                            // bytes of one A box: 128 rows x min(NB, 128) (K-major)
  uint32_t a_sbo, a_layout;            // its UMMA descriptor: 8-row stride, swizzle (SW128 / SW64 / SW32)
  int* acc;                 // ksplit > 1: int32 totals [K][M] (atomics), scaled in k_bwd_finalize
  unsigned long long* acc64;  // ... int64 (two's complement) when the layer total can pass 2^31
  int wide;                   // (plane, phase) combine in int64 (a unit's total can pass 2^31)
  double F, vu, ifs_fac, lev_e;
  int adc_scaled;
  const DevScalars* sc;
  AdcConst adc;
  double* dx;
  int64_t ldx;  // column stride of dx (M, or the caller's ld for a mapped host buffer)
  unsigned long long* ctr;
  unsigned int* wsync;  // wave alignment counter (zeroed before the launch), or null
};

// Row block index -> (row tile, 64-row half); blocks made only of padding
// (beyond K in the last row tile) are not scheduled.
template <bool FAST>
__device__ __forceinline__ void row_block(int rb, const BwdArgs& a, int& tr, int& rh) {
  tr = udiv<FAST>(rb, a.live, a.f_live);
  if (tr >= a.GR - 1) {
    tr = a.GR - 1;
    rh = rb - (a.GR - 1) * a.live;
  } else {
    rh = rb - tr * a.live;
  }
}

// Unit index -> (M-block pair, row block, column-tile range).
template <bool FAST>
__device__ __forceinline__ void bwd_unit(int u, const BwdArgs& a, int& mbp, int& rb, int& tc0, int& tc1) {
  const int sp = udiv<FAST>(u, a.nbase, a.f_nbase), ub = u - sp * a.nbase;
  if (!FAST && a.grp > 1) {  // grouped order, as fwd_unit (xbs_fwd_tc.cu); full-width instantiations only
    const int per = a.grp * a.num_mbp, gi = ub / per, r = ub - gi * per;
    const int gl = min(a.grp, a.n_rb - gi * a.grp);
    mbp = r / gl;
    rb = gi * a.grp + (r - mbp * gl);
  } else if (a.mfast) {
    rb = udiv<FAST>(ub, a.num_mbp, a.f_mbp);
    mbp = ub - rb * a.num_mbp;
  } else {
    mbp = udiv<FAST>(ub, a.n_rb, a.f_nrb);
    rb = ub - mbp * a.n_rb;
  }
  tc0 = sp * a.tcs;
  tc1 = min(a.GC, tc0 + a.tcs);
}

// dx scale of layers.cpp:375-377 (same expression on every path)
__device__ __forceinline__ double bwd_k_out(const BwdArgs& a) {
  const double se = a.sc->se;
  const double step_e = se > 0 ? se / a.lev_e : 0.0;
  double k_out = step_e * a.F / a.vu;
  if (a.adc_scaled) k_out *= a.ifs_fac;
  return k_out;
}

// TRIM: the layer has padded crossbar columns (N not a multiple of the tile
// width, or tiles narrower than the 128-column device tile), so the MMA
// issuer skips K = 32 steps made only of padding, or padded crossbar rows
// inside a scheduled 64-row block, whose conversions the epilogue warps
// skip; without padding the issue and epilogue loops are the plain ones.
template <int KB, bool TRIM, bool WIDE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_bwd_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, const BwdArgs a) {
  using namespace bw;
  constexpr int kAStage = bw::kAStage<KB>, kAStages = bw::kAStages<KB>, kBStages = bw::kBStages<KB>;
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
        if (!TRIM && a.wsync) {  // all producers start a round of units together (xbs_tc_common.cuh)
          if (lane == 0) wwait = wave_align(a.wsync, 2u * uint32_t(min(a.num_units, (round + 1) * ncl)), wwait);
          __syncwarp();
        }
        int mbp, rb, tc0, tc1;
        bwd_unit<TRIM>(u, a, mbp, rb, tc0, tc1);
        int tr, rh;
        row_block<TRIM>(rb, a, tr, rh);
        const int mrow = (2 * mbp + int(rank)) * 128;
        for (int tc = tc0; tc < tc1; ++tc) {
          mbar_wait(&a_empty[as], aph ^ 1);
          if (elect_one()) {
            if (rank == 0) mbar_expect_tx(&a_full[as], 2 * 2 * KB * a.abox);
            const uint32_t fa = mapa(smem_u32(&a_full[as]), 0);
#pragma unroll
            for (int dh = 0; dh < 2; ++dh)
#pragma unroll
              for (int kb = 0; kb < KB; ++kb) {
                uint8_t* dst = sA + as * kAStage + (dh * KB + kb) * kPlane;
                if (a.hinta) tma_load_2d_pair_hint(dst, &mapA, fa, tc * a.C + kb * 128, int(dh * a.rowsB) + mrow, pol_a);
                else tma_load_2d_pair(dst, &mapA, fa, tc * a.C + kb * 128, int(dh * a.rowsB) + mrow);
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
                uint8_t* dst = sB + bs * kBStage;
                // digit plane d of polarity p, this unit's 64 device rows
                auto row = [&](int p, int d) {
                  return ((((s * 2 + p) * a.GR + tr) * a.GC + tc) * kLimbs + d) * a.R + rh * 64;
                };
                // leader: d0_pos, d0_neg, d1_pos; peer: d2_pos, d2_neg, d1_neg
                const int dpair = rank == 0 ? 0 : 2;
                if (a.hint) {
                  tma_load_2d_pair_hint(dst, &mapB, fb, kb * 128, row(0, dpair), pol_b);
                  tma_load_2d_pair_hint(dst + kBHalf, &mapB, fb, kb * 128, row(1, dpair), pol_b);
                  tma_load_2d_pair_hint(dst + 2 * kBHalf, &mapB, fb, kb * 128, row(int(rank), 1), pol_b);
                } else {
                  tma_load_2d_pair(dst, &mapB, fb, kb * 128, row(0, dpair));
                  tma_load_2d_pair(dst + kBHalf, &mapB, fb, kb * 128, row(1, dpair));
                  tma_load_2d_pair(dst + 2 * kBHalf, &mapB, fb, kb * 128, row(int(rank), 1));
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
      constexpr uint32_t idesc_a = idesc_i8(256, 256, /*b_mn_major=*/false);  // A_bits phase
      constexpr uint32_t idesc_b = idesc_i8(256, 128, /*b_mn_major=*/false);  // A_255 phase
      uint32_t as = 0, aph = 0, bs = 0, bph = 0, ab = 0, abph = 0;
      for (int u = cid; u < a.num_units; u += ncl) {
        const int tc0 = udiv<TRIM>(u, a.nbase, a.f_nbase) * a.tcs, ntc = min(a.GC, tc0 + a.tcs) - tc0;
        for (int tc = 0; tc < ntc; ++tc) {
          // crossbar columns holding logical outputs: padded columns carry a
          // zero error, so K = 32 steps made only of padding are not issued
          const int lcol = min(a.tile_cols, a.N - (tc0 + tc) * a.tile_cols);
          mbar_wait(&a_full[as], aph);
          tc_fence_after();
          const uint64_t a0d = sdesc(smem_u32(sA + as * kAStage), 16, a.a_sbo, a.a_layout);
          for (int s = 0; s < a.S; ++s) {
            mbar_wait(&t_empty[ab], abph ^ 1);  // both polarities' accumulator
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              mbar_wait(&b_full[bs], bph);
              tc_fence_after();
              // B K-major SW128; the A_bits phase spans the two 64-row boxes
              // (128 N rows per CTA, 8-row groups 1024 B apart)
              const uint64_t b0d = sdesc(smem_u32(sB + bs * kBStage), 16, 1024, 2);
              const int nks = TRIM ? min(4, (lcol - kb * 128 + 31) >> 5) : 4;  // >= 1 for kb 0
              if (elect_one()) {
                const uint32_t td = tmem + ab * 256;
#pragma unroll
                for (int dh = 0; dh < 2; ++dh)
#pragma unroll
                  for (int ks = 0; ks < 4; ++ks) {
                    if (TRIM && ks >= nks) break;
                    const uint64_t ad = sdesc_add(a0d, (dh * KB + kb) * kPlane + 32 * ks);
                    const uint64_t bd = sdesc_add(b0d, dh * 2 * kBHalf + 32 * ks);
#ifndef XBS_STUB_MMA  // perf experiment hook (tools/build_variant.sh): no tensor work
                    umma_i8_pair(td, ad, bd, dh ? idesc_b : idesc_a, (kb | dh | ks) != 0);
#else
                    (void)ad; (void)bd; (void)td;
#endif
                  }
                if (kb == KB - 1) umma_commit_pair(&t_full[ab]);
                umma_commit_pair(&b_empty[bs]);
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
    // Per (tc, s) a warp converts kRows (16 or 32) device rows x 2 polarities
    // (polarity p: lo at +64 p, hi at +128 + 64 p of the 256-column buffer).
    constexpr int kRows = 64 / (kEpiWarps / 4);  // output rows per epilogue warp
    const int lg = warp & 3, ch = (warp - 2) >> 2;
    const int ml = 32 * lg + lane;
    const int phi = ml & 1;
    const uint32_t tl = tmem + (uint32_t(32 * lg) << 16) + kRows * ch;
    const uint32_t te0 = mapa(smem_u32(&t_empty[0]), 0);  // leader's barriers, 8 B apart
    uint32_t ab = 0, abph = 0, exact = 0;
    const AdcConst k = a.adc;
    const double k_out = bwd_k_out(a);  // layers.cpp:375-377
    for (int u = cid; u < a.num_units; u += ncl) {
      int mbp, rb, tc0, tc1;
      bwd_unit<TRIM>(u, a, mbp, rb, tc0, tc1);
      const int nchain = (tc1 - tc0) * a.S;
      int tr, rh;
      row_block<TRIM>(rb, a, tr, rh);
      // logical device rows among this warp's kRows: rows beyond K (or the
      // tile height) are discarded (layers.cpp:378), so a warp holding only
      // padding skips its TMEM reads and conversions (barrier protocol kept)
      const int nvr = TRIM ? min(a.tile_rows, a.K - tr * a.tile_rows) - rh * 64 - kRows * ch : kRows;
      float P[kRows];
#pragma unroll
      for (int j = 0; j < kRows; ++j) P[j] = 0.f;
      bool nchain_done = false;
      const float wstep = float(1 << a.db);
      float wmag = k.unscale;
      int s = 0;
#ifdef XBS_BWD_PIPE
      if constexpr (kRows == 16) {
        if (!TRIM || nvr > 0) {
          // software-pipelined TMEM reads (as in the forward epilogue): the
          // negative polarity's 16 rows load while the positive ones are
          // converted, and the next chain's positive rows while the negative
          // ones are
          uint32_t alo[16], ahi[16], blo[16], bhi[16];
          mbar_wait_hint(&t_full[ab], abph);
          tc_fence_after();
          tmem_ld16(tl + ab * 256, alo);
          tmem_ld16(tl + ab * 256 + 128, ahi);
          tmem_wait_ld();
          for (int c = 0; c < nchain; ++c) {
            const float w = wmag;
            if (++s == a.S) {
              s = 0;
              wmag = k.unscale;
            } else {
              wmag = __fmul_rn(wmag, wstep);
            }
            const float wpos = phi == 0 ? w : -w;
            const float wneg = phi == 1 ? w : -w;
            const uint32_t tb = tl + ab * 256;
            tmem_ld16(tb + 64, blo);
            tmem_ld16(tb + 192, bhi);
#ifdef XBS_BWD_G16
            if (!TRIM || nvr > 8) adc_conv8<0, 16, kRows, 16>(alo, ahi, k, wpos, P, 0, exact);
            else adc_conv8<0, 16, kRows>(alo, ahi, k, wpos, P, 0, exact);
#else
            adc_conv8<0, 16, kRows>(alo, ahi, k, wpos, P, 0, exact);
            if (!TRIM || nvr > 8) adc_conv8<8, 16, kRows>(alo, ahi, k, wpos, P, 8, exact);
#endif
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(te0 + 8 * ab);
            if (++ab == kTBufs) { ab = 0; abph ^= 1; }
            if (c + 1 < nchain) {
              mbar_wait_hint(&t_full[ab], abph);
              tc_fence_after();
              tmem_ld16(tl + ab * 256, alo);
              tmem_ld16(tl + ab * 256 + 128, ahi);
            }
#ifdef XBS_BWD_G16
            if (!TRIM || nvr > 8) adc_conv8<0, 16, kRows, 16>(blo, bhi, k, wneg, P, 0, exact);
            else adc_conv8<0, 16, kRows>(blo, bhi, k, wneg, P, 0, exact);
#else
            adc_conv8<0, 16, kRows>(blo, bhi, k, wneg, P, 0, exact);
            if (!TRIM || nvr > 8) adc_conv8<8, 16, kRows>(blo, bhi, k, wneg, P, 8, exact);
#endif
            tmem_wait_ld();
          }
          nchain_done = true;
        }
      }
#endif
      for (int c = 0; c < nchain && !nchain_done; ++c) {
        // chains run tc-major, then slice: weight 2^(s db) k.unscale
        const float w = wmag;
        if (++s == a.S) {
          s = 0;
          wmag = k.unscale;
        } else {
          wmag = __fmul_rn(wmag, wstep);
        }
        const float wpos = phi == 0 ? w : -w;  // polarity 0 (gp): + for the plus phase
        const float wneg = phi == 1 ? w : -w;  // polarity 1 (gn): + for the minus phase
        uint32_t lo[kRows], hi[kRows];
        mbar_wait_hint(&t_full[ab], abph);
        tc_fence_after();
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint32_t ta = tl + ab * 256 + 64 * p;
          if (!TRIM || nvr > 0) {
#pragma unroll
            for (int h = 0; h < kRows / 16; ++h) {
              tmem_ld16(ta + 16 * h, *reinterpret_cast<uint32_t(*)[16]>(&lo[16 * h]));
              tmem_ld16(ta + 128 + 16 * h, *reinterpret_cast<uint32_t(*)[16]>(&hi[16 * h]));
            }
            tmem_wait_ld();
          }
          if (p == 1) {  // both polarities read: the buffer goes back to the MMA issuer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(te0 + 8 * ab);
            if (++ab == kTBufs) { ab = 0; abph ^= 1; }
          }
          if (TRIM && nvr <= 0) continue;
          const float wp = p == 0 ? wpos : wneg;
#ifdef XBS_STUB_EPI  // perf experiment hook: TMEM loads and barriers only
          if (lo[0] == 0xdeadbeef && hi[kRows - 1] == 0x12345) P[0] += wp;
          continue;
#endif
#ifdef XBS_BWD_G16
          if (kRows == 16 && (!TRIM || nvr > 8)) {
            adc_conv8<0, kRows, kRows, 16>(lo, hi, k, wp, P, 0, exact);
          } else {
            adc_conv8<0>(lo, hi, k, wp, P, 0, exact);
            if (!TRIM || nvr > 8) adc_conv8<8>(lo, hi, k, wp, P, 8, exact);
          }
#else
          adc_conv8<0>(lo, hi, k, wp, P, 0, exact);
          if (!TRIM || nvr > 8) adc_conv8<8>(lo, hi, k, wp, P, 8, exact);
#endif
          if constexpr (kRows >= 32) {
            if (!TRIM || nvr > 16) adc_conv8<16>(lo, hi, k, wp, P, 16, exact);
            if (!TRIM || nvr > 24) adc_conv8<24>(lo, hi, k, wp, P, 24, exact);
          }
        }
      }
      if (TRIM && nvr <= 0) continue;  // no logical output rows: nothing to combine
      // combine the 2*TPe (plane, phase) lanes of each batch row (exact in
      // int32: host-checked bound); lane q ends with the totals of rows
      // q * (16 / grp) + i (grp = 32: lanes q, q ^ 1 share row q >> 1)
      const int grp = 2 * a.TPe;
      const int q = TRIM ? ml & (grp - 1) : ml % grp, kk = q >> 1;
      const int64_t b = TRIM ? int64_t(2 * mbp + int(rank)) * (128 >> a.lg_grp) + (ml >> a.lg_grp)
                             : int64_t(2 * mbp + int(rank)) * (128 / grp) + ml / grp;
      const int per = grp <= 16 ? (TRIM ? 16 >> a.lg_grp : 16 / grp) : 1;
      const int j0 = grp <= 16 ? q * per : (q >> 1);
      const bool writer = grp <= 16 || (q & 1) == 0;
      auto emit = [&](auto zero) {
        using T = decltype(zero);
#pragma unroll
        for (int h = 0; h < kRows / 16; ++h) {
          T v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = T(__float2int_rn(P[16 * h + j])) * (T(1) << kk);
          group_reduce16(v, q, grp);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i >= per) break;
            const int rloc = rh * 64 + kRows * ch + 16 * h + j0 + i;
            const int ig = tr * a.tile_rows + rloc;
            if (writer && b < a.M && rloc < a.tile_rows && ig < a.K) {
              if (a.acc) atomicAdd(&a.acc[int64_t(ig) * a.M + b], int(v[i]));  // split-K partial (exact)
              else if (a.acc64) atomicAdd(&a.acc64[int64_t(ig) * a.M + b], (unsigned long long)(long long)v[i]);
              else a.dx[int64_t(ig) * a.ldx + b] = double(v[i]) * k_out;
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

__global__ void k_bwd_finalize(const BwdArgs a, int64_t M, int K) {
  const double k_out = bwd_k_out(a);
  const int64_t n = M * K;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / M, b = t - i * M;
    if (a.acc) {
      a.dx[i * a.ldx + b] = double(a.acc[t]) * k_out;
      a.acc[t] = 0;
    } else {
      a.dx[i * a.ldx + b] = double(static_cast<long long>(a.acc64[t])) * k_out;  // |total| < 2^53: exact
      a.acc64[t] = 0;
    }
  }
}

}  // namespace tc

bool launch_bwd_tc(xbs_core* c, int64_t M, double* d_dx, int64_t ldx, cudaStream_t st) {
  using namespace tc;
  const Geo& g = c->g;
  if ((g.R != 128 && g.R != 256) || (g.C != 128 && g.C != 256) || g.TPe > 16 || c->adc_b.passthrough) return false;
  // Exactness bounds per crossbar column tile of a unit (both error-sign
  // phases): fp32 P < 2^24 (wider layers split into column-tile ranges),
  // (plane, phase) combine and totals in int64 where they can pass 2^31
  // (the WIDE instantiation; see launch_fwd_tc)
  const double sw = (std::pow(2.0, g.wb) - 1) / (std::pow(2.0, g.db) - 1);
  const double per_tile = double(c->adc_b.maxc) * sw * 2.0;
  const int tcs_cap = int(16777215.0 / per_tile);
  if (tcs_cap < 1) return false;
  const bool wide = double(g.GC) * per_tile * (std::pow(2.0, g.Te) - 1) >= 2147483648.0;
  const int64_t rowsB = rows_bwd(M, g.TPe);
  CUtensorMap mA, mB;
  // A: K-major error planes, row pitch NB; narrow layers load 32 / 64-byte
  // boxes with the matching swizzle (the K = 32 steps never pass N)
  const int awid = std::min(g.NB, 128);
  if (!make_map(&mA, c->d_Ab, uint64_t(g.NB), uint64_t(2 * rowsB), uint32_t(awid), 128,
                awid == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : awid == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                            : CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  if (!make_map(&mB, c->d_digits, uint64_t(g.C), uint64_t(g.digits_bytes() / g.C), 128, 64)) return false;
  const int KB = g.C / 128;
  BwdArgs a{};
  a.wide = wide ? 1 : 0;
  a.GR = g.GR;
  a.GC = g.GC;
  a.S = g.S;
  a.db = g.db;
  a.TPe = g.TPe;
  a.abox = 128 * awid;
  a.a_sbo = uint32_t(8 * awid);                                // 8 rows of awid bytes
  a.a_layout = awid == 32 ? 6u : awid == 64 ? 4u : 2u;        // SWIZZLE_32B / 64B / 128B
  a.lg_grp = 1;
  while ((1 << a.lg_grp) < 2 * g.TPe) ++a.lg_grp;
  a.tile_rows = g.tile_rows;
  a.tile_cols = g.tile_cols;
  a.R = g.R;
  a.C = g.C;
  a.K = g.K;
  a.N = g.N;
  a.M = M;
  a.rowsB = rowsB;
  a.num_mbp = int(rowsB / 256);
  a.live = (g.tile_rows + 63) / 64;
  a.live_last = (g.K - (g.GR - 1) * g.tile_rows + 63) / 64;
  a.n_rb = (g.GR - 1) * a.live + a.live_last;
  a.nbase = a.num_mbp * a.n_rb;
  // small layers: split the crossbar column tiles of a unit across CTA pairs
  // (exact int32 totals, summed with atomics; see launch_fwd_tc)
  const int pairs = sm_count() / 2;
  a.ksplit = 1;
  if (2 * a.nbase <= pairs && g.GC > 1) a.ksplit = std::min(g.GC, pairs / a.nbase);
  a.ksplit = std::max(a.ksplit, (g.GC + tcs_cap - 1) / tcs_cap);
  a.tcs = (g.GC + a.ksplit - 1) / a.ksplit;
  a.ksplit = (g.GC + a.tcs - 1) / a.tcs;
  if (int64_t(a.nbase) * a.ksplit >= (int64_t{1} << 31)) return false;
  a.num_units = a.nbase * a.ksplit;
  a.f_nbase = make_fdiv(uint32_t(a.nbase));
  a.f_mbp = make_fdiv(uint32_t(a.num_mbp));
  a.f_nrb = make_fdiv(uint32_t(a.n_rb));
  a.f_live = make_fdiv(uint32_t(a.live));
  a.acc = nullptr;
  a.acc64 = nullptr;
  if (a.ksplit > 1) {
    void* buf = acc32(c, size_t(M) * g.K * (wide ? 8 : 4), st);
    if (!buf) return false;
    if (wide) a.acc64 = static_cast<unsigned long long*>(buf);
    else a.acc = static_cast<int*>(buf);
  }
  {  // sweep the larger operand once: A' (error planes) vs the conductance digits
    const double bytesA = 2.0 * double(rowsB) * g.NB, bytesB = double(g.digits_bytes()) / g.GR * (double(a.n_rb) / a.live);
    // an operand that fits in L2 (126 MB; use half) is re-read for free
    const double l2 = 64.0 * 1024 * 1024;
    const double costM = (bytesA <= l2 ? bytesA : bytesA * a.n_rb) + bytesB;  // M-blocks fastest
    const double costO = bytesA + (bytesB <= l2 ? bytesB : bytesB * a.num_mbp);        // other index fastest
    a.mfast = costM <= costO ? 1 : 0;
    a.hint = a.mfast && bytesA > l2 ? 1 : 0;  // as in launch_fwd_tc (C5 backward -5.3 %)
    if (std::getenv("XBS_NO_L2_HINTS")) a.hint = 0;  // A/B switch (perf experiments only)
  }
  a.F = c->F;
  a.vu = c->vu;
  a.ifs_fac = c->ifs_fac_b;
  a.lev_e = c->lev_e;
  a.adc_scaled = c->adc_scaled ? 1 : 0;
  a.sc = c->d_sc;
  a.adc = make_adc_const(c->adc_b, c->d_adc_tab_b);
  if (a.adc.unscale == 0.0f) return false;
  a.dx = d_dx;
  a.ldx = ldx;
  a.ctr = &c->d_sc->exact_path;
  // as launch_fwd_tc: rounds kept in step, 4 row blocks x pairs / 4 M-block
  // pairs per round (C5 backward: DRAM reads 152 -> 83 GB per launch,
  // 136.8 -> 131.5 ms)
  a.wsync = nullptr;
  a.grp = 1;
  a.hinta = a.hint;
  const bool trim_any = (g.N % g.tile_cols) != 0 || g.tile_cols <= g.C - 32 || (g.tile_rows % 64) != 0 ||
                        ((g.K - (g.GR - 1) * g.tile_rows) % 64) != 0;  // the TRIM instantiations (below)
  if (a.hint && !trim_any && !c->out_host && !std::getenv("XBS_NO_WAVE_SYNC")) {
    a.grp = std::getenv("XBS_WAVE_GROUP") ? std::max(1, std::atoi(std::getenv("XBS_WAVE_GROUP"))) : 4;
    a.hinta = a.grp > 1 && !std::getenv("XBS_WAVE_AHINT") ? 0 : 1;
    a.wsync = &c->d_sc->wave_sync[1];
    cudaMemsetAsync(a.wsync, 0, sizeof(unsigned int), st);
  }
  const int grid_ = 2 * std::min(a.num_units, sm_count() / 2);  // CTA pairs
  auto launch = [&](auto kern, int smem) {
    static const void* done[8];
    static int ndone = 0;
    bool seen = false;
    for (int k = 0; k < ndone; ++k) seen |= done[k] == reinterpret_cast<const void*>(kern);
    if (!seen) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (ndone < 8) done[ndone++] = reinterpret_cast<const void*>(kern);
    }
    kern<<<grid_, kThreads, smem, st>>>(mA, mB, a);
  };
  const bool trim = (g.N % g.tile_cols) != 0 || g.tile_cols <= g.C - 32 || (g.tile_rows % 64) != 0 ||
                    ((g.K - (g.GR - 1) * g.tile_rows) % 64) != 0;
  const int sel = (KB == 2 ? 4 : 0) + (trim ? 2 : 0) + (wide ? 1 : 0);
  switch (sel) {
    case 0: launch(k_bwd_tc<1, false, false>, bw::kSmem<1>); break;
    case 1: launch(k_bwd_tc<1, false, true>, bw::kSmem<1>); break;
    case 2: launch(k_bwd_tc<1, true, false>, bw::kSmem<1>); break;
    case 3: launch(k_bwd_tc<1, true, true>, bw::kSmem<1>); break;
    case 4: launch(k_bwd_tc<2, false, false>, bw::kSmem<2>); break;
    case 5: launch(k_bwd_tc<2, false, true>, bw::kSmem<2>); break;
    case 6: launch(k_bwd_tc<2, true, false>, bw::kSmem<2>); break;
    default: launch(k_bwd_tc<2, true, true>, bw::kSmem<2>); break;
  }
  if (a.acc || a.acc64) {
    const int64_t n = M * g.K;
    k_bwd_finalize<<<int(std::min<int64_t>((n + 255) / 256, 4 * sm_count())), 256, 0, st>>>(a, M, g.K);
    c->launches += 1;
  }
  return cudaPeekAtLastError() == cudaSuccess;
}

}  // namespace xbs
