// tcgen05 crossbar VMM kernels (K1 forward, K2 backward) for sm_100a.
//
// K1 (layers.cpp:246-283).  One CTA-persistent unit = (128 input bit-plane
// rows = 128/TPi batch rows x TPi planes, 128 device output columns of one
// crossbar tile column).  For every crossbar row tile tr, slice s and
// polarity p the MMA warp issues a K = 2*128 chain of tcgen05.mma kind::i8
// (M=128, N=256, K=32):
//     D[:, 0:128]   = A_bits . d0 + A_255 . d1   (lo digit pair of q)
//     D[:, 128:256] = A_bits . d2 + A_255 . d3   (hi digit pair of q)
// so the TMEM accumulator holds the exact column current of every
// (row, bit plane, column) split as hi*65025 + lo.  The K-extent of one
// accumulation is exactly one crossbar (128 rows): the epilogue then applies
// the ADC (exact, see xbs_tc_common.cuh) and the signed shift-add
// P += +-2^(s*db) * code in fp32 registers (exact integers < 2^24), double-
// buffered against the next chain in TMEM.  After the last tile the TPi
// bit-plane lanes of each batch row are combined as sum 2^k * P_k in int64
// and scaled once by k_out (layers.cpp:272-283), so y is bit-identical to the
// snapped oracle.
//
// Warp roles (320 threads, 1 CTA / SM): warp 0 TMA producer, warp 1 TMEM
// allocator + single-thread MMA issuer, warps 2..9 epilogue (warp w reads
// TMEM lanes 32*(w%4).. and column half (w-2)/4).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "xbs_internal.cuh"
#include "xbs_tc_common.cuh"

namespace xbs {
namespace tc {

constexpr int kEpiWarps = 16;                 // 4 per SM sub-partition
constexpr int kThreads = 64 + 32 * kEpiWarps;  // + TMA producer, MMA issuer
constexpr int kBStages = 2;
constexpr int kPlane = 128 * 128;          // one 128x128 u8 digit / bit box
constexpr int kBStage = 4 * kPlane;        // one k-block: d0 d2 | d1 d3
// KB = 128-column k-blocks per crossbar (C = 128 KB)
template <int KB> constexpr int kAStage = 2 * KB * kPlane;  // [dh][kb]
template <int KB> constexpr int kAStages = KB == 1 ? 2 : 1;
template <int KB> constexpr int kSmem = kAStages<KB> * kAStage<KB> + kBStages * kBStage + 1024 + 256;

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

AdcConst make_adc_const(const xbs_core* c) {
  AdcConst k{};
  const double cn = std::ldexp(1.0, c->adc.sh) / c->adc.i_fs * c->adc.maxc_d;  // codes per current unit
  k.c_lo = float(cn);
  k.c_hi = float(65025.0 * cn);
  // |x_fast - scaled| <= 3 2^-24 x (constants' rounding, FMUL, FFMA) with
  // x <= maxc + 1 wherever the code is not saturated; delta = 4x that.
  const double maxc = double(c->adc.maxc);
  const double delta = 4.0 * 3.0 * 0x1p-24 * (maxc + 1.0);
  k.thr = float(0.5 - delta);
  k.maxc = float(c->adc.maxc);
  k.maxc_i = c->adc.maxc;
  k.tab = c->d_adc_tab;
  return k;
}

}  // namespace tc

// ---------------------------------------------------------------------------
// K2 backward (layers.cpp:339-379).  Unit = (128 error bit-plane rows: 128 /
// (2 TPe) batch rows x TPe planes x {plus, minus} phase, 64 device rows of
// one crossbar row tile).  For each crossbar column tile tc and slice s one
// chain of K = 2 x 128 (tile columns, bits | 255*bits) computes, with the
// transposed tiles read K-major straight from the same digit planes,
//     D[:, p*128 + acc*64 + r] = sum_c v_phi[c] * q_acc(s, p, tr, tc; r, c)
// i.e. all four products vp.gp, vp.gn, vm.gp, vm.gn of the reference in one
// accumulator (phase in M, polarity in N).  The epilogue converts every one
// of them through the ADC and accumulates  +-2^(s db) * code  with sign
// +1 when phase == polarity (acc_pos) and -1 otherwise (acc_neg).
namespace tc {

struct BwdArgs {
  int GR, GC, S, db, TPe, tile_rows, R, C, K;
  int64_t M, rowsB;
  int num_mb, num_units;
  double F, vu, ifs_fac, lev_e;
  int adc_scaled;
  const DevScalars* sc;
  AdcConst adc;
  double* dx;
  unsigned long long* ctr;
};

constexpr int kBHalf = 64 * 128;  // one [64 rows][128 cols] digit box

template <int KB>
__global__ void __launch_bounds__(kThreads, 1)
    k_bwd_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, const BwdArgs a) {
  constexpr int kAStage = tc::kAStage<KB>, kAStages = tc::kAStages<KB>;
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
  uint64_t* t_empty = t_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], kEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int rhalves = a.R / 64;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------- TMA producer
      uint32_t as = 0, aph = 0, bs = 0, bph = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
        const int mb = u % a.num_mb, rb = u / a.num_mb;
        const int tr = rb / rhalves, rh = rb % rhalves;
        for (int tc = 0; tc < a.GC; ++tc) {
          mbar_wait_sleep(&a_empty[as], aph ^ 1);
          mbar_expect_tx(&a_full[as], kAStage);
#pragma unroll
          for (int dh = 0; dh < 2; ++dh)
#pragma unroll
            for (int kb = 0; kb < KB; ++kb)
              tma_load_2d(sA + as * kAStage + (dh * KB + kb) * kPlane, &mapA, &a_full[as], tc * a.C + kb * 128,
                          int(dh * a.rowsB) + mb * 128);
          if (++as == kAStages) { as = 0; aph ^= 1; }
          for (int s = 0; s < a.S; ++s)
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
            mbar_wait_sleep(&b_empty[bs], bph ^ 1);
            mbar_expect_tx(&b_full[bs], kBStage);
            uint8_t* dst = sB + bs * kBStage;
            // smem order [dh][p][acc][64 r][128 c]; digit d = 2*acc + dh
#pragma unroll
            for (int dh = 0; dh < 2; ++dh)
#pragma unroll
              for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int acc = 0; acc < 2; ++acc) {
                  const int row = (((((s * 2 + p) * a.GR + tr) * a.GC + tc) * 4) + 2 * acc + dh) * a.R + rh * 64;
                  tma_load_2d(dst + ((dh * 2 + p) * 2 + acc) * kBHalf, &mapB, &b_full[bs], kb * 128, row);
                }
            if (++bs == kBStages) { bs = 0; bph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_i8(128, 256, /*b_mn_major=*/false);
      uint32_t as = 0, aph = 0, bs = 0, bph = 0, ab = 0, abph = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
        for (int tc = 0; tc < a.GC; ++tc) {
          mbar_wait_sleep(&a_full[as], aph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + as * kAStage);
          for (int s = 0; s < a.S; ++s) {
            mbar_wait_sleep(&t_empty[ab], abph ^ 1);
            const uint32_t td = tmem + ab * 256;
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              mbar_wait_sleep(&b_full[bs], bph);
              tc_fence_after();
              const uint32_t b0 = smem_u32(sB + bs * kBStage);
#pragma unroll
              for (int dh = 0; dh < 2; ++dh)
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                  const uint64_t ad = sdesc(a0 + (dh * KB + kb) * kPlane + 32 * ks, 16, 1024, 2);
                  const uint64_t bd = sdesc(b0 + dh * 4 * kBHalf + 32 * ks, 16, 1024, 2);
                  umma_i8(td, ad, bd, idesc, (kb | dh | ks) != 0);
                }
              umma_commit(&b_empty[bs]);
              if (++bs == kBStages) { bs = 0; bph ^= 1; }
            }
            umma_commit(&t_full[ab]);
            if (++ab == 2) { ab = 0; abph ^= 1; }
          }
          umma_commit(&a_empty[as]);
          if (++as == kAStages) { as = 0; aph ^= 1; }
        }
      }
    }
  } else {  // ---------------------------------------------------- epilogue
    // Per chain a warp converts kRows = 16 rows x 2 polarities as four
    // 8-column chunks, TMEM loads software-pipelined as in K1.
    constexpr int kRows = 64 / (kEpiWarps / 4);  // output rows per epilogue warp
    static_assert(kRows == 16, "four 8-column chunks per chain");
    const int lg = warp & 3, ch = (warp - 2) >> 2;
    const int ml = 32 * lg + lane;
    const int phi = ml & 1;
    const uint32_t tl = tmem + (uint32_t(32 * lg) << 16) + kRows * ch;
    uint32_t ab = 0, abph = 0, exact = 0;
    bool pref = false;
    uint32_t lA[8], hA[8], lB[8], hB[8];
    const AdcConst k = a.adc;
    const double se = a.sc->se;
    const double step_e = se > 0 ? se / a.lev_e : 0.0;
    double k_out = step_e * a.F / a.vu;  // layers.cpp:375-377
    if (a.adc_scaled) k_out *= a.ifs_fac;
    const int nchain = a.GC * a.S;
    for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
      const int mb = u % a.num_mb, rb = u / a.num_mb;
      const int tr = rb / rhalves, rh = rb % rhalves;
      float P[kRows];
#pragma unroll
      for (int j = 0; j < kRows; ++j) P[j] = 0.f;
      for (int c = 0; c < nchain; ++c) {
        const int s = c % a.S;  // chains run tc-major, then slice
        const float w = float(1 << (s * a.db));
        const float wpos = phi == 0 ? w : -w;  // polarity 0 (gp): + for the plus phase
        const float wneg = phi == 1 ? w : -w;  // polarity 1 (gn): + for the minus phase
        const uint32_t ta = tl + ab * 256;
        if (!pref) {
          mbar_wait_sleep(&t_full[ab], abph);
          tc_fence_after();
          tmem_ld8(ta, lA);
          tmem_ld8(ta + 64, hA);
        }
        tmem_wait_ld();
        tmem_ld8(ta + 8, lB);
        tmem_ld8(ta + 64 + 8, hB);
        adc_conv8<0>(lA, hA, k, wpos, P, 0, exact);
        tmem_wait_ld();
        tmem_ld8(ta + 128, lA);
        tmem_ld8(ta + 128 + 64, hA);
        adc_conv8<0>(lB, hB, k, wpos, P, 8, exact);
        tmem_wait_ld();
        tmem_ld8(ta + 128 + 8, lB);
        tmem_ld8(ta + 128 + 64 + 8, hB);
        adc_conv8<0>(lA, hA, k, wneg, P, 0, exact);
        tmem_wait_ld();
        tmem_release(&t_empty[ab]);
        if (++ab == 2) { ab = 0; abph ^= 1; }
        pref = mbar_try(&t_full[ab], abph);
        if (pref) {
          tc_fence_after();
          tmem_ld8(tl + ab * 256, lA);
          tmem_ld8(tl + ab * 256 + 64, hA);
        }
        adc_conv8<0>(lB, hB, k, wneg, P, 8, exact);
      }
      // combine the 2*TPe (plane, phase) lanes of each batch row
      const int grp = 2 * a.TPe;
      const int kk = (ml % grp) >> 1;
      const int64_t b = int64_t(mb) * (128 / grp) + ml / grp;
#pragma unroll
      for (int j = 0; j < kRows; ++j) {
        long long v = (long long)__float2ll_rn(P[j]) << kk;
        for (int o = 1; o < grp; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const int rloc = rh * 64 + kRows * ch + j;
        const int ig = tr * a.tile_rows + rloc;
        if ((ml % grp) == 0 && b < a.M && rloc < a.tile_rows && ig < a.K) a.dx[int64_t(ig) * a.M + b] = double(v) * k_out;
      }
    }
    if (a.ctr) atomicAdd(&a.ctr[0], (unsigned long long)exact);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace tc

bool launch_bwd_tc(xbs_core* c, int64_t M, double* d_dx, cudaStream_t st) {
  using namespace tc;
  const Geo& g = c->g;
  if ((g.R != 128 && g.R != 256) || (g.C != 128 && g.C != 256) || g.TPe > 16 || c->adc.passthrough) return false;
  const double sw = (std::pow(2.0, g.wb) - 1) / (std::pow(2.0, g.db) - 1);
  if (double(g.GC) * c->adc.maxc * sw * 2.0 >= 16777216.0) return false;
  const int64_t rowsB = rows_bwd(M, g.TPe);
  CUtensorMap mA, mB;
  if (!make_map(&mA, c->d_Ab, uint64_t(g.NI), uint64_t(2 * rowsB), 128, 128)) return false;
  if (!make_map(&mB, c->d_digits, uint64_t(g.C), uint64_t(g.digits_bytes() / g.C), 128, 64)) return false;
  const int KB = g.C / 128;
  BwdArgs a{};
  a.GR = g.GR;
  a.GC = g.GC;
  a.S = g.S;
  a.db = g.db;
  a.TPe = g.TPe;
  a.tile_rows = g.tile_rows;
  a.R = g.R;
  a.C = g.C;
  a.K = g.K;
  a.M = M;
  a.rowsB = rowsB;
  a.num_mb = int(rowsB / 128);
  a.num_units = a.num_mb * (g.KI / 64);
  a.F = c->F;
  a.vu = c->vu;
  a.ifs_fac = c->ifs_fac;
  a.lev_e = c->lev_e;
  a.adc_scaled = c->adc_scaled ? 1 : 0;
  a.sc = c->d_sc;
  a.adc = make_adc_const(c);
  a.dx = d_dx;
  a.ctr = &c->d_sc->exact_path;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_bwd_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem<1>);
    cudaFuncSetAttribute(k_bwd_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem<2>);
    attr = true;
  }
  const int grid = std::min(a.num_units, sm_count());
  if (KB == 1) k_bwd_tc<1><<<grid, kThreads, kSmem<1>, st>>>(mA, mB, a);
  else k_bwd_tc<2><<<grid, kThreads, kSmem<2>, st>>>(mA, mB, a);
  return cudaPeekAtLastError() == cudaSuccess;
}

}  // namespace xbs
