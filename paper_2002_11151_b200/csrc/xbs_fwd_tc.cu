// K1: tcgen05 forward crossbar VMM (layers.cpp:246-283) for sm_100a.
//
// Unit = (two 128-row M-blocks of input bit-plane rows [b * TPi + k],
//         64 device output columns of one crossbar tile column).
// For every crossbar row tile tr, slice s and polarity p the MMA thread
// issues, per M-block, a K = 2 x R chain of tcgen05.mma.kind::i8
// (M=128, N=128, K=32) against the SAME B tile:
//     D[:,  0: 64] = A_bits . d0 + A_255 . d1    (lo digit pair of q)
//     D[:, 64:128] = A_bits . d2 + A_255 . d3    (hi digit pair of q)
// i.e. the exact column current of every (row, bit plane, column) split as
// hi * 65025 + lo in s32 TMEM accumulators.  The accumulation K-extent is
// exactly one crossbar (R = 128 or 256 rows, one or two k-blocks); the
// epilogue then applies the ADC (fp32 fast path + exact threshold fix-up,
// xbs_tc_common.cuh) and the signed shift-add P += +-2^(s db) * code.  The
// B tile (4 digit planes x 128 rows x 64 columns, 32 KB, SW64) is shared by
// both M-blocks (N = 128 keeps an MMA's 8 KB of SMEM operand reads within
// the 128 B/clk SMEM port).  After the last tile the TPi bit-plane lanes of
// each batch row are combined in int64 as sum_k 2^k P_k and scaled once by
// k_out (layers.cpp:272-283).
//
// Scheduling: persistent CTAs take units round-robin; when the last wave
// would leave SMs idle (C2-4096: 512 units = 3.46 waves on 148 SMs), its
// units are split into single-M-block half units (3.5 waves instead of 4).
// Column blocks made only of tile padding are never scheduled (C3's N = 16
// / 32 layers compute 64 of a padded 128-column tile).
//
// Roles (576 threads, 1 CTA / SM): warp 0 TMA producer, warp 1 TMEM
// allocator + MMA issuer, warps 2..17 epilogue: warp w reads TMEM lanes
// 32 (w % 4).., M-block ((w-2)/4) & 1, columns 32 ((w-2)/8)...
// Pipelines: A (64 KB per k-block: 2 M-blocks x {bits, 255 bits}) x 2 stages
// (1 for 256-row crossbars), B (32 KB) x 3 stages, TMEM accumulators
// (2 M-blocks x 128 columns) x 2 buffers.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>

#include "xbs_internal.cuh"
#include "xbs_tc_common.cuh"

namespace xbs {
namespace tc {

namespace fw {
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kCW = 64;               // device columns per unit
constexpr int kABox = 128 * 128;      // 128 rows x 128 B (one k-block), SW128
constexpr int kBBox = 128 * kCW;      // 128 crossbar rows x 64 columns, SW64
constexpr int kBStage = 4 * kBBox;    // one k-block of the 4 digit planes
constexpr int kBStages = 3;
constexpr int kTBufs = 2;             // TMEM buffers of 2 M-blocks x 128 columns
// KB = 128-row k-blocks per crossbar (1: 128-row tiles, 2: 256-row tiles)
template <int KB> constexpr int kAStage = 4 * KB * kABox;  // [mb][dh][kb]
template <int KB> constexpr int kAStages = KB == 1 ? 2 : 1;
template <int KB> constexpr int kSmem = kAStages<KB> * kAStage<KB> + kBStages * kBStage + 1024 + 256;
}  // namespace fw

struct FwdArgs {
  int GR, GC, S, db, TPi, tile_cols, C, R, N;
  int live;  // 64-column units per tile column that hold logical columns
  int64_t M, rowsF;
  int num_mbp, num_units;
  int n_full, sched;  // units [n_full, num_units) run as 2 half units each
  double k_out;
  AdcConst adc;
  double* y;
  unsigned long long* ctr;
};

struct Unit {
  int mbp, nb, only;  // only: -1 both M-blocks, else the single M-block
};
__device__ __forceinline__ Unit unit_of(int u, const FwdArgs& a) {
  if (u < a.n_full) return {u % a.num_mbp, u / a.num_mbp, -1};
  const int v = u - a.n_full, base = a.n_full + (v >> 1);
  return {base % a.num_mbp, base / a.num_mbp, v & 1};
}

template <int KB>
__global__ void __launch_bounds__(fw::kThreads, 1)
    k_fwd_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, const FwdArgs a) {
  using namespace fw;
  constexpr int kAStage = fw::kAStage<KB>, kAStages = fw::kAStages<KB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kAStages * kAStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kBStages * kBStage);
  uint64_t* a_full = bars;
  uint64_t* a_empty = a_full + kAStages;
  uint64_t* b_full = a_empty + kAStages;
  uint64_t* b_empty = b_full + kBStages;
  uint64_t* t_full = b_empty + kBStages;    // [buffer][M-block]
  uint64_t* t_empty = t_full + 2 * kTBufs;  // [buffer][M-block]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2 * kTBufs);

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
    for (int i = 0; i < 2 * kTBufs; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], kEpiWarps / 2);
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

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------- TMA producer
      uint32_t as = 0, aph = 0, bs = 0, bph = 0;
      for (int u = blockIdx.x; u < a.sched; u += gridDim.x) {
        const Unit un = unit_of(u, a);
        const int tc = un.nb / a.live, h = un.nb % a.live;
        for (int tr = 0; tr < a.GR; ++tr) {
          mbar_wait(&a_empty[as], aph ^ 1);
          mbar_expect_tx(&a_full[as], un.only < 0 ? kAStage : kAStage / 2);
#pragma unroll
          for (int mb = 0; mb < 2; ++mb) {
            if (un.only >= 0 && mb != un.only) continue;
#pragma unroll
            for (int dh = 0; dh < 2; ++dh)
#pragma unroll
              for (int kb = 0; kb < KB; ++kb)
                tma_load_2d(sA + as * kAStage + ((mb * 2 + dh) * KB + kb) * kABox, &mapA, &a_full[as],
                            tr * a.R + kb * 128, int(dh * a.rowsF) + (2 * un.mbp + mb) * 128);
          }
          if (++as == kAStages) { as = 0; aph ^= 1; }
          for (int s = 0; s < a.S; ++s)
            for (int p = 0; p < 2; ++p)
#pragma unroll
              for (int kb = 0; kb < KB; ++kb) {
                mbar_wait(&b_empty[bs], bph ^ 1);
                mbar_expect_tx(&b_full[bs], kBStage);
                const int row0 = ((((s * 2 + p) * a.GR + tr) * a.GC + tc) * 4) * a.R + kb * 128;
                uint8_t* dst = sB + bs * kBStage;  // [dh][acc]: d0 d2 | d1 d3
                tma_load_2d(dst + 0 * kBBox, &mapB, &b_full[bs], h * kCW, row0 + 0 * a.R);
                tma_load_2d(dst + 1 * kBBox, &mapB, &b_full[bs], h * kCW, row0 + 2 * a.R);
                tma_load_2d(dst + 2 * kBBox, &mapB, &b_full[bs], h * kCW, row0 + 1 * a.R);
                tma_load_2d(dst + 3 * kBBox, &mapB, &b_full[bs], h * kCW, row0 + 3 * a.R);
                if (++bs == kBStages) { bs = 0; bph ^= 1; }
              }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_i8(128, 2 * kCW, /*b_mn_major=*/true);
      uint32_t as = 0, aph = 0, bs = 0, bph = 0, ab = 0, abph = 0;
      for (int u = blockIdx.x; u < a.sched; u += gridDim.x) {
        const int only = unit_of(u, a).only;
        for (int tr = 0; tr < a.GR; ++tr) {
          mbar_wait(&a_full[as], aph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + as * kAStage);
          for (int sp = 0; sp < 2 * a.S; ++sp) {
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              mbar_wait(&b_full[bs], bph);
              const uint32_t b0 = smem_u32(sB + bs * kBStage);
#pragma unroll
              for (int mb = 0; mb < 2; ++mb) {
                if (only >= 0 && mb != only) continue;  // a half unit is the CTA's last
                if (kb == 0) mbar_wait(&t_empty[ab * 2 + mb], abph ^ 1);
                tc_fence_after();
#pragma unroll
                for (int dh = 0; dh < 2; ++dh)
#pragma unroll
                  for (int ks = 0; ks < 4; ++ks) {
                    // A: K-major SW128 (LBO 16, SBO 1024); B: MN-major SW64,
                    // the lo / hi 64-column boxes kBBox apart (LBO), 8-row
                    // K groups 512 B apart (SBO), 32 K rows per MMA = 2 KB
                    const uint64_t ad = sdesc(a0 + ((mb * 2 + dh) * KB + kb) * kABox + 32 * ks, 16, 1024, 2);
                    const uint64_t bd = sdesc(b0 + dh * 2 * kBBox + 2048 * ks, kBBox, 512, 4);
                    umma_i8(tmem + ab * 256 + mb * 128, ad, bd, idesc, (kb | dh | ks) != 0);
                  }
                if (kb == KB - 1) umma_commit(&t_full[ab * 2 + mb]);
              }
              umma_commit(&b_empty[bs]);
              if (++bs == kBStages) { bs = 0; bph ^= 1; }
            }
            if (++ab == kTBufs) { ab = 0; abph ^= 1; }
          }
          umma_commit(&a_empty[as]);
          if (++as == kAStages) { as = 0; aph ^= 1; }
        }
      }
    }
  } else {  // ---------------------------------------------------- epilogue
    const int lg = warp & 3, sel = (warp - 2) >> 2;
    const int mb = sel & 1, ch = sel >> 1;  // M-block, 32-column half
    const int ml = 32 * lg + lane;
    uint32_t ab = 0, abph = 0, exact = 0;
    const AdcConst k = a.adc;
    for (int u = blockIdx.x; u < a.sched; u += gridDim.x) {
      const Unit un = unit_of(u, a);
      if (un.only >= 0 && un.only != mb) break;  // half unit of the other M-block (last unit)
      const int mbp = un.mbp, nb = un.nb;
      float P[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) P[j] = 0.f;
      for (int tr = 0; tr < a.GR; ++tr)
        for (int s = 0; s < a.S; ++s)
          for (int p = 0; p < 2; ++p) {
            const float w = p == 0 ? float(1 << (s * a.db)) : -float(1 << (s * a.db));
            mbar_wait(&t_full[ab * 2 + mb], abph);
            tc_fence_after();
            const uint32_t ta = tmem + (uint32_t(32 * lg) << 16) + ab * 256 + mb * 128 + 32 * ch;
            adc_chunk16s(ta, ta + kCW, k, w, P, 0, exact, nullptr);
            adc_chunk16s(ta + 16, ta + kCW + 16, k, w, P, 16, exact, &t_empty[ab * 2 + mb]);
            if (++ab == kTBufs) { ab = 0; abph ^= 1; }
          }
      // combine the TPi bit-plane lanes of each batch row: total = sum 2^k P_k
      const int kk = ml % a.TPi;
      const int64_t b = (int64_t(2 * mbp + mb) * 128 + ml) / a.TPi;
      const int tc = nb / a.live, h = nb % a.live;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        long long v = (long long)__float2ll_rn(P[j]) << kk;
        for (int o = 1; o < a.TPi; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const int c = h * kCW + 32 * ch + j;
        const int jg = tc * a.tile_cols + c;
        if (kk == 0 && b < a.M && c < a.tile_cols && jg < a.N) a.y[int64_t(jg) * a.M + b] = double(v) * a.k_out;
      }
    }
    if (a.ctr) atomicAdd(&a.ctr[0], (unsigned long long)exact);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace tc

bool launch_fwd_tc(xbs_core* c, int64_t M, double* d_y, cudaStream_t st) {
  using namespace tc;
  const Geo& g = c->g;
  if ((g.R != 128 && g.R != 256) || g.TPi > 16 || c->adc.passthrough) return false;
  // fp32 P accumulators must stay exact: GR * maxc * sum_s 2^(s db) < 2^24
  const double sw = (std::pow(2.0, g.wb) - 1) / (std::pow(2.0, g.db) - 1);
  if (double(g.GR) * c->adc.maxc * sw >= 16777216.0) return false;
  const int64_t rowsF = rows_fwd(M, g.TPi);
  CUtensorMap mA, mB;
  if (!make_map_u8(&mA, c->d_Af, uint64_t(g.KI), uint64_t(2 * rowsF), 128, 128, 128)) return false;
  if (!make_map_u8(&mB, c->d_digits, uint64_t(g.C), uint64_t(g.digits_bytes() / g.C), fw::kCW, 128, 64))
    return false;
  FwdArgs a{};
  a.GR = g.GR;
  a.GC = g.GC;
  a.S = g.S;
  a.db = g.db;
  a.TPi = g.TPi;
  a.tile_cols = g.tile_cols;
  a.C = g.C;
  a.R = g.R;
  a.N = g.N;
  a.live = (g.tile_cols + fw::kCW - 1) / fw::kCW;
  a.M = M;
  a.rowsF = rowsF;
  a.num_mbp = int(rowsF / 256);
  a.num_units = a.num_mbp * g.GC * a.live;
  a.k_out = c->k_out_fwd;
  a.adc = make_adc_const(c);
  a.y = d_y;
  a.ctr = &c->d_sc->exact_path;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fwd_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, fw::kSmem<1>);
    cudaFuncSetAttribute(k_fwd_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, fw::kSmem<2>);
    attr = true;
  }
  const int grid = std::min(a.num_units, num_sms());
  // last-wave balancing: leftover full units run as 2 single-M-block halves
  // when those all fit in one extra wave
  const int rounds = a.num_units / grid, rem = a.num_units - rounds * grid;
  a.n_full = a.num_units;
  a.sched = a.num_units;
  if (rem > 0 && 2 * rem <= grid) {
    a.n_full = rounds * grid;
    a.sched = a.n_full + 2 * rem;
  }
  if (g.R == 128) k_fwd_tc<1><<<grid, fw::kThreads, fw::kSmem<1>, st>>>(mA, mB, a);
  else k_fwd_tc<2><<<grid, fw::kThreads, fw::kSmem<2>, st>>>(mA, mB, a);
  return cudaPeekAtLastError() == cudaSuccess;
}

}  // namespace xbs
