// K3a: the digital weight gradient dW = x_values^T dy_q / grad_divisor
// (layers.cpp:304) as an exact integer outer product on tcgen05 kind::i8:
//     S[i, j] = sum_b xcode[b, i] * (plus[b, j] - minus[b, j])
// computed transposed, D[j, i]: the u8 plus and minus error magnitudes are
// two A operands (M = 128 columns j, MN-major), the u8 activation codes the
// B operand (N = 128 rows i, MN-major), two s32 TMEM accumulators (exact for
// batch <= 33025).  dW = ((S * sx) * step_e) / grad_divisor in fp64 (the
// snapped-mode contract), written row-major [i][j]: TMEM lane
// = column j, so each warp store covers 32 consecutive j (256 B) of a row.
//
// Unit = 128 columns j x 128 rows i x one slice of the batch (K loop over
// its 128-row blocks).  Deep, narrow im2col layers (C3/C4: up to 401408
// batch rows, K x N of one or two tiles) are split along the batch so every
// SM has work and every partial stays exact in s32 (<= 32768 rows x 255 x
// 255); the partials are added in int64 (atomics on S64) and k_dw_finalize
// applies the fp64 contract.  Shallow layers write dW directly.
// Warp roles as in the VMM kernels (TMA producer, MMA issuer, 8 epilogue
// warps); the TMEM accumulator pair is double buffered so the epilogue's
// stores overlap the next unit's MMAs.
#include <cuda.h>
#include <cmath>
#include <cuda_runtime.h>

#include "xbs_internal.cuh"
#include "xbs_tc_common.cuh"

namespace xbs {
namespace tc {

namespace dw {
constexpr int kThreads = 320;
constexpr int kStages = 4;
constexpr int kBox = 128 * 128;
constexpr int kStage = 3 * kBox;  // plus | minus | x codes
constexpr int kSmem = kStages * kStage + 1024 + 256;
}  // namespace dw

struct DwArgs {
  int K, N, num_ib, num_units, kblocks;
  int ntiles, kb_chunk;  // units = ntiles x batch chunks of kb_chunk 128-row blocks
  int NA;
  unsigned long long* S64;  // split mode: int64 partial sums [KA][NA]; nullptr: direct dW
  int64_t Mcap8;
  double sx, lev_e, gd;
  double rgd;  // 1 / gd when gd is a power of two (then x / gd == x * rgd exactly), else 0
  DevScalars* sc;
  double* dW;
};

// ((S * sx) * step_e) / gd; a power-of-two divisor (the
// usual grad_divisor = 1) is an exact multiply by its reciprocal
__device__ __forceinline__ double dw_value(long long S, double sx, double step_e, double gd, double rgd) {
  const double t = (double(S) * sx) * step_e;
  return rgd != 0.0 ? t * rgd : t / gd;
}

__global__ void __launch_bounds__(dw::kThreads, 1)
    k_dw_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapE, const DwArgs a) {
  using namespace dw;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* t_full = empty + kStages;
  uint64_t* t_empty = t_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 8);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      uint32_t st = 0, ph = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
        const int t = u % a.ntiles, chunk = u / a.ntiles;
        const int ib = t % a.num_ib, jb = t / a.num_ib;
        const int kb1 = min(a.kblocks, (chunk + 1) * a.kb_chunk);
        for (int kb = chunk * a.kb_chunk; kb < kb1; ++kb) {
          mbar_wait(&empty[st], ph ^ 1);
          mbar_expect_tx(&full[st], kStage);
          uint8_t* dst = smem + st * kStage;
          tma_load_2d(dst, &mapE, &full[st], jb * 128, kb * 128);
          tma_load_2d(dst + kBox, &mapE, &full[st], jb * 128, int(a.Mcap8) + kb * 128);
          tma_load_2d(dst + 2 * kBox, &mapA, &full[st], ib * 128, kb * 128);
          if (++st == kStages) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: A = plus / minus (MN-major, j), B = x codes (MN-major, i)
      constexpr uint32_t idesc = idesc_i8(128, 128, true) | (1u << 15);
      uint32_t st = 0, ph = 0, ab = 0, abph = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
        mbar_wait(&t_empty[ab], abph ^ 1);
        tc_fence_after();
        const uint32_t td = tmem + ab * 256;
        const int chunk = u / a.ntiles, kb0 = chunk * a.kb_chunk, kb1 = min(a.kblocks, kb0 + a.kb_chunk);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint32_t s0 = smem_u32(smem + st * kStage);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t bd = sdesc(s0 + 2 * kBox + 4096 * ks, kBox, 1024, 2);
#pragma unroll
            for (int pm = 0; pm < 2; ++pm) {
              const uint64_t ad = sdesc(s0 + pm * kBox + 4096 * ks, kBox, 1024, 2);
              umma_i8(td + pm * 128, ad, bd, idesc, (kb != kb0 || ks != 0));
            }
          }
          umma_commit(&empty[st]);
          if (++st == kStages) { st = 0; ph ^= 1; }
        }
        umma_commit(&t_full[ab]);
        if (++ab == 2) { ab = 0; abph ^= 1; }
      }
    }
  } else {  // epilogue
    const int lg = warp & 3, ch = (warp - 2) >> 2;
    const double se = a.sc->se;
    const double step_e = se > 0 ? se / a.lev_e : 0.0;
    bool nonfinite = false;  // scale_gradient's finiteness check (update.cpp:18-19), raised at apply time
    uint32_t ab = 0, abph = 0;
    for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
      const int t = u % a.ntiles;
      const int ib = t % a.num_ib, jb = t / a.num_ib;
      const int j = jb * 128 + 32 * lg + lane;
      mbar_wait(&t_full[ab], abph);
      tc_fence_after();
      const uint32_t ta = tmem + (uint32_t(32 * lg) << 16) + ab * 256 + 64 * ch;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t pv[16], mv[16];
        tmem_ld16(ta + 16 * q, pv);
        tmem_ld16(ta + 128 + 16 * q, mv);
        tmem_wait_ld();
        if (q == 3) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&t_empty[ab]);
        }
        const int i0 = ib * 128 + 64 * ch + 16 * q;
        if (j < a.N) {
#pragma unroll
          for (int ii = 0; ii < 16; ++ii) {
            const int S = int(pv[ii]) - int(mv[ii]);
            if (i0 + ii < a.K) {
              if (a.S64) {
                if (S != 0) atomicAdd(&a.S64[int64_t(i0 + ii) * a.NA + j], (unsigned long long)(long long)S);
              } else {
                const double v = dw_value(S, a.sx, step_e, a.gd, a.rgd);
                nonfinite |= !isfinite(v);
                a.dW[int64_t(i0 + ii) * a.N + j] = v;
              }
            }
          }
        }
      }
      if (++ab == 2) { ab = 0; abph ^= 1; }
    }
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(&a.sc->dw_nonfinite, 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// Split mode: dW = ((S * sx) * step_e) / grad_divisor from the int64 sums,
// then S64 is cleared for the next call.
__global__ void k_dw_finalize(int K, int N, int NA, double sx, double lev_e, double gd, double rgd,
                              DevScalars* sc, unsigned long long* __restrict__ S64, double* __restrict__ dW) {
  const double se = sc->se;
  const double step_e = se > 0 ? se / lev_e : 0.0;
  const int64_t n = int64_t(K) * N;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / N), j = int(t % N);
    unsigned long long* p = &S64[int64_t(i) * NA + j];
    const long long S = (long long)*p;
    *p = 0ull;
    const double v = dw_value(S, sx, step_e, gd, rgd);
    if (!isfinite(v)) sc->dw_nonfinite = 1;
    dW[t] = v;
  }
}

}  // namespace tc

bool launch_dw_tc(xbs_core* c, int64_t M, double grad_divisor, cudaStream_t st) {
  using namespace tc;
  if (!c->d_xc8 || !c->d_e8 || M == 0) return false;
  const int64_t Mp = ((M + 127) / 128) * 128;
  CUtensorMap mA, mE;
  if (!make_map_u8(&mA, c->d_xc8, uint64_t(c->KA), uint64_t(Mp), 128, 128)) return false;
  if (!make_map_u8(&mE, c->d_e8, uint64_t(c->NA), uint64_t(2 * c->M_cap8), 128, 128)) return false;
  DwArgs a{};
  a.K = c->g.K;
  a.N = c->g.N;
  a.num_ib = c->KA / 128;
  a.ntiles = a.num_ib * (c->NA / 128);
  a.kblocks = int(Mp / 128);
  a.NA = c->NA;
  // batch chunks: exact s32 partials (<= 256 blocks = 32768 rows) and at
  // least ~2 units per SM when the K x N tiles alone cannot fill the GPU
  const int want = std::max((a.kblocks + 255) / 256, (2 * num_sms() + a.ntiles - 1) / a.ntiles);
  const int nchunks = std::max(1, std::min(a.kblocks, want));
  a.kb_chunk = (a.kblocks + nchunks - 1) / nchunks;
  const int nch = (a.kblocks + a.kb_chunk - 1) / a.kb_chunk;
  a.num_units = a.ntiles * nch;
  a.S64 = nullptr;
  if (nch > 1) {
    const size_t bytes = size_t(c->KA) * c->NA * 8;
    if (c->S64_bytes < bytes) {
      cudaFree(c->d_S64);
      c->d_S64 = nullptr;
      c->S64_bytes = 0;
      if (cudaMalloc(&c->d_S64, bytes) != cudaSuccess) {
        c->d_S64 = nullptr;
        (void)cudaGetLastError();  // the SIMT dW runs instead; do not leave the error pending
        return false;
      }
      cudaMemsetAsync(c->d_S64, 0, bytes, st);
      c->S64_bytes = bytes;
      ++c->gen;
    }
    a.S64 = c->d_S64;
  }
  a.Mcap8 = c->M_cap8;
  a.sx = c->sx;
  a.lev_e = c->lev_e;
  a.gd = grad_divisor;
  {
    int e;
    const double m = std::frexp(grad_divisor, &e);  // gd = m 2^e, m = 0.5 for a power of two
    a.rgd = (std::isfinite(grad_divisor) && std::fabs(m) == 0.5) ? 1.0 / grad_divisor : 0.0;
    if (a.rgd != 0.0 && (!std::isfinite(a.rgd) || std::fabs(std::frexp(a.rgd, &e)) != 0.5)) a.rgd = 0.0;
  }
  a.sc = c->d_sc;
  a.dW = c->d_dW;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, dw::kSmem);
    attr = true;
  }
  const int grid = std::min(a.num_units, num_sms());
  k_dw_tc<<<grid, dw::kThreads, dw::kSmem, st>>>(mA, mE, a);
  if (a.S64) {
    const int64_t n = int64_t(c->g.K) * c->g.N;
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
    c->launches += 1;  // the finalize pass (the caller counts k_dw_tc)
    k_dw_finalize<<<blocks, 256, 0, st>>>(c->g.K, c->g.N, c->NA, c->sx, c->lev_e, grad_divisor, a.rgd, c->d_sc,
                                          c->d_S64, c->d_dW);
  }
  return cudaPeekAtLastError() == cudaSuccess;
}

}  // namespace xbs
