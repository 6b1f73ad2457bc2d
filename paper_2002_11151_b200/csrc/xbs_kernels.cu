// Bandwidth-bound kernels of the hot path (SIMT, sm_100a):
//   map_weights   mapping.cpp:83-131      W -> per-slice signed master
//   regen/update  update.cpp:43-88 fused with mapping.cpp:28-58 (variation),
//                 aam.cpp:14-31 (AAM), the 2^-e snap and radix-255 digit
//                 emission, implied-weight / |dW| maxima (layers.cpp:384-386)
//   prep_x/_dy    tensor.cpp:8-51 quantisers + DAC bit-planes (layers.cpp:236-241,
//                 316-331)
//   dw            layers.cpp:304 as the exact integer contract
//   vmm_simt      exact SIMT forward/backward (cross-check kernel; also the
//                 pass-through-ADC path, layers.cpp:202)
//   ideal         fully-ideal fast path (layers.cpp:226, 307)
// Compiled with --fmad=false: every fp64 expression rounds exactly as the
// reference's x86-64 code does (no contraction).
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "xbs_internal.cuh"
#include "xbs_rng.cuh"
#include "xbs_tc_common.cuh"

namespace xbs {

__device__ __forceinline__ void atomic_max_pos(unsigned long long* p, double v) {
  atomicMax(p, (unsigned long long)__double_as_longlong(v));
}

template <class T>
__device__ __forceinline__ T warp_max(T v) {
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ------------------------------------------------- conductance conversion
// aam.cpp:5-12: series path resistance of tile position (r, c), summed left
// to right like the reference.
__device__ __forceinline__ double aam_rpath(const RegenP& rp, const Geo& g, int r, int c) {
  return rp.r_source + double(c + 1) * rp.r_row + double(g.tile_rows - r) * rp.r_col + rp.r_sense;
}

// mapping.cpp:39-58 (polarity split, variation) + aam.cpp:14-31 + snap of one
// device (slice s, polarity p, padded index idx = i * Np + j) from its master
// value u.  __drcp_rn is the correctly rounded 1/x (= the reference's 1.0 / x)
// and gv * 2^e is exact (= ldexp), so q is bit-identical to the oracle's.
__device__ __forceinline__ uint32_t convert_q(const RegenP& rp, double u, int s, int p, uint64_t idx,
                                              double rpath) {
  double gv = (p == 0 ? fmax(u, 0.0) : fmax(-u, 0.0)) + rp.g_min;
  if (rp.sigma != 0.0) gv = fmin(gv * rp.varm[(uint64_t(s) * 2 + p) * rp.kpnp + idx], rp.g_max);
  if (rp.aam) {
    if (gv == 0.0) gv = 0.0;
    else if (rpath != 0.0) gv = __drcp_rn(__dadd_rn(__drcp_rn(gv), rpath));
  }
  return __double2uint_rn(__dmul_rn(gv, rp.snap_scale));  // nearbyint(ldexp(gv, e))
}

// mapping.cpp:28-35: m = max(1 + sigma * N(0, 1), 1e-12), keyed by
// (seed, 2 s + p, padded device index), computed once per core.
__global__ void k_varm(Geo g, RegenP rp, double* __restrict__ varm) {
  const uint64_t n = uint64_t(g.S) * 2 * rp.kpnp;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n; t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t sp = t / rp.kpnp, idx = t - sp * rp.kpnp;
    double m = 1.0 + rp.sigma * rng_gaussian(rng_key(rp.vseed, sp, idx, 0));
    varm[t] = m > 1e-12 ? m : 1e-12;
  }
}

void launch_varm(const xbs_core* c, cudaStream_t st) {
  const uint64_t n = uint64_t(c->g.S) * 2 * c->rp.kpnp;
  const int blocks = int(std::min<uint64_t>((n + 255) / 256, 148 * 32));
  k_varm<<<blocks, 256, 0, st>>>(c->g, c->rp, c->d_varm);
}

// Compile-time specialised conversion for the update kernel.  VAR: sigma
// != 0; AAM: AAM engine with a non-zero path resistance.  g_min > 0
// (CrossbarConfig::validate) and the variation multiplier >= 1e-12, so gv
// is never 0 here; max(+-u, 0) + g_min is written as a select (an exact -0
// or +0 adds to g_min identically).
template <bool VAR, bool AAM>
__device__ __forceinline__ uint32_t convert_qt(const RegenP& rp, double u, int s, int p, uint64_t idx,
                                               double rpath) {
  const double up = p == 0 ? u : -u;
  double gv = (up > 0.0 ? up : 0.0) + rp.g_min;
  if constexpr (VAR) gv = fmin(gv * __ldg(&rp.varm[(uint64_t(s) * 2 + p) * rp.kpnp + idx]), rp.g_max);
  if constexpr (AAM) gv = __drcp_rn(__dadd_rn(__drcp_rn(gv), rpath));
  return __double2uint_rn(__dmul_rn(gv, rp.snap_scale));
}

__device__ __forceinline__ void store_digits(uint8_t* digits, const Geo& g, int s, int p, int i, int j,
                                             uint32_t q) {
  const int tr = i / g.tile_rows, r = i % g.tile_rows, tc = j / g.tile_cols, c = j % g.tile_cols;
  const uint32_t lo = q % 65025u, hi = q / 65025u;
  const size_t off = size_t(r) * g.C + c;
  digits[g.tile_digit_offset(s, p, tr, tc, 0) + off] = uint8_t(lo % 255u);
  digits[g.tile_digit_offset(s, p, tr, tc, 1) + off] = uint8_t(lo / 255u);
  digits[g.tile_digit_offset(s, p, tr, tc, 2) + off] = uint8_t(hi);
}

__device__ __forceinline__ uint32_t load_q(const uint8_t* digits, const Geo& g, int s, int p, int tr, int tc,
                                           int r, int c) {
  const size_t off = size_t(r) * g.C + c;
  const size_t base = g.tile_digit_offset(s, p, tr, tc, 0) + off, ps = g.plane_bytes();
  const uint32_t d0 = digits[base], d1 = digits[base + ps], d2 = digits[base + 2 * ps];
  return (d0 + 255u * d1) + 65025u * d2;
}

// -------------------------------------------------------------- map_weights
__global__ void __launch_bounds__(256) k_absmax(const double* __restrict__ x, int64_t n,
                                                unsigned long long* out) {
  // four 16-byte loads in flight per thread
  double m = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (reinterpret_cast<uintptr_t>(x) & 15) {  // caller's device pointer not 16-byte aligned
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += stride) m = fmax(m, fabs(x[k]));
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomic_max_pos(out, m);
    return;
  }
  const int64_t n2 = n / 2;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  for (; k + 3 * stride < n2; k += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(x2 + k + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) m = fmax(m, fmax(fabs(v[u].x), fabs(v[u].y)));
  }
  for (; k < n2; k += stride) {
    const double2 v = __ldg(x2 + k);
    m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) m = fmax(m, fabs(x[n - 1]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_pos(out, m);
}

void launch_absmax(const double* d_x, int64_t n, unsigned long long* out_bits, cudaStream_t st) {
  int blocks = int(std::min<int64_t>((n / 2 + 255) / 256, 148 * 8));
  if (blocks < 1) blocks = 1;
  k_absmax<<<blocks, 256, 0, st>>>(d_x, n, out_bits);
}

// mapping.cpp:104-129.  W col-major K x N (ld = K); writes every padded
// master element (0 outside the logical region).
__global__ void k_map_weights(const double* __restrict__ W, Geo g, double scale, uint64_t q_levels,
                              uint64_t d_levels, double level_step, double* __restrict__ master) {
  const int64_t n = int64_t(g.Kp) * g.Np;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / g.Np), j = int(t % g.Np);
    uint64_t q = 0;
    double sign = 1.0;
    if (i < g.K && j < g.N) {
      const double w = W[int64_t(j) * g.K + i];
      const double mag = fabs(w) / scale * double(q_levels);
      q = uint64_t(llround(mag));
      if (q > q_levels) q = q_levels;
      sign = w < 0 ? -1.0 : 1.0;
    }
    for (int s = 0; s < g.S; ++s) {
      const uint64_t digit = (q >> (s * g.db)) & d_levels;
      master[(size_t(s) * g.Kp + i) * g.Np + j] = digit != 0 ? sign * (double(digit) * level_step) : 0.0;
    }
  }
}

void launch_map_weights(const xbs_core* c, const double* d_W, cudaStream_t st) {
  const int64_t n = int64_t(c->g.Kp) * c->g.Np;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 32));
  k_map_weights<<<blocks, 256, 0, st>>>(d_W, c->g, c->layer_scale, (uint64_t{1} << c->g.wb) - 1,
                                        (uint64_t{1} << c->g.db) - 1, c->level_step, c->d_master);
}

// regenerate() (layers.cpp:129-179) over every padded device, all slices and
// polarities.
__global__ void k_regen_all(Geo g, RegenP rp, const double* __restrict__ master, uint8_t* __restrict__ digits) {
  const int64_t n = int64_t(g.Kp) * g.Np;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / g.Np), j = int(t % g.Np);
    const double rpath = rp.aam ? aam_rpath(rp, g, i % g.tile_rows, j % g.tile_cols) : 0.0;
    for (int s = 0; s < g.S; ++s) {
      const double u = master[(size_t(s) * g.Kp + i) * g.Np + j];
      for (int p = 0; p < 2; ++p)
        store_digits(digits, g, s, p, i, j, convert_q(rp, u, s, p, uint64_t(i) * g.Np + j, rpath));
    }
  }
}

void launch_regen_all(const xbs_core* c, cudaStream_t st) {
  const int64_t n = int64_t(c->g.Kp) * c->g.Np;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 32));
  k_regen_all<<<blocks, 256, 0, st>>>(c->g, c->rp, c->d_master, c->d_digits);
}

// ----------------------------------------------------------- apply_updates
// K3b: update.cpp:43-88 for every slice of a logical weight (i, j), the
// regeneration of both devices of every slice (layers.cpp:388 ->
// mapping.cpp:39-58 variation, aam.cpp:14-31, snap, radix-255 digits) and
// the implied-weight Horner (mapping.cpp:70-81) for the |W| statistic.
//
// Layout for HBM: blockIdx.y walks rows i, each thread owns JPT consecutive
// columns j (vector dW / master loads, all S slices loaded up front; each
// digit plane row segment written as one packed JPT-byte store so every
// 32-byte sector is written whole -- a partial sector costs a DRAM read).
// Compile-time flags strip the variation / non-linearity / noise code when
// those are off.  With sigma == 0 the inactive polarity of each device sits
// exactly at g_min, whose snapped conductance depends on the tile position
// only (qmin table), so one conversion per device and slice suffices.
template <int JPT>
struct VecT;
template <>
struct VecT<2> {
  using D = double2;
  using Q = uint2;
  using B = uint16_t;
};
template <>
struct VecT<4> {
  using D = double4;
  using Q = uint4;
  using B = uint32_t;
};

template <int JPT>
__device__ __forceinline__ void ld_vec(const double* p, double (&v)[JPT]) {
  const typename VecT<JPT>::D t = *reinterpret_cast<const typename VecT<JPT>::D*>(p);
  if constexpr (JPT == 2) {
    v[0] = t.x;
    v[1] = t.y;
  } else {
    v[0] = t.x;
    v[1] = t.y;
    v[2] = t.z;
    v[3] = t.w;
  }
}
template <int JPT>
__device__ __forceinline__ void st_vec(double* p, const double (&v)[JPT]) {
  typename VecT<JPT>::D t;
  if constexpr (JPT == 2) {
    t.x = v[0];
    t.y = v[1];
  } else {
    t.x = v[0];
    t.y = v[1];
    t.z = v[2];
    t.w = v[3];
  }
  *reinterpret_cast<typename VecT<JPT>::D*>(p) = t;
}

template <int S_T, int JPT, bool VAR, bool NL, bool NOISE, bool AAM, bool CONV = true>
__global__ void __launch_bounds__(256) k_update(Geo g, RegenP rp, UpdP up, const double* __restrict__ dW,
                                                double* __restrict__ master, uint8_t* __restrict__ digits,
                                                DevScalars* sc, const uint32_t* __restrict__ qmin) {
  constexpr int S = S_T;
  if (sc->dw_nonfinite) {  // scale_gradient throws before touching the master (update.cpp:18-19)
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0) atomicOr(&sc->err_flag, 2);
    return;
  }
  const double range = rp.range;
  double wmax = 0.0, dwmax = 0.0;
  const int j0 = JPT * (blockIdx.x * blockDim.x + threadIdx.x);
  if (j0 < g.N) {
    // column-only terms, hoisted out of the row loop (a block covers
    // blockDim.y rows: narrow layers keep every thread busy)
    const int tc = j0 / g.tile_cols, c0 = j0 - tc * g.tile_cols;  // JPT | tile_cols (host-checked)
    double rrow[JPT];
#pragma unroll
    for (int jj = 0; jj < JPT; ++jj) rrow[jj] = rp.r_source + double(c0 + jj + 1) * rp.r_row;
    const size_t plane = g.plane_bytes();
    const size_t sp_stride = size_t(g.GR) * g.GC * kLimbs * plane;
    const size_t sstride = size_t(g.Kp) * g.Np;
    for (int i = blockIdx.y * blockDim.y + threadIdx.y; i < g.K; i += gridDim.y * blockDim.y) {
      const int tr = i / g.tile_rows, r = i - tr * g.tile_rows;
      const double rcol = double(g.tile_rows - r) * rp.r_col;
      constexpr int PRE = S < 4 ? S : 4;  // slices loaded per group (register budget)
      double dg[JPT], u[PRE][JPT], acc[JPT];
      {
        double dw[JPT];
        ld_vec<JPT>(dW + size_t(i) * g.N + j0, dw);
#pragma unroll
        for (int jj = 0; jj < JPT; ++jj) {
          dwmax = fmax(dwmax, fabs(dw[jj]));
          dg[jj] = dw[jj] * up.factor;  // scale_gradient (update.cpp:16-24)
          acc[jj] = 0.0;
        }
      }
      double* mrow = master + size_t(i) * g.Np + j0;
      uint32_t qi[JPT];
      if constexpr (!VAR && CONV) {
        const typename VecT<JPT>::Q t =
            *reinterpret_cast<const typename VecT<JPT>::Q*>(qmin + size_t(r) * g.tile_cols + c0);
        qi[0] = t.x;
        qi[1] = t.y;
        if constexpr (JPT == 4) {
          qi[2] = reinterpret_cast<const uint4&>(t).z;
          qi[3] = reinterpret_cast<const uint4&>(t).w;
        }
      }
      uint8_t* dbase = digits + (size_t(tr) * g.GC + tc) * kLimbs * plane + size_t(r) * g.C + c0;
#pragma unroll
      for (int s = S - 1; s >= 0; --s) {  // Horner order: most significant slice first
        const int qs = (S - 1 - s) % PRE;  // position within the current group
        if (qs == 0) {                     // all slices of the next group in flight at once
#pragma unroll
          for (int q = 0; q < PRE; ++q) ld_vec<JPT>(mrow + (s - q) * sstride, u[q]);
        }
        uint32_t q[2][JPT];
#pragma unroll
        for (int jj = 0; jj < JPT; ++jj) {
          const double ui = u[qs][jj];
          double du = dg[jj];
          if constexpr (NL) {
            if (dg[jj] != 0.0) {
              const bool pos_active = ui > 0.0 || (ui == 0.0 && dg[jj] < 0.0);
              const double dev_arg = pos_active ? -dg[jj] : dg[jj];
              const double gg = rp.g_min + fabs(ui);
              if (gg < rp.g_min || gg > rp.g_max) atomicOr(&sc->err_flag, 1);  // update.cpp:28-29
              const double x = dev_arg >= 0.0 ? (gg - rp.g_min) / range : (rp.g_max - gg) / range;
              const double nl = dev_arg * exp(-up.v * x);
              du = pos_active ? -nl : nl;
            }
          }
          double noise = 0.0;
          if constexpr (NOISE) {
            if (dg[jj] != 0.0) {
              const double sigma = up.gamma * sqrt(range * fabs(dg[jj]));
              if (sigma != 0.0)
                noise = sigma * rng_gaussian(rng_key(up.seed, up.iteration, uint64_t(s),
                                                     uint64_t(int64_t(i) * g.N + j0 + jj)));
            }
          }
          double nu = ui - up.lr * (du + noise);
          nu = nu > range ? range : nu;
          nu = nu < -range ? -range : nu;
          u[qs][jj] = nu;
          acc[jj] = acc[jj] * double(1u << g.db) + nu;
          if constexpr (!CONV) continue;  // tile engines regenerate per tile afterwards
          const double rpath = AAM ? (rrow[jj] + rcol) + rp.r_sense : 0.0;
          const uint64_t idx = uint64_t(i) * g.Np + j0 + jj;
          if constexpr (VAR) {
            q[0][jj] = convert_qt<true, AAM>(rp, nu, s, 0, idx, rpath);
            q[1][jj] = convert_qt<true, AAM>(rp, nu, s, 1, idx, rpath);
          } else {
            const int pa = nu > 0.0 ? 0 : 1;
            const uint32_t qa = convert_qt<false, AAM>(rp, nu, s, pa, idx, rpath);
            q[0][jj] = pa == 0 ? qa : qi[jj];
            q[1][jj] = pa == 0 ? qi[jj] : qa;
          }
        }
        st_vec<JPT>(mrow + s * sstride, u[qs]);
        if constexpr (!CONV) continue;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          typename VecT<JPT>::B w[kLimbs] = {0, 0, 0};
#pragma unroll
          for (int jj = 0; jj < JPT; ++jj) {
            const uint32_t lo = q[p][jj] % 65025u, hi = q[p][jj] / 65025u;
            w[0] |= typename VecT<JPT>::B((lo % 255u) << (8 * jj));
            w[1] |= typename VecT<JPT>::B((lo / 255u) << (8 * jj));
            w[2] |= typename VecT<JPT>::B(hi << (8 * jj));
          }
          uint8_t* d = dbase + (size_t(s) * 2 + p) * sp_stride;
#pragma unroll
          for (int k = 0; k < kLimbs; ++k) *reinterpret_cast<typename VecT<JPT>::B*>(d + k * plane) = w[k];
        }
      }
#pragma unroll
      for (int jj = 0; jj < JPT; ++jj) wmax = fmax(wmax, fabs(up.wfactor * acc[jj]));
    }
  }
  wmax = warp_max(wmax);
  dwmax = warp_max(dwmax);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_pos(&sc->wmax, wmax);
    atomic_max_pos(&sc->dwmax, dwmax);
  }
}

// Generic fallback (any S, ragged shapes): one weight per thread, runtime
// flags, scalar stores.  Used when S is not 1/2/4/8 or JPT does not divide
// N and tile_cols.
__global__ void __launch_bounds__(256) k_update_any(Geo g, RegenP rp, UpdP up, const double* __restrict__ dW,
                                                    double* __restrict__ master, uint8_t* __restrict__ digits,
                                                    DevScalars* sc) {
  if (sc->dw_nonfinite) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicOr(&sc->err_flag, 2);
    return;
  }
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double wmax = 0.0, dwmax = 0.0;
  if (j < g.N) {
    const int tc = j / g.tile_cols, c = j - tc * g.tile_cols;
    const double range = rp.range;
    for (int i = blockIdx.y; i < g.K; i += gridDim.y) {
      const int tr = i / g.tile_rows, r = i - tr * g.tile_rows;
      const double dw = dW[size_t(i) * g.N + j];
      dwmax = fmax(dwmax, fabs(dw));
      const double dg = dw * up.factor;
      const double rpath = rp.aam ? aam_rpath(rp, g, r, c) : 0.0;
      const uint64_t idx = uint64_t(i) * g.Np + j;
      double acc = 0.0;
      for (int s = g.S - 1; s >= 0; --s) {
        double* mp = master + (size_t(s) * g.Kp + i) * g.Np + j;
        const double ui = *mp;
        double du = dg;
        if (!up.linear && dg != 0.0) {
          const bool pos_active = ui > 0.0 || (ui == 0.0 && dg < 0.0);
          const double dev_arg = pos_active ? -dg : dg;
          const double gg = rp.g_min + fabs(ui);
          if (gg < rp.g_min || gg > rp.g_max) atomicOr(&sc->err_flag, 1);
          const double x = dev_arg >= 0.0 ? (gg - rp.g_min) / range : (rp.g_max - gg) / range;
          const double nl = dev_arg * exp(-up.v * x);
          du = pos_active ? -nl : nl;
        }
        double noise = 0.0;
        if (up.gamma != 0.0 && dg != 0.0) {
          const double sigma = up.gamma * sqrt(range * fabs(dg));
          if (sigma != 0.0)
            noise = sigma * rng_gaussian(rng_key(up.seed, up.iteration, uint64_t(s), uint64_t(int64_t(i) * g.N + j)));
        }
        double nu = ui - up.lr * (du + noise);
        if (nu > range) nu = range;
        if (nu < -range) nu = -range;
        *mp = nu;
        acc = acc * double(1u << g.db) + nu;
        if (digits)
          for (int p = 0; p < 2; ++p) store_digits(digits, g, s, p, i, j, convert_q(rp, nu, s, p, idx, rpath));
      }
      wmax = fmax(wmax, fabs(up.wfactor * acc));
    }
  }
  wmax = warp_max(wmax);
  dwmax = warp_max(dwmax);
  if ((threadIdx.x & 31) == 0) {
    atomic_max_pos(&sc->wmax, wmax);
    atomic_max_pos(&sc->dwmax, dwmax);
  }
}

// ------------------------------------------------- K3b, bulk-copy pipeline
// Same per-weight arithmetic as k_update, restructured for HBM: a persistent
// CTA runs one producer warp that streams "units" (rpu rows x cw columns of
// dW, the S master slices and, sigma != 0, the 2S variation multiplier
// planes) into a ring of shared-memory stages with cp.async.bulk (one
// contiguous copy per array row, completion counted on the stage's full
// mbarrier), while 8 consumer warps take one device column per thread from
// the stage that has landed.  Loads therefore stay in flight while the fp64
// conversion (two correctly rounded reciprocals per AAM device) runs: the
// register-staged k_update issued the next row's loads only after the
// current row's stores (23% warps active, 0.30-0.60 of HBM).
namespace updp {
constexpr int kConsumers = 256;         // one device column per consumer thread
constexpr int kThreads = kConsumers + 32;
constexpr int kMaxStages = 8;
constexpr int kHdr = 2 * kMaxStages * 8;  // full[] + empty[] mbarriers

__device__ __forceinline__ uint32_t s_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(s_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16),
// streamed past L2 with an evict-first policy: every byte is read once
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(bar)), "l"(pol)
      : "memory");
}
}  // namespace updp

// AAM conversion + snap for the update kernel: q = rint(2^e / (1/gv + rpath))
// with the reference's correctly rounded chain (aam.cpp:14-31, the 1.0 / x of
// convert_qt).  The chain's value x_e is within 3 2^-53 x of the real
// X = 2^e gv / (1 + gv rpath); the fast form below (one fma, one reciprocal
// refined to ~2^-52 from MUFU.RCP64H, two products) is within 6 2^-53 X of
// X.  With X < 2^24 the two differ by < 2^-25, so whenever the fast value is
// farther than 2^-20 from a half-integer both round to the same integer;
// otherwise (about 2e-6 of conversions) the exact chain decides.
__device__ __forceinline__ uint32_t aam_snap(double gv, double rpath, double scale) {
  const double w = __fma_rn(gv, rpath, 1.0);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(w));
  double e = __fma_rn(-w, r, 1.0);
  e = __fma_rn(e, e, e);
  r = __fma_rn(r, e, r);
  const double x = __dmul_rn(__dmul_rn(gv, scale), r);
  const double xr = rint(x);
  if (fabs(__dsub_rn(x, xr)) < 0.5 - 0x1p-20) return __double2uint_rn(xr);
  return __double2uint_rn(__dmul_rn(__drcp_rn(__dadd_rn(__drcp_rn(gv), rpath)), scale));
}

struct UpdTmaP {
  int cw_log;     // log2 of the unit width (columns), cw * rpu == 256
  int rpu;        // rows per unit
  int nch;        // column chunks per row block
  int nst;        // pipeline stages
  int nunits;     // row blocks * nch (< 2^31, host-checked)
  tc::FDiv fd_nch, fd_tr, fd_tc;  // unit and tile decode by multiply-shift
};

template <int S, bool VAR, bool NL, bool NOISE, bool AAM, bool CONV>
__global__ void __launch_bounds__(updp::kThreads, 2)
    k_update_tma(Geo g, RegenP rp, UpdP up, UpdTmaP tp, const double* __restrict__ dW, double* __restrict__ master,
                 uint8_t* __restrict__ digits, DevScalars* sc, const uint32_t* __restrict__ qmin) {
  using namespace updp;
  constexpr int NA = 1 + S + (VAR ? 2 * S : 0);  // double arrays per unit row: dW, master[S], varm[S][2]
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kMaxStages;
  double* stages = reinterpret_cast<double*>(smem + kHdr);
  constexpr int kStageD = kConsumers * NA;  // doubles per stage
  if (sc->dw_nonfinite) {  // scale_gradient throws before touching the master (update.cpp:18-19)
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&sc->err_flag, 2);
    return;
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < tp.nst; ++k) {
      bar_init(&full[k], 1);
      bar_init(&empty[k], kConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int cw = 1 << tp.cw_log;
  if (threadIdx.x >= kConsumers) {  // producer warp
    if (threadIdx.x != kConsumers) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const size_t sstride = size_t(g.Kp) * g.Np;
    int slot = 0;
    uint32_t phase = 0;
    bool wrapped = false;
    for (int u = blockIdx.x; u < tp.nunits; u += gridDim.x) {
      if (wrapped) bar_wait(&empty[slot], phase ^ 1);
      const int rb = tc::fdiv(u, tp.fd_nch);
      const int j0 = (u - rb * tp.nch) << tp.cw_log;
      const int ncols = min(cw, g.N - j0);
      const int i0 = rb * tp.rpu, nrows = min(tp.rpu, g.K - i0);
      const uint32_t rbytes = uint32_t(ncols) * 8;  // N even (host-checked): a multiple of 16
      bar_expect(&full[slot], rbytes * NA * nrows);
      double* st = stages + size_t(slot) * kStageD;
      for (int rr = 0; rr < nrows; ++rr) {
        const int i = i0 + rr;
        double* d = st + size_t(rr) * NA * cw;
        bulk_g2s(d, dW + size_t(i) * g.N + j0, rbytes, &full[slot], pol);
        const double* m = master + size_t(i) * g.Np + j0;
        for (int s = 0; s < S; ++s) bulk_g2s(d + (1 + s) * cw, m + s * sstride, rbytes, &full[slot], pol);
        if constexpr (VAR)
          for (int sp = 0; sp < 2 * S; ++sp)
            bulk_g2s(d + (1 + S + sp) * cw, rp.varm + sp * rp.kpnp + size_t(i) * g.Np + j0, rbytes, &full[slot],
                     pol);
      }
      if (++slot == tp.nst) {
        slot = 0;
        phase ^= 1;
        wrapped = true;
      }
    }
    return;
  }
  // consumers: thread t owns column cc of unit row rr
  const int t = threadIdx.x, rr = t >> tp.cw_log, cc = t & (cw - 1);
  const double range = rp.range;
  const int64_t sstride = int64_t(g.Kp) * g.Np;
  const int64_t plane = int64_t(g.R) * g.C;
  const int64_t sp_stride = int64_t(g.GR) * g.GC * kLimbs * plane;
  double wmax = 0.0, dwmax = 0.0;
  int slot = 0;
  uint32_t phase = 0;
  for (int u = blockIdx.x; u < tp.nunits; u += gridDim.x) {
    const int rb = tc::fdiv(u, tp.fd_nch);
    const int j = ((u - rb * tp.nch) << tp.cw_log) + cc;
    const int i = rb * tp.rpu + rr;
    bar_wait(&full[slot], phase);
    const double* __restrict__ d = stages + slot * kStageD + rr * NA * cw + cc;
    if (i < g.K && j < g.N) {
      const int tr = tc::fdiv(i, tp.fd_tr), r = i - tr * g.tile_rows;
      const int tcol = tc::fdiv(j, tp.fd_tc), c = j - tcol * g.tile_cols;
      const double rpath = AAM ? ((rp.r_source + double(c + 1) * rp.r_row) + double(g.tile_rows - r) * rp.r_col) +
                                     rp.r_sense
                               : 0.0;
      const double dw = d[0];
      double ui[S];
#pragma unroll
      for (int s = 0; s < S; ++s) ui[s] = d[(1 + s) * cw];
      dwmax = fmax(dwmax, fabs(dw));
      const double dg = dw * up.factor;  // scale_gradient (update.cpp:16-24)
      uint32_t qi = 0;
      if constexpr (!VAR && CONV) qi = __ldg(qmin + r * g.tile_cols + c);
      // slice S-1 first (Horner order); pointers step down one slice at a time
      double* mp = master + (int64_t(S - 1) * sstride + int64_t(i) * g.Np + j);
      uint8_t* dp = digits + (int64_t(S - 1) * 2 * sp_stride + (int64_t(tr) * g.GC + tcol) * kLimbs * plane +
                              int64_t(r) * g.C + c);
      double acc = 0.0;
#pragma unroll
      for (int s = S - 1; s >= 0; --s, mp -= sstride, dp -= 2 * sp_stride) {
        const double u0 = ui[s];
        double du = dg;
        if constexpr (NL) {
          if (dg != 0.0) {
            const bool pos_active = u0 > 0.0 || (u0 == 0.0 && dg < 0.0);
            const double dev_arg = pos_active ? -dg : dg;
            const double gg = rp.g_min + fabs(u0);
            if (gg < rp.g_min || gg > rp.g_max) atomicOr(&sc->err_flag, 1);  // update.cpp:28-29
            const double x = dev_arg >= 0.0 ? (gg - rp.g_min) / range : (rp.g_max - gg) / range;
            const double nl = dev_arg * exp(-up.v * x);
            du = pos_active ? -nl : nl;
          }
        }
        double noise = 0.0;
        if constexpr (NOISE) {
          if (dg != 0.0) {
            const double sigma = up.gamma * sqrt(range * fabs(dg));
            if (sigma != 0.0)
              noise = sigma * rng_gaussian(rng_key(up.seed, up.iteration, uint64_t(s), uint64_t(int64_t(i) * g.N + j)));
          }
        }
        double nu = u0 - up.lr * (du + noise);
        nu = nu > range ? range : nu;
        nu = nu < -range ? -range : nu;
        *mp = nu;
        acc = acc * double(1u << g.db) + nu;
        if constexpr (CONV) {
          uint32_t q[2];
          if constexpr (VAR) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
              const double up_ = p == 0 ? nu : -nu;
              double gv = (up_ > 0.0 ? up_ : 0.0) + rp.g_min;
              gv = fmin(gv * d[(1 + S + 2 * s + p) * cw], rp.g_max);  // mapping.cpp:39-58
              if constexpr (AAM) q[p] = aam_snap(gv, rpath, rp.snap_scale);
              else q[p] = __double2uint_rn(__dmul_rn(gv, rp.snap_scale));
            }
          } else {
            const int pa = nu > 0.0 ? 0 : 1;
            double gv = (nu > 0.0 ? nu : -nu) + rp.g_min;  // |nu| + g_min: the active device (nu == 0: either)
            const uint32_t qa = AAM ? aam_snap(gv, rpath, rp.snap_scale) : __double2uint_rn(__dmul_rn(gv, rp.snap_scale));
            q[0] = pa == 0 ? qa : qi;
            q[1] = pa == 0 ? qi : qa;
          }
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const uint32_t lo = q[p] % 65025u, hi = q[p] / 65025u;
            uint8_t* o = dp + p * sp_stride;
            o[0] = uint8_t(lo % 255u);
            o[plane] = uint8_t(lo / 255u);
            o[2 * plane] = uint8_t(hi);
          }
        }
      }
      wmax = fmax(wmax, fabs(up.wfactor * acc));
    }
    __syncwarp();
    if ((t & 31) == 0) bar_arrive(&empty[slot]);
    if (++slot == tp.nst) {
      slot = 0;
      phase ^= 1;
    }
  }
  wmax = warp_max(wmax);
  dwmax = warp_max(dwmax);
  if ((t & 31) == 0) {
    atomic_max_pos(&sc->wmax, wmax);
    atomic_max_pos(&sc->dwmax, dwmax);
  }
}

template <int S>
static bool launch_update_tma_s(const xbs_core* c, const UpdP& up, cudaStream_t st, bool master_only) {
  const Geo& g = c->g;
  UpdTmaP tp{};
  int cw = 32;
  while (cw < 256 && cw < g.N) cw *= 2;
  tp.cw_log = __builtin_ctz(unsigned(cw));
  tp.rpu = 256 / cw;
  tp.nch = (g.N + cw - 1) / cw;
  const int64_t nunits = int64_t((g.K + tp.rpu - 1) / tp.rpu) * tp.nch;
  if (nunits >= (int64_t{1} << 31)) return false;
  tp.nunits = int(nunits);
  tp.fd_nch = tc::make_fdiv(uint32_t(tp.nch));
  tp.fd_tr = tc::make_fdiv(uint32_t(g.tile_rows));
  tp.fd_tc = tc::make_fdiv(uint32_t(g.tile_cols));
  const bool var = !master_only && c->rp.sigma != 0.0, nl = !up.linear, noise = up.gamma != 0.0;
  const bool aam = c->rp.aam && (c->rp.r_source + c->rp.r_row + c->rp.r_col + c->rp.r_sense) > 0.0;
  const int na = 1 + S + (var ? 2 * S : 0);
  const size_t stage_bytes = size_t(updp::kConsumers) * na * 8;
  tp.nst = int(std::min<size_t>(updp::kMaxStages, std::max<size_t>(2, (100u << 10) / stage_bytes)));
  const size_t smem = updp::kHdr + tp.nst * stage_bytes;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(tp.nunits, 2 * 148)));
  auto go = [&](auto kern) {
    // one attribute call per instantiation (stages never exceed 2 x 50 KB)
    static const void* done[64];
    static int ndone = 0;
    bool seen = false;
    for (int k = 0; k < ndone; ++k) seen |= done[k] == reinterpret_cast<const void*>(kern);
    if (!seen) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(updp::kHdr + (100u << 10)));
      if (ndone < 64) done[ndone++] = reinterpret_cast<const void*>(kern);
    }
    kern<<<grid, updp::kThreads, smem, st>>>(g, c->rp, up, tp, c->d_dW, c->d_master, c->d_digits, c->d_sc,
                                             c->d_qmin);
  };
#define XBS_UPD(V, N, A) go(k_update_tma<S, V, N, N, A, true>)
  if (master_only) {
    if (!nl && !noise) go(k_update_tma<S, false, false, false, false, false>);
    else go(k_update_tma<S, false, true, true, false, false>);
  } else if (aam) {
    if (!var && !nl && !noise) XBS_UPD(false, false, true);
    else if (var && !nl && !noise) XBS_UPD(true, false, true);
    else if (!var) XBS_UPD(false, true, true);
    else XBS_UPD(true, true, true);
  } else {
    if (!var && !nl && !noise) XBS_UPD(false, false, false);
    else if (var && !nl && !noise) XBS_UPD(true, false, false);
    else if (!var) XBS_UPD(false, true, false);
    else XBS_UPD(true, true, false);
  }
#undef XBS_UPD
  return true;
}

// The bulk-copy kernel needs 16-byte aligned row segments: N and Np even.
static bool launch_update_tma(const xbs_core* c, const UpdP& up, cudaStream_t st, bool master_only) {
  if (c->g.N % 2 || c->g.Np % 2 || c->g.K == 0 || c->g.N == 0) return false;
  switch (c->g.S) {
    case 1: return launch_update_tma_s<1>(c, up, st, master_only);
    case 2: return launch_update_tma_s<2>(c, up, st, master_only);
    case 4: return launch_update_tma_s<4>(c, up, st, master_only);
    case 8: return launch_update_tma_s<8>(c, up, st, master_only);
    default: return false;
  }
}

template <int S, int JPT>
static void launch_update_s(const xbs_core* c, const UpdP& up, cudaStream_t st, bool master_only) {
  // threads per row: the row's JPT-weight groups rounded up to whole warps
  // (<= 256); the rest of the 256-thread block takes further rows
  const int tpr = int(std::min<int64_t>(256, ((c->g.N / JPT + 31) / 32) * 32));
  const dim3 block(tpr, 256 / tpr);
  const dim3 grid((c->g.N / JPT + tpr - 1) / tpr, unsigned(std::min<int64_t>((c->g.K + block.y - 1) / block.y, 65535)));
  const bool var = c->rp.sigma != 0.0, nl = !up.linear, noise = up.gamma != 0.0;
  // AAM with a zero path resistance everywhere is the identity conversion
  const bool aam = c->rp.aam && (c->rp.r_source + c->rp.r_row + c->rp.r_col + c->rp.r_sense) > 0.0;
  auto go = [&](auto kern) {
    kern<<<grid, block, 0, st>>>(c->g, c->rp, up, c->d_dW, c->d_master, c->d_digits, c->d_sc, c->d_qmin);
  };
#define XBS_UPD(V, N, A) go(k_update<S, JPT, V, N, N, A>)
  if (master_only) {
    if (!nl && !noise) go(k_update<S, JPT, false, false, false, false, false>);
    else go(k_update<S, JPT, false, true, true, false, false>);
  } else if (aam) {
    if (!var && !nl && !noise) XBS_UPD(false, false, true);
    else if (var && !nl && !noise) XBS_UPD(true, false, true);
    else if (!var) XBS_UPD(false, true, true);
    else XBS_UPD(true, true, true);
  } else {
    if (!var && !nl && !noise) XBS_UPD(false, false, false);
    else if (var && !nl && !noise) XBS_UPD(true, false, false);
    else if (!var) XBS_UPD(false, true, false);
    else XBS_UPD(true, true, false);
  }
#undef XBS_UPD
}

template <int JPT>
static bool launch_update_j(const xbs_core* c, const UpdP& up, cudaStream_t st, bool mo) {
  if (c->g.N % JPT || c->g.tile_cols % JPT || c->g.C % JPT) return false;
  switch (c->g.S) {
    case 1: launch_update_s<1, JPT>(c, up, st, mo); return true;
    case 2: launch_update_s<2, JPT>(c, up, st, mo); return true;
    case 4: launch_update_s<4, JPT>(c, up, st, mo); return true;
    case 8: launch_update_s<8, JPT>(c, up, st, mo); return true;
    default: return false;
  }
}

void launch_update(const xbs_core* c, const UpdP& up, cudaStream_t st, bool master_only) {
  static const bool legacy = [] {  // A/B switch for the register-staged kernel (perf experiments only)
    const char* e = getenv("XBS_UPDATE_LEGACY");
    return e && *e == '1';
  }();
  if (!legacy && launch_update_tma(c, up, st, master_only)) return;
  if (launch_update_j<4>(c, up, st, master_only)) return;
  if (launch_update_j<2>(c, up, st, master_only)) return;
  const dim3 grid((c->g.N + 255) / 256, std::min(c->g.K, 65535));
  k_update_any<<<grid, 256, 0, st>>>(c->g, c->rp, up, c->d_dW, c->d_master, master_only ? nullptr : c->d_digits,
                                     c->d_sc);
}

// q(g_min) per tile position (sigma == 0 only): tile_rows x tile_cols
__global__ void k_qmin(Geo g, RegenP rp, uint32_t* qmin) {
  const int n = g.tile_rows * g.tile_cols;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t / g.tile_cols, c = t % g.tile_cols;
    qmin[t] = convert_q(rp, 0.0, 0, 0, 0, rp.aam ? aam_rpath(rp, g, r, c) : 0.0);
  }
}

void launch_qmin(const xbs_core* c, cudaStream_t st) { k_qmin<<<64, 256, 0, st>>>(c->g, c->rp, c->d_qmin); }

// implied_weights() (mapping.cpp:70-81) -> K x N row-major
__global__ void k_implied(Geo g, double wfactor, const double* __restrict__ master, double* __restrict__ out) {
  const int64_t n = int64_t(g.K) * g.N;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / g.N), j = int(t % g.N);
    double acc = 0.0;
    for (int s = g.S - 1; s >= 0; --s) acc = acc * double(1u << g.db) + master[(size_t(s) * g.Kp + i) * g.Np + j];
    out[t] = wfactor * acc;
  }
}

void launch_implied(const xbs_core* c, double* d_out, cudaStream_t st) {
  const int64_t n = int64_t(c->g.K) * c->g.N;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
  const double levels = double((uint64_t{1} << c->g.wb) - 1), sl = double((uint64_t{1} << c->g.db) - 1);
  const double wf = (c->layer_scale / (c->rp.g_max - c->rp.g_min)) * (sl / levels);
  k_implied<<<blocks, 256, 0, st>>>(c->g, wf, c->d_master, d_out);
}

// non-ideal tile readback: snapped conductance q * 2^-e, tile_rows x tile_cols
// column-major.
__global__ void k_digits_to_g(Geo g, int e, const uint8_t* __restrict__ digits, int s, int p, int tr, int tc,
                              double* out) {
  const int n = g.tile_rows * g.tile_cols;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int r = t % g.tile_rows, c = t / g.tile_rows;
    out[t] = ldexp(double(load_q(digits, g, s, p, tr, tc, r, c)), -e);
  }
}

void launch_digits_to_g(const xbs_core* c, int s, int p, int tr, int tc, double* d_out, cudaStream_t st) {
  k_digits_to_g<<<64, 256, 0, st>>>(c->g, c->rp.snap_e, c->d_digits, s, p, tr, tc, d_out);
}

// ------------------------------------------------------------------ prep_x
// quantize_unsigned_codes (tensor.cpp:8-25) + DAC bit planes (layers.cpp:236-241).
// x is M x K column-major (ld = M) and the planes are row-major [b*TPi+k][KI],
// so the kernel is a tiled transpose: a 64 (batch) x 64 (device column) tile
// of codes is staged in shared memory from coalesced column reads, then the
// code rows, the u8 dW code plane and both bit-plane copies (bits, 255*bits)
// are written as contiguous row segments.
constexpr int kPrepTB = 64, kPrepTI = 64, kPrepThreads = 256;

// min(llround(v / step), levels) for v > 0 (tensor.cpp:8-51), without the
// fp64 division on the common path: t = v * RN(1/step) is within 3 2^-53 t
// of RN(v / step), so rint(t) is the answer unless t sits within 2^-40 of a
// half-integer (then the exact quotient decides).
__device__ __forceinline__ double quant_mag(double v, double step, double inv, double levels) {
  const double t = v * inv;
  if (t >= levels + 1.0) return levels;
  const double k = rint(t);
  if (fabs(t - k) < 0.5 - 0x1p-40) return fmin(k, levels);
  return fmin(double(llround(v / step)), levels);
}

// The plane copies of a 16-column group are written when the group or its
// 32-byte sector partner holds logical columns (a partial sector would make
// L2 read the line back from HBM to merge it); groups whose whole sector is
// tile padding are left as allocated (zero) and never touched.
__device__ __forceinline__ bool plane_sector_live(int r16, int nlive) {
  return (r16 & ~31) < nlive;  // r16: first block column of the group
}

// CT = uint16_t: the tensor-core contract (codes of <= 16 bits and both
// bit-plane copies).  CT = uint32_t: the general converters (volts mode),
// whose exact fp64 kernels read the codes directly -- codes of up to 24 bits
// (layers.cpp:28-31), no planes.
template <bool CONV, class CT>
__global__ void __launch_bounds__(256) k_prep_x(Geo g, const double* __restrict__ x, int64_t M, int64_t rowsF,
                                                double step, double inv, double levels, CT* __restrict__ codes,
                                                uint8_t* __restrict__ A, uint8_t* __restrict__ c8, int ld8,
                                                ConvSrc cv, int64_t bt0) {
  constexpr bool kPlanes = sizeof(CT) == 2;
  __shared__ CT cs[kPrepTB][kPrepTI + 2];
  __shared__ int coff[kPrepTI], cky[kPrepTI], ckx[kPrepTI];  // CONV: image offset and (ky, kx) per column
  const int64_t b0 = (bt0 + blockIdx.y) * kPrepTB;
  const int c0 = blockIdx.x * kPrepTI;  // column blocks fastest: a plane row's segments are written together  // device column (0 .. KI); a block lies in one row tile (R % 64 == 0)
  const int tr = c0 / g.R, r0 = c0 % g.R;
  const int i0 = tr * g.tile_rows + r0;  // logical feature of block column 0
  const int nlive = min(kPrepTI, min(g.tile_rows - r0, g.K - i0));  // logical columns in this block
  if (nlive <= 0) return;  // tile padding only: planes stay zero, no codes
  // CONV: this thread's patch row (blockDim.x is a multiple of kPrepTB, so
  // bl = threadIdx.x % kPrepTB for every element it loads)
  int img = 0, oys = 0, oxs = 0;
  if constexpr (CONV) {
    if (threadIdx.x < nlive) {
      const int i = i0 + threadIdx.x;
      const int kk = cv.k * cv.k, c = i / kk, ky = (i % kk) / cv.k, kx = i % cv.k;
      coff[threadIdx.x] = (c * cv.h + ky) * cv.w + kx;
      cky[threadIdx.x] = ky;
      ckx[threadIdx.x] = kx;
    }
    const int64_t b = b0 + threadIdx.x % kPrepTB;
    if (b < M) {
      const int rb = int(b), ox = rb % cv.ow, t = rb / cv.ow, oy = t % cv.oh;
      img = t / cv.oh;
      oys = oy * cv.stride - cv.pad;
      oxs = ox * cv.stride - cv.pad;
    }
    __syncthreads();
  }
  // all of this thread's loads are issued before any is used (memory-level
  // parallelism); blockDim.x == kPrepThreads
  constexpr int kLd = kPrepTB * kPrepTI / kPrepThreads;
  const int bl = threadIdx.x % kPrepTB, il0 = threadIdx.x / kPrepTB;  // consecutive threads: consecutive rows
  const bool brow = b0 + bl < M;
  double xv[kLd];
#pragma unroll
  for (int n = 0; n < kLd; ++n) {
    const int il = il0 + n * (kPrepThreads / kPrepTB);
    xv[n] = 0.0;
    if (brow && il < nlive) {
      if constexpr (CONV) {
        const int iy = oys + cky[il], ix = oxs + ckx[il];
        if (iy >= 0 && iy < cv.h && ix >= 0 && ix < cv.w)
          xv[n] = __ldg(x + int64_t(coff[il] + oys * cv.w + oxs) * cv.batch + img);
      } else {
        xv[n] = __ldg(x + int64_t(i0 + il) * M + b0 + bl);
      }
    }
  }
#pragma unroll
  for (int n = 0; n < kLd; ++n) {
    // llround of a non-positive quotient is <= 0: code 0 (clamped); columns
    // beyond nlive load 0 and so hold code 0
    const uint32_t code = xv[n] > 0.0 ? uint32_t(quant_mag(xv[n], step, inv, levels)) : 0u;
    cs[bl][il0 + n * (kPrepThreads / kPrepTB)] = CT(code);
  }
  __syncthreads();
  // codes [b][K] (u16) and the u8 dW codes [b][ld8]: one thread per (row, 8
  // columns), vector stores where the row segment is 16-byte aligned
  const bool vec = (g.K % 8) == 0 && (i0 % 8) == 0;
  for (int e = threadIdx.x; e < kPrepTB * (kPrepTI / 8); e += blockDim.x) {
    const int o = e % (kPrepTI / 8) * 8, r = e / (kPrepTI / 8);
    const int64_t b = b0 + r;
    if (b >= M || o >= nlive) continue;
    const CT* src = &cs[r][o];
    if (vec && o + 8 <= nlive) {
      uint32_t w8[2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        w8[h] = (uint32_t(src[4 * h]) & 0xffu) | ((uint32_t(src[4 * h + 1]) & 0xffu) << 8) |
                ((uint32_t(src[4 * h + 2]) & 0xffu) << 16) | (uint32_t(src[4 * h + 3]) << 24);
      if constexpr (kPlanes) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) w[h] = uint32_t(src[2 * h]) | (uint32_t(src[2 * h + 1]) << 16);
        *reinterpret_cast<uint4*>(codes + b * g.K + i0 + o) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
        uint4* co = reinterpret_cast<uint4*>(codes + b * g.K + i0 + o);
        co[0] = make_uint4(src[0], src[1], src[2], src[3]);
        co[1] = make_uint4(src[4], src[5], src[6], src[7]);
      }
      if (c8) *reinterpret_cast<uint2*>(c8 + b * ld8 + i0 + o) = make_uint2(w8[0], w8[1]);
    } else {
      for (int t = 0; t < 8 && o + t < nlive; ++t) {
        codes[b * g.K + i0 + o + t] = src[t];
        if (c8) c8[b * ld8 + i0 + o + t] = uint8_t(src[t]);
      }
    }
  }
  // bit planes: one thread per (batch row, 16 columns) packs the codes'
  // bytes four to a word once; plane k is then (word >> k) & 0x01010101
  if constexpr (!kPlanes) return;
  constexpr int Q = kPrepTI / 16;
  for (int e = threadIdx.x; e < kPrepTB * Q; e += blockDim.x) {
    const int q = e % Q, r = e / Q;
    const int64_t b = b0 + r;
    if (b >= M || !plane_sector_live(q * 16, nlive)) continue;
    uint32_t lo8[4], hi8[4];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t l = 0, h = 0;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const uint32_t v = cs[r][q * 16 + q4 * 4 + qq];
        l |= (v & 0xffu) << (8 * qq);
        h |= (v >> 8) << (8 * qq);
      }
      lo8[q4] = l;
      hi8[q4] = h;
    }
    uint8_t* p0 = A + (b * g.TPi) * g.KI + c0 + q * 16;
    for (int k = 0; k < g.TPi; ++k, p0 += g.KI) {
      uint32_t w0[4];
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) w0[q4] = ((k < 8 ? lo8[q4] >> k : hi8[q4] >> (k - 8))) & 0x01010101u;
      *reinterpret_cast<uint4*>(p0) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
      *reinterpret_cast<uint4*>(p0 + rowsF * g.KI) =
          make_uint4(w0[0] * 255u, w0[1] * 255u, w0[2] * 255u, w0[3] * 255u);
    }
  }
}

void launch_prep_x(const xbs_core* c, const double* d_x, int64_t M, cudaStream_t st, const ConvSrc* conv) {
  const int64_t rowsF = rows_fwd(M, c->g.TPi);
  // zero the M-padding rows once per call (rows [M*TPi, rowsF))
  const int64_t pad0 = M * c->g.TPi;
  if (c->d_Af && rowsF > pad0) {
    cudaMemsetAsync(c->d_Af + pad0 * c->g.KI, 0, size_t(rowsF - pad0) * c->g.KI, st);
    cudaMemsetAsync(c->d_Af + (rowsF + pad0) * c->g.KI, 0, size_t(rowsF - pad0) * c->g.KI, st);
  }
  if (M == 0) return;
  const int64_t nbt = (M + kPrepTB - 1) / kPrepTB;  // batch tiles, launched in chunks of gridDim.y <= 65535
  const double levels = double((1 << c->opt.act_bits) - 1);
  const double step = c->opt.act_full_scale / levels;  // tensor.cpp:11
  if (c->d_xc8) {  // u8 code plane for the tcgen05 dW: rows [M, Mpad) must read 0
    const int64_t Mp = ((M + 127) / 128) * 128;
    if (Mp > M) cudaMemsetAsync(c->d_xc8 + M * c->KA, 0, size_t(Mp - M) * c->KA, st);
  }
  for (int64_t bt0 = 0; bt0 < nbt; bt0 += 65535) {
    const dim3 grid(unsigned(c->g.KI / kPrepTI), unsigned(std::min<int64_t>(nbt - bt0, 65535)));
    if (c->d_xcodes32) {  // volts mode: u32 codes only
      if (conv)
        k_prep_x<true, uint32_t><<<grid, 256, 0, st>>>(c->g, d_x, M, rowsF, step, 1.0 / step, levels, c->d_xcodes32,
                                                        nullptr, c->d_xc8, c->KA, *conv, bt0);
      else
        k_prep_x<false, uint32_t><<<grid, 256, 0, st>>>(c->g, d_x, M, rowsF, step, 1.0 / step, levels,
                                                         c->d_xcodes32, nullptr, c->d_xc8, c->KA, ConvSrc{}, bt0);
    } else if (conv)
      k_prep_x<true, uint16_t><<<grid, 256, 0, st>>>(c->g, d_x, M, rowsF, step, 1.0 / step, levels, c->d_xcodes,
                                                      c->d_Af, c->d_xc8, c->KA, *conv, bt0);
    else
      k_prep_x<false, uint16_t><<<grid, 256, 0, st>>>(c->g, d_x, M, rowsF, step, 1.0 / step, levels, c->d_xcodes,
                                                       c->d_Af, c->d_xc8, c->KA, ConvSrc{}, bt0);
  }
}

// ----------------------------------------------------------------- prep_dy
// se = max|dy| (layers.cpp:298), quantize_signed_codes (tensor.cpp:33-51),
// plus/minus planes (layers.cpp:316-331).  Row (b*TPe + k)*2 + phi, phi=0
// plus, phi=1 minus.  Tiled transpose as in k_prep_x.
__global__ void __launch_bounds__(256) k_prep_dy(Geo g, const double* __restrict__ dy, int64_t M, int64_t rowsB,
                                                 double levels, const DevScalars* __restrict__ sc,
                                                 int32_t* __restrict__ ecodes, uint8_t* __restrict__ A,
                                                 uint8_t* __restrict__ e8, int64_t plane8, int ld8, int64_t bt0) {
  __shared__ int32_t cs[kPrepTB][kPrepTI + 1];
  const double se = sc->se;
  const double step = se / levels;
  const double inv = 1.0 / step;
  const int64_t b0 = (bt0 + blockIdx.y) * kPrepTB;
  const int c0 = blockIdx.x * kPrepTI;  // column blocks fastest: a plane row's segments are written together  // device column (0 .. NI); a block lies in one column tile
  const int tc = c0 / g.C, cc0 = c0 % g.C;
  const int j0 = tc * g.tile_cols + cc0;
  const int nlive = min(kPrepTI, min(g.tile_cols - cc0, g.N - j0));
  if (nlive <= 0) return;  // tile padding only
  constexpr int kLd = kPrepTB * kPrepTI / kPrepThreads;  // loads issued before use, as in k_prep_x
  const int bl = threadIdx.x % kPrepTB, il0 = threadIdx.x / kPrepTB;
  const bool brow = b0 + bl < M && se > 0;
  double dv[kLd];
#pragma unroll
  for (int n = 0; n < kLd; ++n) {
    const int il = il0 + n * (kPrepThreads / kPrepTB);
    dv[n] = brow && il < nlive ? __ldg(dy + int64_t(j0 + il) * M + b0 + bl) : 0.0;
  }
#pragma unroll
  for (int n = 0; n < kLd; ++n) {
    int sm = 0;
    if (dv[n] != 0.0) {
      const double v = dv[n];
      const int mag = int(quant_mag(fabs(v), step, inv, levels));
      sm = mag == 0 ? 0 : (v < 0 ? -mag : mag);
    }
    cs[bl][il0 + n * (kPrepThreads / kPrepTB)] = sm;
  }
  __syncthreads();
  // signed codes [b][N] and the u8 plus / minus dW magnitudes, 8 columns per thread
  const bool vec = (g.N % 8) == 0 && (j0 % 8) == 0;
  for (int e = threadIdx.x; e < kPrepTB * (kPrepTI / 8); e += blockDim.x) {
    const int o = e % (kPrepTI / 8) * 8, r = e / (kPrepTI / 8);
    const int64_t b = b0 + r;
    if (b >= M || o >= nlive) continue;
    const int32_t* src = &cs[r][o];
    if (vec && o + 8 <= nlive) {
      uint32_t wp[2], wm[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t a = 0, m = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int v = src[4 * h + t];
          a |= uint32_t(v > 0 ? v : 0) << (8 * t);
          m |= uint32_t(v < 0 ? -v : 0) << (8 * t);
        }
        wp[h] = a;
        wm[h] = m;
      }
      int4* eo = reinterpret_cast<int4*>(ecodes + b * g.N + j0 + o);
      eo[0] = make_int4(src[0], src[1], src[2], src[3]);
      eo[1] = make_int4(src[4], src[5], src[6], src[7]);
      if (e8) {
        *reinterpret_cast<uint2*>(e8 + b * ld8 + j0 + o) = make_uint2(wp[0], wp[1]);
        *reinterpret_cast<uint2*>(e8 + plane8 + b * ld8 + j0 + o) = make_uint2(wm[0], wm[1]);
      }
    } else {
      for (int t = 0; t < 8 && o + t < nlive; ++t) {
        const int sm = src[t];
        ecodes[b * g.N + j0 + o + t] = sm;
        if (e8) {
          e8[b * ld8 + j0 + o + t] = uint8_t(sm > 0 ? sm : 0);
          e8[plane8 + b * ld8 + j0 + o + t] = uint8_t(sm < 0 ? -sm : 0);
        }
      }
    }
  }
  // bit planes of the plus / minus magnitudes, packed four bytes to a word
  // once per (batch row, 16 columns) as in k_prep_x (full 32-byte sectors);
  // none in volts mode (no plane buffer: the fp64 kernels read the codes)
  if (A == nullptr) return;
  constexpr int Q = kPrepTI / 16;
  for (int e = threadIdx.x; e < kPrepTB * Q; e += blockDim.x) {
    const int q = e % Q, r = e / Q;
    const int64_t b = b0 + r;
    if (b >= M || !plane_sector_live(q * 16, nlive)) continue;
    uint32_t pl[4], ph[4], ml[4], mh[4];  // plus / minus magnitudes: low and high bytes
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const int sm = cs[r][q * 16 + q4 * 4 + qq];
        const uint32_t p = uint32_t(sm > 0 ? sm : 0), m = uint32_t(sm < 0 ? -sm : 0);
        a0 |= (p & 0xffu) << (8 * qq);
        a1 |= (p >> 8) << (8 * qq);
        a2 |= (m & 0xffu) << (8 * qq);
        a3 |= (m >> 8) << (8 * qq);
      }
      pl[q4] = a0;
      ph[q4] = a1;
      ml[q4] = a2;
      mh[q4] = a3;
    }
    uint8_t* p0 = A + (b * g.TPe * 2) * g.NB + c0 + q * 16;
    for (int k = 0; k < g.TPe; ++k) {
#pragma unroll
      for (int phi = 0; phi < 2; ++phi, p0 += g.NB) {
        uint32_t w0[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t lo = phi ? ml[q4] : pl[q4], hi = phi ? mh[q4] : ph[q4];
          w0[q4] = (k < 8 ? lo >> k : hi >> (k - 8)) & 0x01010101u;
        }
        *reinterpret_cast<uint4*>(p0) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
        *reinterpret_cast<uint4*>(p0 + rowsB * g.NB) =
            make_uint4(w0[0] * 255u, w0[1] * 255u, w0[2] * 255u, w0[3] * 255u);
      }
    }
  }
}

__global__ void k_absmax_to_se(DevScalars* sc, const unsigned long long* bits) {
  sc->se = __longlong_as_double((long long)*bits);
}

void launch_prep_dy(const xbs_core* c, const double* d_dy, int64_t M, cudaStream_t st) {
  cudaMemsetAsync(&c->d_sc->wmax_in, 0, sizeof(unsigned long long), st);
  launch_absmax(d_dy, M * c->g.N, &c->d_sc->wmax_in, st);
  k_absmax_to_se<<<1, 1, 0, st>>>(c->d_sc, &c->d_sc->wmax_in);
  const int64_t rowsB = rows_bwd(M, c->g.TPe);
  const int64_t pad0 = M * c->g.TPe * 2;
  if (c->d_Ab && rowsB > pad0) {
    cudaMemsetAsync(c->d_Ab + pad0 * c->g.NB, 0, size_t(rowsB - pad0) * c->g.NB, st);
    cudaMemsetAsync(c->d_Ab + (rowsB + pad0) * c->g.NB, 0, size_t(rowsB - pad0) * c->g.NB, st);
  }
  if (M == 0) return;
  const int64_t plane8 = c->M_cap8 * c->NA;
  if (c->d_e8) {
    const int64_t Mp = ((M + 127) / 128) * 128;
    if (Mp > M) {
      cudaMemsetAsync(c->d_e8 + M * c->NA, 0, size_t(Mp - M) * c->NA, st);
      cudaMemsetAsync(c->d_e8 + plane8 + M * c->NA, 0, size_t(Mp - M) * c->NA, st);
    }
  }
  const int64_t nbt = (M + kPrepTB - 1) / kPrepTB;
  for (int64_t bt0 = 0; bt0 < nbt; bt0 += 65535) {
    const dim3 grid(unsigned((c->g.NB + kPrepTI - 1) / kPrepTI), unsigned(std::min<int64_t>(nbt - bt0, 65535)));
    k_prep_dy<<<grid, 256, 0, st>>>(c->g, d_dy, M, rowsB, double((1 << c->opt.error_bits) - 1), c->d_sc,
                                       c->d_ecodes, c->d_Ab, c->d_e8, plane8, c->NA, bt0);
  }
}

// ---------------------------------------------------------------------- dW
// Exact integer outer product: dW = ((S * sx) * step_e) / gd.
template <class CT>
__global__ void k_dw(Geo g, int64_t M, double sx, double lev_e, double gd, const CT* __restrict__ xc,
                     const int32_t* __restrict__ ec, DevScalars* __restrict__ sc, double* __restrict__ dW) {
  const double se = sc->se;
  const double step_e = se > 0 ? se / lev_e : 0.0;
  const int64_t n = int64_t(g.K) * g.N;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(t / g.N), j = int(t % g.N);
    int64_t S = 0;
    for (int64_t b = 0; b < M; ++b) S += int64_t(xc[b * g.K + i]) * int64_t(ec[b * g.N + j]);
    const double v = ((double(S) * sx) * step_e) / gd;
    if (!isfinite(v)) sc->dw_nonfinite = 1;
    dW[t] = v;
  }
}

void launch_dw(const xbs_core* c, int64_t M, double grad_divisor, cudaStream_t st) {
  const int64_t n = int64_t(c->g.K) * c->g.N;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
  if (c->d_xcodes32)
    k_dw<<<blocks, 256, 0, st>>>(c->g, M, c->sx, c->lev_e, grad_divisor, c->d_xcodes32, c->d_ecodes, c->d_sc,
                                 c->d_dW);
  else
    k_dw<<<blocks, 256, 0, st>>>(c->g, M, c->sx, c->lev_e, grad_divisor, c->d_xcodes, c->d_ecodes, c->d_sc, c->d_dW);
}

// ------------------------------------------------------ general converters
// Multi-bit DAC streams, DAC / ADC transfer tables, ADC resolutions above 16
// bits and non-power-of-two DAC full scales (layers.cpp:52-64, 236-241,
// 316-331; converters.cpp:28-35, 70-88): the column currents are no longer
// integers on the snapped grid, so these layers run exact CUDA-core kernels
// that follow the reference's fp64 expression order term by term -- I =
// sum over ascending crossbar rows (columns, backward) of volts(digit) * g
// on the snapped conductances, the ADC as adc_quantize, then the same
// accumulation order as layers.cpp:246-283 / 340-378 -- so the outputs are
// bit-identical to the oracle's restatement.  No tensor-core path exists for
// them (the radix-255 operands need 1-bit digits and power-of-two volts).
__device__ __forceinline__ double adc_volts(const VoltsP& v, double I, double i_fs) {
  if (v.passthrough) return I;
  if (v.tr_len > 0) {  // converters.cpp:76-82: highest threshold not exceeding I
    int lo = 0, hi = v.tr_len;  // first index with transfer[idx] > I
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (v.adc_tr[mid] > I) hi = mid;
      else lo = mid + 1;
    }
    if (lo == 0) return 0.0;
    const unsigned long long code = (unsigned long long)(lo - 1);
    return double(code < v.maxcode ? code : v.maxcode);
  }
  const double scaled = __dmul_rn(__ddiv_rn(I, i_fs), v.maxc_d);  // converters.cpp:85-87
  if (scaled >= v.maxc_d) return v.maxc_d;
  return double(llround(scaled));
}

__device__ __forceinline__ double g_snapped(const Geo& g, const uint8_t* digits, int e, int s, int p, int tr, int tc,
                                            int r, int c) {
  return ldexp(double(load_q(digits, g, s, p, tr, tc, r, c)), -e);  // exact: q 2^-e
}

__global__ void k_fwd_volts(Geo g, VoltsP v, int e, int64_t M, const uint32_t* __restrict__ xc,
                            const uint8_t* __restrict__ digits, double k_out, double* __restrict__ y) {
  const int64_t n = M * g.N;
  const int nx = g.Ti / v.sb, mask = (1 << v.sb) - 1;
  const double stream_base = double(1 << v.sb);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = t % M;
    const int col = int(t / M);
    const int tc = col / g.tile_cols, c = col % g.tile_cols;
    double out = 0.0;
    for (int tr = 0; tr < g.GR; ++tr) {
      const int rows = min(g.tile_rows, g.K - tr * g.tile_rows);  // padded rows carry volts(0) = 0
      double tile = 0.0;
      for (int s = 0; s < g.S; ++s) {
        const double sw = ldexp(1.0, s * g.db);  // pow(2^db, s)
        for (int p = 0; p < 2; ++p) {
          double acc = 0.0, wk = 1.0;
          for (int k = 0; k < nx; ++k) {
            double I = 0.0;
            for (int r = 0; r < rows; ++r) {
              const int d = (int(xc[b * g.K + tr * g.tile_rows + r]) >> (k * v.sb)) & mask;
              if (d) I = __dadd_rn(I, __dmul_rn(v.lut[d], g_snapped(g, digits, e, s, p, tr, tc, r, c)));
            }
            acc = __dadd_rn(acc, __dmul_rn(wk, adc_volts(v, I, v.i_fs)));
            wk = __dmul_rn(wk, stream_base);
          }
          tile = __dadd_rn(tile, __dmul_rn(p == 0 ? sw : -sw, acc));
        }
      }
      out = __dadd_rn(out, tile);
    }
    y[int64_t(col) * M + b] = __dmul_rn(out, k_out);
  }
}

__global__ void k_bwd_volts(Geo g, VoltsP v, int e, int64_t M, const int32_t* __restrict__ ec,
                            const uint8_t* __restrict__ digits, double F, double vu, double ifs_fac, int adc_scaled,
                            double lev_e, const DevScalars* __restrict__ sc, double* __restrict__ dx) {
  const double se = sc->se;
  const double step_e = se > 0 ? se / lev_e : 0.0;
  double k_out = step_e * F / vu;  // layers.cpp:375-377
  if (adc_scaled) k_out *= ifs_fac;
  const int64_t n = M * g.K;
  const int ne = g.Te / v.sb, mask = (1 << v.sb) - 1;
  const double stream_base = double(1 << v.sb);
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = t % M;
    const int i = int(t / M);
    const int tr = i / g.tile_rows, r = i % g.tile_rows;
    double acc_dx = 0.0;
    if (se > 0)
      for (int tc = 0; tc < g.GC; ++tc) {
        const int cols = min(g.tile_cols, g.N - tc * g.tile_cols);
        double tile = 0.0;
        for (int s = 0; s < g.S; ++s) {
          const double sw = ldexp(1.0, s * g.db);
          double ap = 0.0, an = 0.0, wk = 1.0;
          for (int k = 0; k < ne; ++k) {
            double Ipp = 0.0, Imn = 0.0, Ipn = 0.0, Imp = 0.0;  // (vp, gp) (vm, gn) (vp, gn) (vm, gp)
            for (int c = 0; c < cols; ++c) {
              const int code = ec[b * g.N + tc * g.tile_cols + c];
              const int dp = ((code > 0 ? code : 0) >> (k * v.sb)) & mask;
              const int dm = ((code < 0 ? -code : 0) >> (k * v.sb)) & mask;
              if (dp) {
                const double vp = v.lut[dp];
                Ipp = __dadd_rn(Ipp, __dmul_rn(vp, g_snapped(g, digits, e, s, 0, tr, tc, r, c)));
                Ipn = __dadd_rn(Ipn, __dmul_rn(vp, g_snapped(g, digits, e, s, 1, tr, tc, r, c)));
              }
              if (dm) {
                const double vm = v.lut[dm];
                Imn = __dadd_rn(Imn, __dmul_rn(vm, g_snapped(g, digits, e, s, 1, tr, tc, r, c)));
                Imp = __dadd_rn(Imp, __dmul_rn(vm, g_snapped(g, digits, e, s, 0, tr, tc, r, c)));
              }
            }
            ap = __dadd_rn(ap, __dmul_rn(wk, __dadd_rn(adc_volts(v, Ipp, v.i_fs_b), adc_volts(v, Imn, v.i_fs_b))));
            an = __dadd_rn(an, __dmul_rn(wk, __dadd_rn(adc_volts(v, Ipn, v.i_fs_b), adc_volts(v, Imp, v.i_fs_b))));
            wk = __dmul_rn(wk, stream_base);
          }
          tile = __dadd_rn(tile, __dmul_rn(sw, __dsub_rn(ap, an)));
        }
        acc_dx = __dadd_rn(acc_dx, tile);
      }
    dx[int64_t(i) * M + b] = __dmul_rn(acc_dx, k_out);
  }
}

void launch_fwd_volts(const xbs_core* c, int64_t M, double* d_y, cudaStream_t st) {
  const int64_t n = M * c->g.N;
  if (n == 0) return;
  const int blocks = int(std::min<int64_t>((n + 127) / 128, 148 * 64));
  k_fwd_volts<<<blocks, 128, 0, st>>>(c->g, c->volts, c->rp.snap_e, M, c->d_xcodes32, c->d_digits, c->k_out_fwd,
                                      d_y);
}

void launch_bwd_volts(const xbs_core* c, int64_t M, double* d_dx, cudaStream_t st) {
  const int64_t n = M * c->g.K;
  if (n == 0) return;
  const int blocks = int(std::min<int64_t>((n + 127) / 128, 148 * 64));
  k_bwd_volts<<<blocks, 128, 0, st>>>(c->g, c->volts, c->rp.snap_e, M, c->d_ecodes, c->d_digits, c->F, c->vu,
                                      c->ifs_fac_b, c->adc_scaled ? 1 : 0, c->lev_e, c->d_sc, d_dx);
}

// --------------------------------------------------------------- SIMT VMM
__device__ __forceinline__ int64_t adc_apply(const AdcP& a, int64_t n, unsigned long long* conv) {
  if (a.passthrough) return n;
  const double I = ldexp(double(n), a.sh);
  const double scaled = I / a.i_fs * a.maxc_d;
  if (scaled >= a.maxc_d) return a.maxc;
  return llround(scaled);
}

// forward (layers.cpp:246-283): one thread per (b, logical output column).
// Pass-through sensing (adc.bits = 0, or auto-calibration batches): the
// currents themselves are summed, in fp64, so the totals follow the
// reference's accumulation order exactly (units of 2^sh; every product is by
// a power of two, only the additions round):
//   forward  (layers.cpp:246-270): out += tile_out over tr; tile_out +=
//            +-sw * acc over (s, p); acc += wk * I over k
//   backward (layers.cpp:340-366): dx += tile_dx over tc; tile_dx += sw *
//            (acc_pos - acc_neg) over s; acc_pos += wk * (I_pp + I_mn) over k
__device__ double fwd_passthrough(const Geo& g, const uint8_t* A, const uint8_t* digits, int64_t b, int tc, int c) {
  double out = 0.0;
  for (int tr = 0; tr < g.GR; ++tr) {
    double tile = 0.0;
    for (int s = 0; s < g.S; ++s)
      for (int p = 0; p < 2; ++p) {
        double acc = 0.0;
        for (int k = 0; k < g.Ti; ++k) {
          const uint8_t* arow = A + (b * g.TPi + k) * g.KI + size_t(tr) * g.R;
          int64_t nn = 0;
          for (int r = 0; r < g.tile_rows; ++r)
            if (arow[r]) nn += load_q(digits, g, s, p, tr, tc, r, c);
          acc = __dadd_rn(acc, ldexp(double(nn), k));
        }
        const double w = ldexp(acc, s * g.db);
        tile = __dadd_rn(tile, p == 0 ? w : -w);
      }
    out = __dadd_rn(out, tile);
  }
  return out;
}

__global__ void k_fwd_simt(Geo g, AdcP a, int64_t M, int64_t rowsF, const uint8_t* __restrict__ A,
                           const uint8_t* __restrict__ digits, double k_out, double* __restrict__ y) {
  const int64_t n = M * g.N;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = t % M;
    const int col = int(t / M);
    const int tc = col / g.tile_cols, c = col % g.tile_cols;
    if (a.passthrough) {
      y[int64_t(col) * M + b] = ldexp(fwd_passthrough(g, A, digits, b, tc, c), a.sh) * k_out;
      continue;
    }
    int64_t total = 0;
    for (int k = 0; k < g.Ti; ++k) {
      const uint8_t* arow = A + (b * g.TPi + k) * g.KI;
      for (int tr = 0; tr < g.GR; ++tr)
        for (int s = 0; s < g.S; ++s)
          for (int p = 0; p < 2; ++p) {
            int64_t nn = 0;
            for (int r = 0; r < g.tile_rows; ++r)
              if (arow[tr * g.R + r]) nn += load_q(digits, g, s, p, tr, tc, r, c);
            const int64_t v = adc_apply(a, nn, nullptr);
            const int64_t w = (v << (s * g.db)) << k;
            total += p == 0 ? w : -w;
          }
    }
    y[int64_t(col) * M + b] = double(total) * k_out;
  }
}

void launch_fwd_simt(const xbs_core* c, int64_t M, double* d_y, cudaStream_t st) {
  const int64_t n = M * c->g.N;
  if (n == 0) return;
  const int blocks = int(std::min<int64_t>((n + 127) / 128, 148 * 64));
  const int64_t rowsF = rows_fwd(M, c->g.TPi);
  k_fwd_simt<<<blocks, 128, 0, st>>>(c->g, c->adc, M, rowsF, c->d_Af, c->d_digits, c->k_out_fwd, d_y);
}

// backward (layers.cpp:339-379): one thread per (b, logical input row i).
__global__ void k_bwd_simt(Geo g, AdcP a, int64_t M, const uint8_t* __restrict__ A, const uint8_t* __restrict__ digits,
                           double F, double vu, double ifs_fac, int adc_scaled, double lev_e,
                           const DevScalars* __restrict__ sc, double* __restrict__ dx) {
  const double se = sc->se;
  const double step_e = se > 0 ? se / lev_e : 0.0;
  double k_out = step_e * F / vu;  // layers.cpp:375
  if (adc_scaled) k_out *= ifs_fac;
  const int64_t n = M * g.K;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = t % M;
    const int i = int(t / M);
    const int tr = i / g.tile_rows, r = i % g.tile_rows;
    if (a.passthrough) {
      double acc_dx = 0.0;
      if (se > 0)
        for (int tc = 0; tc < g.GC; ++tc) {
          double tile = 0.0;
          for (int s = 0; s < g.S; ++s) {
            double apos = 0.0, aneg = 0.0;
            for (int k = 0; k < g.Te; ++k) {
              const uint8_t* ap = A + ((b * g.TPe + k) * 2 + 0) * g.NB + size_t(tc) * g.C;
              const uint8_t* am = A + ((b * g.TPe + k) * 2 + 1) * g.NB + size_t(tc) * g.C;
              int64_t pp = 0, mn = 0, pn = 0, mp = 0;
              for (int c = 0; c < min(g.tile_cols, g.NB - tc * g.C); ++c) {
                const int64_t qp = load_q(digits, g, s, 0, tr, tc, r, c), qn = load_q(digits, g, s, 1, tr, tc, r, c);
                if (ap[c]) { pp += qp; pn += qn; }
                if (am[c]) { mn += qn; mp += qp; }
              }
              apos = __dadd_rn(apos, ldexp(__dadd_rn(double(pp), double(mn)), k));
              aneg = __dadd_rn(aneg, ldexp(__dadd_rn(double(pn), double(mp)), k));
            }
            tile = __dadd_rn(tile, ldexp(__dsub_rn(apos, aneg), s * g.db));
          }
          acc_dx = __dadd_rn(acc_dx, tile);
        }
      dx[int64_t(i) * M + b] = ldexp(acc_dx, a.sh) * k_out;
      continue;
    }
    int64_t total = 0;
    if (se > 0)
      for (int k = 0; k < g.Te; ++k) {
        const uint8_t* ap = A + ((b * g.TPe + k) * 2 + 0) * g.NB;
        const uint8_t* am = A + ((b * g.TPe + k) * 2 + 1) * g.NB;
        for (int tc = 0; tc < g.GC; ++tc)
          for (int s = 0; s < g.S; ++s) {
            int64_t pp = 0, mn = 0, pn = 0, mp = 0;
            for (int c = 0; c < min(g.tile_cols, g.NB - tc * g.C); ++c) {
              const int64_t qp = load_q(digits, g, s, 0, tr, tc, r, c), qn = load_q(digits, g, s, 1, tr, tc, r, c);
              if (ap[tc * g.C + c]) { pp += qp; pn += qn; }
              if (am[tc * g.C + c]) { mn += qn; mp += qp; }
            }
            const int64_t v = adc_apply(a, pp, nullptr) + adc_apply(a, mn, nullptr) - adc_apply(a, pn, nullptr) -
                              adc_apply(a, mp, nullptr);
            total += (v << (s * g.db)) << k;
          }
      }
    dx[int64_t(i) * M + b] = double(total) * k_out;
  }
}

void launch_bwd_simt(const xbs_core* c, int64_t M, double* d_dx, cudaStream_t st) {
  const int64_t n = M * c->g.K;
  if (n == 0) return;
  const int blocks = int(std::min<int64_t>((n + 127) / 128, 148 * 64));
  k_bwd_simt<<<blocks, 128, 0, st>>>(c->g, c->adc_b, M, c->d_Ab, c->d_digits, c->F, c->vu, c->ifs_fac_b,
                                      c->adc_scaled ? 1 : 0, c->lev_e, c->d_sc, d_dx);
}

// ------------------------------------------------------ fully-ideal path
// y = x_values * wimp (layers.cpp:226), ascending k, unfused mul/add.
template <class CT>
__global__ void k_fwd_ideal(Geo g, int64_t M, double sx, const CT* __restrict__ xc,
                            const double* __restrict__ w, double* __restrict__ y) {
  const int64_t n = M * g.N;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = t % M;
    const int j = int(t / M);
    double a = 0.0;
    for (int k = 0; k < g.K; ++k) a = a + (double(xc[b * g.K + k]) * sx) * w[int64_t(k) * g.N + j];
    y[int64_t(j) * M + b] = a;
  }
}

void launch_fwd_ideal(const xbs_core* c, int64_t M, double* d_y, cudaStream_t st) {
  const int64_t n = M * c->g.N;
  if (n == 0) return;
  const int blocks = int(std::min<int64_t>((n + 127) / 128, 148 * 64));
  if (c->d_xcodes32) k_fwd_ideal<<<blocks, 128, 0, st>>>(c->g, M, c->sx, c->d_xcodes32, c->d_wimp, d_y);
  else k_fwd_ideal<<<blocks, 128, 0, st>>>(c->g, M, c->sx, c->d_xcodes, c->d_wimp, d_y);
}

// dx = dy_q * wimp^T (layers.cpp:307), dy_q = (sign*mag)*step_e (layers.cpp:301-302)
__global__ void k_bwd_ideal(Geo g, int64_t M, double lev_e, const int32_t* __restrict__ ec,
                            const DevScalars* __restrict__ sc, const double* __restrict__ w, double* __restrict__ dx) {
  const double se = sc->se;
  const double step_e = se > 0 ? se / lev_e : 0.0;
  const int64_t n = M * g.K;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = t % M;
    const int i = int(t / M);
    double a = 0.0;
    for (int j = 0; j < g.N; ++j) {
      const int e = ec[b * g.N + j];
      const int sg = e > 0 ? 1 : (e < 0 ? -1 : 0);
      const double dq = double(sg) * double(e < 0 ? -e : e) * step_e;
      a = a + dq * w[int64_t(i) * g.N + j];
    }
    dx[int64_t(i) * M + b] = a;
  }
}

void launch_bwd_ideal(const xbs_core* c, const double* d_dy, int64_t M, double* d_dx, cudaStream_t st) {
  (void)d_dy;
  const int64_t n = M * c->g.K;
  if (n == 0) return;
  const int blocks = int(std::min<int64_t>((n + 127) / 128, 148 * 64));
  k_bwd_ideal<<<blocks, 128, 0, st>>>(c->g, M, c->lev_e, c->d_ecodes, c->d_sc, c->d_wimp, d_dx);
}

}  // namespace xbs
