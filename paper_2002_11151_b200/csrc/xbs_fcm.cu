// FCM regeneration (fcm.cpp:18-224) and the interp-FCM distortion cache
// (distortion.cpp:10-48) on the GPU.
//
// One CTA per (slice, polarity, tile) job, persistent over the jobs.  The
// working conductances of the tile (master polarity + variation,
// mapping.cpp:39-58, padded cells included as in mapping.cpp:60-67) are
// staged in a per-CTA scratch area together with the top / bottom node
// voltages; each sweep of the block Gauss-Seidel solves every row ladder
// (thread i runs row i's Thomas recurrence) and then every column ladder
// (thread j), in exactly the reference's operation order, so the converted
// conductances are bit-identical to the oracle's restatement.  Convergence
// is the max node-voltage change over the tile (block reduction) against
// tol * v_fs.  The result G = clamp(g (v_top - v_bot) / v_fs, 0, g) is then
// snapped and written as radix-255 digits like every other engine.
//
// Scratch layouts (fp64): G and V_top column-major ([j][i]: row threads
// coalesce), V_bot row-major ([i][j]: column threads coalesce), and the
// Thomas coefficients [step][thread].  Each thread streams its own row /
// column through L1 in the other sweep.
#include <cuda_runtime.h>

#include <algorithm>

#include "xbs_internal.cuh"

namespace xbs {

namespace {

__device__ __forceinline__ double working_g(const Geo& g, const RegenP& rp, const double* __restrict__ master, int s,
                                            int p, int64_t i, int64_t j) {
  const double u = master[(size_t(s) * g.Kp + i) * g.Np + j];
  const double up = p == 0 ? u : -u;
  double gv = (up > 0.0 ? up : 0.0) + rp.g_min;  // mapping.cpp:39-45
  if (rp.sigma != 0.0) gv = fmin(gv * rp.varm[(uint64_t(s) * 2 + p) * rp.kpnp + uint64_t(i) * g.Np + j], rp.g_max);
  return gv;
}

__device__ __forceinline__ void store_q(uint8_t* digits, const Geo& g, int s, int p, int tr, int tc, int r, int c,
                                        uint32_t q) {
  const uint32_t lo = q % 65025u, hi = q / 65025u;
  const size_t off = size_t(r) * g.C + c;
  digits[g.tile_digit_offset(s, p, tr, tc, 0) + off] = uint8_t(lo % 255u);
  digits[g.tile_digit_offset(s, p, tr, tc, 1) + off] = uint8_t(lo / 255u);
  digits[g.tile_digit_offset(s, p, tr, tc, 2) + off] = uint8_t(hi);
}

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double m = red[0];
  for (int k = 1; k < nw; ++k) m = fmax(m, red[k]);
  return m;
}

}  // namespace

// mode 0: fcm; mode 1: interp refresh (fcm or aam base) -- also stores the
// distortion profile d, g at refresh and the converted g (fp64, [s][p][Kp][Np])
__global__ void __launch_bounds__(256) k_fcm_regen(Geo g, RegenP rp, FcmP f, const double* __restrict__ master,
                                                   uint8_t* __restrict__ digits, double* __restrict__ scratch,
                                                   double* __restrict__ cache_d, double* __restrict__ cache_g,
                                                   double* __restrict__ cache_gn, DevScalars* sc, int mode) {
  __shared__ double red[8];
  const int TR = g.tile_rows, TC = g.tile_cols;
  const int MX = TR > TC ? TR : TC;
  const int64_t njobs = int64_t(g.S) * 2 * g.GR * g.GC;
  double* G = scratch + size_t(blockIdx.x) * (3 * size_t(TR) * TC + 5 * size_t(MX) * blockDim.x);
  double* VT = G + size_t(TR) * TC;
  double* VB = VT + size_t(TR) * TC;
  double* DW = VB + size_t(TR) * TC;
  // The Thomas denominators and c coefficients depend on the conductances
  // only, so they are computed in the first sweep and reused (the values
  // are the ones every sweep of the reference recomputes, bit for bit).
  double* CWR = DW + size_t(MX) * blockDim.x;   // rows: c_j
  double* DNR = CWR + size_t(MX) * blockDim.x;  // rows: denom_j
  double* CWC = DNR + size_t(MX) * blockDim.x;  // columns: c_i
  double* DNC = CWC + size_t(MX) * blockDim.x;  // columns: denom_i
  const int t = threadIdx.x, nt = blockDim.x;
  const bool zero_par = f.r_row == 0.0 && f.r_col == 0.0 && f.r_source == 0.0 && f.r_sense == 0.0;

  for (int64_t job = blockIdx.x; job < njobs; job += gridDim.x) {
    const int tc = int(job % g.GC), tr = int((job / g.GC) % g.GR);
    const int p = int((job / (int64_t(g.GC) * g.GR)) % 2), s = int(job / (int64_t(g.GC) * g.GR * 2));
    // stage the working conductances and the initial node voltages
    for (int e = t; e < TR * TC; e += nt) {
      const int i = e % TR, j = e / TR;
      G[size_t(j) * TR + i] = working_g(g, rp, master, s, p, int64_t(tr) * TR + i, int64_t(tc) * TC + j);
      VT[size_t(j) * TR + i] = f.v_fs;  // v_in = v_fs on every row (layers.cpp:95-97 defaults)
      VB[size_t(i) * TC + j] = 0.0;
    }
    __syncthreads();
    bool converged = zero_par || !f.use_fcm;
    double residual = 0.0;
    int sweep = 0;
    while (!converged && sweep < f.max_iter) {
      ++sweep;
      double delta = 0.0;
      // ---- rows (fcm.cpp:18-46 / 78-92): top nodes, bottom nodes fixed
      if (t < TR) {
        const int i = t;
        if (f.r_row != 0.0) {
          const double g_seg = 1.0 / f.r_row;
          const double g_drv = 1.0 / (f.r_source + f.r_row);
          double prev_c = 0.0, prev_d = 0.0;
          if (sweep == 1) {
            for (int j = 0; j < TC; ++j) {
              const double gij = G[size_t(j) * TR + i];
              const double gl = (j == 0) ? g_drv : g_seg;
              const double gr = (j < TC - 1) ? g_seg : 0.0;
              const double diag = gl + gr + gij;
              double rhs = gij * VB[size_t(i) * TC + j];
              if (j == 0) rhs += gl * f.v_fs;
              const double denom = diag - gl * prev_c;
              prev_c = gr / denom;
              prev_d = (rhs + gl * prev_d) / denom;
              CWR[size_t(j) * nt + t] = prev_c;
              DNR[size_t(j) * nt + t] = denom;
              DW[size_t(j) * nt + t] = prev_d;
            }
          } else {
#pragma unroll 4
            for (int j = 0; j < TC; ++j) {
              const double gij = G[size_t(j) * TR + i];
              const double gl = (j == 0) ? g_drv : g_seg;
              double rhs = gij * VB[size_t(i) * TC + j];
              if (j == 0) rhs += gl * f.v_fs;
              prev_d = (rhs + gl * prev_d) / DNR[size_t(j) * nt + t];
              DW[size_t(j) * nt + t] = prev_d;
            }
          }
          double x = DW[size_t(TC - 1) * nt + t];
          delta = fmax(delta, fabs(x - VT[size_t(TC - 1) * TR + i]));
          VT[size_t(TC - 1) * TR + i] = x;
          for (int j = TC - 2; j >= 0; --j) {
            x = DW[size_t(j) * nt + t] + CWR[size_t(j) * nt + t] * x;
            delta = fmax(delta, fabs(x - VT[size_t(j) * TR + i]));
            VT[size_t(j) * TR + i] = x;
          }
        } else {
          double v;
          if (f.r_source == 0.0) {
            v = f.v_fs;
          } else {
            double num = f.v_fs / f.r_source, den = 1.0 / f.r_source;
            for (int j = 0; j < TC; ++j) {
              const double gij = G[size_t(j) * TR + i];
              num += gij * VB[size_t(i) * TC + j];
              den += gij;
            }
            v = num / den;
          }
          for (int j = 0; j < TC; ++j) {
            delta = fmax(delta, fabs(v - VT[size_t(j) * TR + i]));
            VT[size_t(j) * TR + i] = v;
          }
        }
      }
      __syncthreads();
      // ---- columns (fcm.cpp:48-76 / 94-108): bottom nodes, top nodes fixed
      if (t < TC) {
        const int j = t;
        if (f.r_col != 0.0) {
          const double g_seg = 1.0 / f.r_col;
          const double g_foot = 1.0 / (f.r_col + f.r_sense);
          double prev_c = 0.0, prev_d = 0.0;
          if (sweep == 1) {
            for (int i = 0; i < TR; ++i) {
              const double gij = G[size_t(j) * TR + i];
              const double gu = (i > 0) ? g_seg : 0.0;
              const double gd = (i < TR - 1) ? g_seg : g_foot;
              const double diag = gu + gd + gij;
              const double rhs = gij * VT[size_t(j) * TR + i];
              const double denom = diag - gu * prev_c;
              prev_c = gd / denom;
              prev_d = (rhs + gu * prev_d) / denom;
              CWC[size_t(i) * nt + t] = prev_c;
              DNC[size_t(i) * nt + t] = denom;
              DW[size_t(i) * nt + t] = prev_d;
            }
          } else {
#pragma unroll 4
            for (int i = 0; i < TR; ++i) {
              const double gij = G[size_t(j) * TR + i];
              const double gu = (i > 0) ? g_seg : 0.0;
              const double rhs = gij * VT[size_t(j) * TR + i];
              prev_d = (rhs + gu * prev_d) / DNC[size_t(i) * nt + t];
              DW[size_t(i) * nt + t] = prev_d;
            }
          }
          double x = DW[size_t(TR - 1) * nt + t];
          delta = fmax(delta, fabs(x - VB[size_t(TR - 1) * TC + j]));
          VB[size_t(TR - 1) * TC + j] = x;
          for (int i = TR - 2; i >= 0; --i) {
            x = DW[size_t(i) * nt + t] + CWC[size_t(i) * nt + t] * x;
            delta = fmax(delta, fabs(x - VB[size_t(i) * TC + j]));
            VB[size_t(i) * TC + j] = x;
          }
        } else {
          double v = 0.0;
          if (f.r_sense != 0.0) {
            double num = 0.0, den = 1.0 / f.r_sense;
            for (int i = 0; i < TR; ++i) {
              const double gij = G[size_t(j) * TR + i];
              num += gij * VT[size_t(j) * TR + i];
              den += gij;
            }
            v = num / den;
          }
          for (int i = 0; i < TR; ++i) {
            delta = fmax(delta, fabs(v - VB[size_t(i) * TC + j]));
            VB[size_t(i) * TC + j] = v;
          }
        }
      }
      residual = block_max(delta, red) / f.v_fs;  // also the barrier before the next sweep
      converged = residual <= f.tol;
    }
    if (!converged && t == 0) {
      atomicAdd(&sc->fcm_fail, 1u);
      atomicMax(&sc->fcm_residual, (unsigned long long)__double_as_longlong(residual));
    }
    // ---- G_non = clamp(g (v_top - v_bot) / v_fs, 0, g) (fcm.cpp:194-201)
    for (int e = t; e < TR * TC; e += nt) {
      const int i = e % TR, j = e / TR;
      const double gij = G[size_t(j) * TR + i];
      double gn;
      if (!f.use_fcm) {  // interp with the AAM base (aam.cpp:14-31)
        const double rpath = f.r_source + double(j + 1) * f.r_row + double(TR - i) * f.r_col + f.r_sense;
        gn = (gij == 0.0) ? 0.0 : (rpath == 0.0 ? gij : __drcp_rn(__dadd_rn(__drcp_rn(gij), rpath)));
      } else if (zero_par) {
        gn = gij;
      } else {
        const double v_dev = VT[size_t(j) * TR + i] - VB[size_t(i) * TC + j];
        const double eff = gij * v_dev / f.v_fs;
        gn = fmin(fmax(eff, 0.0), gij);
      }
      const int64_t gi = int64_t(tr) * TR + i, gj = int64_t(tc) * TC + j;
      if (mode == 1) {  // distortion.cpp:10-30
        const size_t ci = (size_t(s) * 2 + p) * rp.kpnp + size_t(gi) * g.Np + size_t(gj);
        cache_d[ci] = (gij == 0.0) ? 0.0 : (gij - gn) / gij;
        cache_g[ci] = gij;
        cache_gn[ci] = gn;
      }
      store_q(digits, g, s, p, tr, tc, i, j, __double2uint_rn(__dmul_rn(gn, rp.snap_scale)));
    }
    __syncthreads();
  }
}

// distortion.cpp:32-48: between refreshes G = g (1 - d), or the stored
// conversion when the whole tile is unchanged since the refresh.
__global__ void __launch_bounds__(256) k_interp_apply(Geo g, RegenP rp, const double* __restrict__ master,
                                                      uint8_t* __restrict__ digits,
                                                      const double* __restrict__ cache_d,
                                                      const double* __restrict__ cache_g,
                                                      const double* __restrict__ cache_gn) {
  const int TR = g.tile_rows, TC = g.tile_cols;
  const int64_t njobs = int64_t(g.S) * 2 * g.GR * g.GC;
  for (int64_t job = blockIdx.x; job < njobs; job += gridDim.x) {
    const int tc = int(job % g.GC), tr = int((job / g.GC) % g.GR);
    const int p = int((job / (int64_t(g.GC) * g.GR)) % 2), s = int(job / (int64_t(g.GC) * g.GR * 2));
    const size_t base = (size_t(s) * 2 + p) * rp.kpnp;
    int same = 1;
    for (int e = threadIdx.x; e < TR * TC; e += blockDim.x) {
      const int i = e % TR, j = e / TR;
      const int64_t gi = int64_t(tr) * TR + i, gj = int64_t(tc) * TC + j;
      same &= working_g(g, rp, master, s, p, gi, gj) == cache_g[base + size_t(gi) * g.Np + size_t(gj)];
    }
    same = __syncthreads_and(same);
    for (int e = threadIdx.x; e < TR * TC; e += blockDim.x) {
      const int i = e % TR, j = e / TR;
      const int64_t gi = int64_t(tr) * TR + i, gj = int64_t(tc) * TC + j;
      const size_t ci = base + size_t(gi) * g.Np + size_t(gj);
      const double gn = same ? cache_gn[ci] : working_g(g, rp, master, s, p, gi, gj) * (1.0 - cache_d[ci]);
      store_q(digits, g, s, p, tr, tc, i, j, __double2uint_rn(__dmul_rn(gn, rp.snap_scale)));
    }
    __syncthreads();
  }
}

void launch_fcm_regen(xbs_core* c, bool refresh_interp, cudaStream_t st) {
  const Geo& g = c->g;
  const int MX = std::max(g.tile_rows, g.tile_cols);
  const int nt = ((MX + 31) / 32) * 32;
  const int64_t njobs = int64_t(g.S) * 2 * g.GR * g.GC;
  // Latency-bound serial recurrences with a ~1 MB per-tile working set: 4
  // CTAs per SM is where more tiles in flight stop paying (ncu: L2-miss bound).
  const int grid = int(std::min<int64_t>(njobs, 4 * 148));
  const size_t per = 3 * size_t(g.tile_rows) * g.tile_cols + 5 * size_t(MX) * nt;
  const size_t need = per * size_t(grid) * sizeof(double);
  if (c->fcm_scratch_bytes < need) {
    cudaFree(c->d_fcm_scratch);
    ck_cuda(cudaMalloc(&c->d_fcm_scratch, need), "cudaMalloc fcm scratch");
    c->fcm_scratch_bytes = need;
  }
  FcmP f = c->fcm;
  f.use_fcm = (c->opt.engine == XBS_ENGINE_FCM || c->opt.interp_base == XBS_ENGINE_FCM) ? 1 : 0;
  k_fcm_regen<<<grid, nt, 0, st>>>(g, c->rp, f, c->d_master, c->d_digits, c->d_fcm_scratch, c->d_cache_d,
                                   c->d_cache_g, c->d_cache_gn, c->d_sc, refresh_interp ? 1 : 0);
}

void launch_interp_apply(const xbs_core* c, cudaStream_t st) {
  const Geo& g = c->g;
  const int64_t njobs = int64_t(g.S) * 2 * g.GR * g.GC;
  const int grid = int(std::min<int64_t>(njobs, 148 * 8));
  k_interp_apply<<<grid, 256, 0, st>>>(g, c->rp, c->d_master, c->d_digits, c->d_cache_d, c->d_cache_g,
                                       c->d_cache_gn);
}

}  // namespace xbs
