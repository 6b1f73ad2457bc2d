// ADC auto-calibration (layers.cpp:74, 189-213,
// converters.cpp:90-107).
//
// While a core calibrates, its VMMs run with pass-through sensing and every
// sensed current is recorded: forward currents of training batches (one per
// batch row x input bit x tile x slice x polarity x tile column, padding
// columns included) and all backward currents (x 4 phase/polarity readouts
// per tile row).  On the snapped grid each current is I = n 2^sh exactly, so
// the record is the integer n (u64) and the reference's sorted[rank] is the
// rank-th smallest n.  The freeze selects it exactly with a 4-pass radix
// select (11 bits per pass over n < 2^44) on the device.
//
// The record is what the reference's calibrator keeps (one value per
// observation, converters.cpp:90-94); it lives in HBM and grows by doubling.
// A sample that no longer fits on the device fails loudly (XBS_UNSUPPORTED).
#include <algorithm>
#include <cstring>
#include <string>

#include "xbs_internal.cuh"

namespace xbs {
namespace {

__device__ __forceinline__ uint32_t q_at(const uint8_t* digits, const Geo& g, int s, int p, int tr, int tc, int r,
                                         int c) {
  const size_t base = g.tile_digit_offset(s, p, tr, tc, 0) + size_t(r) * g.C + c, ps = g.plane_bytes();
  return (digits[base] + 255u * digits[base + ps]) + 65025u * digits[base + 2 * ps];
}

// Forward observations (layers.cpp:252-257): n of column c of tile (tr, tc)
// for slice s, polarity p, input bit k, batch row b.  Index order
// [b][k][tc][tr][s][p][c] (c fastest: coalesced digit reads).
__global__ void k_observe_fwd(Geo g, int64_t M, const uint8_t* __restrict__ A, const uint8_t* __restrict__ digits,
                              const unsigned long long* __restrict__ count, unsigned long long* __restrict__ out) {
  const int64_t per_b = int64_t(g.Ti) * g.GC * g.GR * g.S * 2 * g.tile_cols;
  const int64_t n = M * per_b;
  const unsigned long long base = *count;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t u = t;
    const int c = int(u % g.tile_cols);
    u /= g.tile_cols;
    const int p = int(u % 2);
    u /= 2;
    const int s = int(u % g.S);
    u /= g.S;
    const int tr = int(u % g.GR);
    u /= g.GR;
    const int tc = int(u % g.GC);
    u /= g.GC;
    const int k = int(u % g.Ti);
    const int64_t b = u / g.Ti;
    const uint8_t* arow = A + (b * g.TPi + k) * g.KI + size_t(tr) * g.R;
    unsigned long long nn = 0;
    for (int r = 0; r < g.tile_rows; ++r)
      if (arow[r]) nn += q_at(digits, g, s, p, tr, tc, r, c);
    out[base + t] = nn;
  }
}

// Backward observations (layers.cpp:352-361): the four readouts vp.gp^T,
// vm.gn^T, vp.gn^T, vm.gp^T of tile row r.  Index order
// [b][k][tr][tc][s][readout][r].  Nothing is observed when max|dy| = 0
// (layers.cpp:308 returns before sensing).
__global__ void k_observe_bwd(Geo g, int64_t M, const uint8_t* __restrict__ A, const uint8_t* __restrict__ digits,
                              const DevScalars* __restrict__ sc, const unsigned long long* __restrict__ count,
                              unsigned long long* __restrict__ out) {
  if (!(sc->se > 0)) return;
  const int64_t per_b = int64_t(g.Te) * g.GR * g.GC * g.S * 4 * g.tile_rows;
  const int64_t n = M * per_b;
  const unsigned long long base = *count;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t u = t;
    const int r = int(u % g.tile_rows);
    u /= g.tile_rows;
    const int ro = int(u % 4);
    u /= 4;
    const int s = int(u % g.S);
    u /= g.S;
    const int tc = int(u % g.GC);
    u /= g.GC;
    const int tr = int(u % g.GR);
    u /= g.GR;
    const int k = int(u % g.Te);
    const int64_t b = u / g.Te;
    // readout 0: plus x pos, 1: minus x neg, 2: plus x neg, 3: minus x pos
    const int phase = ro & 1, pol = (ro == 0 || ro == 3) ? 0 : 1;
    const uint8_t* arow = A + ((b * g.TPe + k) * 2 + phase) * g.NB + size_t(tc) * g.C;
    unsigned long long nn = 0;
    for (int c = 0; c < min(g.tile_cols, g.NB - int(tc) * g.C); ++c)
      if (arow[c]) nn += q_at(digits, g, s, pol, tr, tc, r, c);
    out[base + t] = nn;
  }
}

// General converters (volts mode: multi-bit DAC streams, DAC tables, codes
// above 16 bits): the sensed currents are fp64 sums in the reference's order
// (ascending crossbar rows forward, columns backward, as k_fwd_volts /
// k_bwd_volts), recorded as their bit patterns -- non-negative doubles order
// as u64, so the same radix select (over 64 bits) finds sorted[rank].
__global__ void k_observe_fwd_volts(Geo g, VoltsP v, int e, int64_t M, const uint32_t* __restrict__ xc,
                                    const uint8_t* __restrict__ digits, const unsigned long long* __restrict__ count,
                                    unsigned long long* __restrict__ out) {
  const int nx = g.Ti / v.sb, mask = (1 << v.sb) - 1;
  const int64_t per_b = int64_t(nx) * g.GC * g.GR * g.S * 2 * g.tile_cols;
  const int64_t n = M * per_b;
  const unsigned long long base = *count;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t u = t;
    const int c = int(u % g.tile_cols);
    u /= g.tile_cols;
    const int p = int(u % 2);
    u /= 2;
    const int s = int(u % g.S);
    u /= g.S;
    const int tr = int(u % g.GR);
    u /= g.GR;
    const int tc = int(u % g.GC);
    u /= g.GC;
    const int k = int(u % nx);
    const int64_t b = u / nx;
    const int rows = min(g.tile_rows, g.K - tr * g.tile_rows);  // padded rows carry volts(0) = 0
    double I = 0.0;
    for (int r = 0; r < rows; ++r) {
      const int d = int(xc[b * g.K + tr * g.tile_rows + r] >> (k * v.sb)) & mask;
      if (d) I = __dadd_rn(I, __dmul_rn(v.lut[d], ldexp(double(q_at(digits, g, s, p, tr, tc, r, c)), -e)));
    }
    out[base + t] = (unsigned long long)__double_as_longlong(I);
  }
}

__global__ void k_observe_bwd_volts(Geo g, VoltsP v, int e, int64_t M, const int32_t* __restrict__ ec,
                                    const uint8_t* __restrict__ digits, const DevScalars* __restrict__ sc,
                                    const unsigned long long* __restrict__ count,
                                    unsigned long long* __restrict__ out) {
  if (!(sc->se > 0)) return;
  const int ne = g.Te / v.sb, mask = (1 << v.sb) - 1;
  const int64_t per_b = int64_t(ne) * g.GR * g.GC * g.S * 4 * g.tile_rows;
  const int64_t n = M * per_b;
  const unsigned long long base = *count;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    int64_t u = t;
    const int r = int(u % g.tile_rows);
    u /= g.tile_rows;
    const int ro = int(u % 4);
    u /= 4;
    const int s = int(u % g.S);
    u /= g.S;
    const int tc = int(u % g.GC);
    u /= g.GC;
    const int tr = int(u % g.GR);
    u /= g.GR;
    const int k = int(u % ne);
    const int64_t b = u / ne;
    const int phase = ro & 1, pol = (ro == 0 || ro == 3) ? 0 : 1;  // as k_observe_bwd
    const int cols = min(g.tile_cols, g.N - tc * g.tile_cols);
    double I = 0.0;
    for (int c = 0; c < cols; ++c) {
      const int code = ec[b * g.N + tc * g.tile_cols + c];
      const int mag = phase == 0 ? (code > 0 ? code : 0) : (code < 0 ? -code : 0);
      const int d = (mag >> (k * v.sb)) & mask;
      if (d) I = __dadd_rn(I, __dmul_rn(v.lut[d], ldexp(double(q_at(digits, g, s, pol, tr, tc, r, c)), -e)));
    }
    out[base + t] = (unsigned long long)__double_as_longlong(I);
  }
}

__global__ void k_obs_advance(unsigned long long* count, unsigned long long added, const DevScalars* sc,
                              int need_se) {
  if (need_se && !(sc->se > 0)) return;
  *count += added;
}

// One radix-select pass: histogram of bits [shift, shift + 11) of the values
// whose bits above match `prefix` under `mask`.
__global__ void k_obs_hist(const unsigned long long* __restrict__ v, int64_t n, unsigned long long prefix,
                           unsigned long long mask, int shift, unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long x = v[t];
    if ((x & mask) == prefix) atomicAdd(&h[(x >> shift) & 2047u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

int grid_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8))); }

// Room for `add` more observations in direction `dir` (doubling growth).
void reserve(xbs_core* c, int dir, int64_t add, cudaStream_t st) {
  const int64_t need = c->obs_used[dir] + add;
  if (need <= c->obs_cap[dir]) return;
  const int64_t cap = std::max<int64_t>(need, 2 * c->obs_cap[dir]);
  unsigned long long* p = nullptr;
  if (cudaMalloc(&p, size_t(cap) * 8) != cudaSuccess) {
    (void)cudaGetLastError();
    fail_conv(XBS_UNSUPPORTED, "ADC auto-calibration: " + std::to_string(double(need) * 8 / 1e9) +
                                   " GB of observed currents do not fit on the device; pin adc.i_fs or lower "
                                   "adc_cal_batches");
  }
  if (c->obs_used[dir] > 0)
    ck_cuda(cudaMemcpyAsync(p, c->d_obs[dir], size_t(c->obs_used[dir]) * 8, cudaMemcpyDeviceToDevice, st),
            "calibration record copy");
  ck_cuda(cudaStreamSynchronize(st), "calibration record grow");
  cudaFree(c->d_obs[dir]);
  c->d_obs[dir] = p;
  c->obs_cap[dir] = cap;
}

}  // namespace

void calib_observe_fwd(xbs_core* c, int64_t M, cudaStream_t st) {
  const Geo& g = c->g;
  const int streams = c->volts_mode ? g.Ti / c->volts.sb : g.Ti;
  const int64_t n = M * streams * g.GC * g.GR * g.S * 2 * g.tile_cols;
  if (n == 0) return;
  reserve(c, 0, n, st);
  if (c->volts_mode)
    k_observe_fwd_volts<<<grid_for(n), 256, 0, st>>>(g, c->volts, c->rp.snap_e, M, c->d_xcodes32, c->d_digits,
                                                     c->d_obs_count, c->d_obs[0]);
  else
    k_observe_fwd<<<grid_for(n), 256, 0, st>>>(g, M, c->d_Af, c->d_digits, c->d_obs_count, c->d_obs[0]);
  k_obs_advance<<<1, 1, 0, st>>>(c->d_obs_count, (unsigned long long)n, c->d_sc, 0);
  c->obs_used[0] += n;
  c->launches += 2;
}

void calib_observe_bwd(xbs_core* c, int64_t M, cudaStream_t st) {
  const Geo& g = c->g;
  const int streams = c->volts_mode ? g.Te / c->volts.sb : g.Te;
  const int64_t n = M * streams * g.GR * g.GC * g.S * 4 * g.tile_rows;
  if (n == 0) return;
  reserve(c, 1, n, st);
  if (c->volts_mode)
    k_observe_bwd_volts<<<grid_for(n), 256, 0, st>>>(g, c->volts, c->rp.snap_e, M, c->d_ecodes, c->d_digits, c->d_sc,
                                                     c->d_obs_count + 1, c->d_obs[1]);
  else
    k_observe_bwd<<<grid_for(n), 256, 0, st>>>(g, M, c->d_Ab, c->d_digits, c->d_sc, c->d_obs_count + 1,
                                               c->d_obs[1]);
  k_obs_advance<<<1, 1, 0, st>>>(c->d_obs_count + 1, (unsigned long long)n, c->d_sc, 1);
  c->obs_used[1] += n;  // upper bound (zero-error batches add nothing on the device)
  c->launches += 2;
}

// converters.cpp:96-107: rank = size_t(pct * n), clamped to n - 1.
bool calib_select(xbs_core* c, int dir, double pct, uint64_t* n_out) {
  cudaStream_t st = c->stream;
  unsigned long long count = 0;
  if (c->d_obs_count)
    ck_cuda(cudaMemcpyAsync(&count, c->d_obs_count + dir, 8, cudaMemcpyDeviceToHost, st), "D2H calibration count");
  ck_cuda(cudaStreamSynchronize(st), "calibration count");
  if (count == 0) return false;
  uint64_t rank = uint64_t(pct * double(count));
  if (rank >= count) rank = count - 1;
  unsigned long long* d_hist = nullptr;
  ck_cuda(cudaMalloc(&d_hist, 2048 * 8), "cudaMalloc calibration histogram");
  unsigned long long h[2048];
  unsigned long long prefix = 0, mask = 0;
  // integer currents n < 2^44: 4 passes; fp64 bit patterns (volts mode): 6
  for (int shift = c->volts_mode ? 55 : 33; shift >= 0; shift -= 11) {
    ck_cuda(cudaMemsetAsync(d_hist, 0, 2048 * 8, st), "memset histogram");
    k_obs_hist<<<grid_for(int64_t(count)), 256, 0, st>>>(c->d_obs[dir], int64_t(count), prefix, mask, shift, d_hist);
    ck_cuda(cudaMemcpyAsync(h, d_hist, sizeof(h), cudaMemcpyDeviceToHost, st), "D2H histogram");
    ck_cuda(cudaStreamSynchronize(st), "calibration select");
    c->launches += 1;
    int bin = 0;
    for (; bin < 2047 && rank >= h[bin]; ++bin) rank -= h[bin];
    prefix |= (unsigned long long)bin << shift;
    mask |= 2047ull << shift;
  }
  cudaFree(d_hist);
  *n_out = prefix;
  return true;
}

void calib_release(xbs_core* c) {
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (int d = 0; d < 2; ++d) {
    cudaFree(c->d_obs[d]);
    c->d_obs[d] = nullptr;
    c->obs_cap[d] = c->obs_used[d] = 0;
  }
}

}  // namespace xbs
