// Internal declarations shared by the C-ABI implementation and the kernels.
//
// HBM layout (all per core, sized once at create, batch buffers grow on
// demand) — DESIGN.md §"Data layout in HBM":
//   master  u[s][i][j]        fp64, S x Kp x Np, row-major (j fastest)
//   digits  D[s][p][tr][tc][d][r][c]  u8 radix-255 digits of the snapped
//           conductance q = (d0 + 255 d1) + 65025 d2; each digit
//           plane is an R x C row-major tile (R, C = tile dims rounded up to
//           128; the internal pad holds 0 and never conducts)
//   A_fwd   [dh][b*TPi + k][KI] u8 {0,1} (dh=0) / {0,255} (dh=1) input
//           bit-planes, feature i at column (i / tile_rows) * R + i % tile_rows
//   A_bwd   [dh][(b*TPe + k)*2 + phi][NB] u8 error bit-planes, phi = sign
//           (NB = NI, or 32 / 64 bytes for a single narrow column tile)
//   xcodes  [b][i] u16 activation codes; ecodes [b][j] i32 signed error codes
//   dW      [i][j] fp64 (row-major K x N)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <string>
#include <vector>

#include "../../include/xbarsim_b200.h"

namespace xbs {

// Snapped exactness grid (radix-255 variant): q <= kQMax,
// three u8 digits (tensor-core limbs) per conductance.
constexpr int kLimbs = 3;
constexpr double kQMax = 16581374.0;  // 255^3 - 1

// Rows of the forward / backward bit-plane operands, padded to whole
// 256-row MMA unit pairs (rows beyond M*TP are zero).
inline int64_t rows_fwd(int64_t M, int TPi) { return ((M * TPi + 255) / 256) * 256; }
inline int64_t rows_bwd(int64_t M, int TPe) { return ((M * TPe * 2 + 255) / 256) * 256; }

struct Geo {
  int K = 0, N = 0;                 // logical in / out features
  int tile_rows = 0, tile_cols = 0; // logical tile (MappingSpec)
  int GR = 0, GC = 0;               // grid_rows, grid_cols
  int Kp = 0, Np = 0;               // reference padded dims
  int R = 0, C = 0;                 // device tile dims (multiples of 128)
  int KI = 0, NI = 0;               // GR*R, GC*C
  int NB = 0;                       // A_bwd row pitch: NI, or 32 / 64 for one 128-column tile holding
                                    // <= 32 / <= 64 logical columns (the rest of NI is zero padding)
  int S = 0, db = 0, wb = 0;        // slices, device_bits, weight_bits
  int Ti = 0, TPi = 0;              // act_bits, padded to a power of two
  int Te = 0, TPe = 0;              // error_bits, padded
  __host__ __device__ size_t plane_bytes() const { return size_t(R) * C; }
  __host__ __device__ size_t tile_digit_offset(int s, int p, int tr, int tc, int d) const {
    return ((((size_t(s) * 2 + p) * GR + tr) * GC + tc) * kLimbs + d) * plane_bytes();
  }
  __host__ __device__ size_t digits_bytes() const { return size_t(S) * 2 * GR * GC * kLimbs * plane_bytes(); }
};

// Conversion / regeneration parameters (mapping.cpp:28-58, aam.cpp:5-31).
struct RegenP {
  double g_min, g_max, range, sigma;
  uint64_t vseed;
  double r_row, r_col, r_source, r_sense;
  int aam;     // 1: AAM conversion, 0: identity (ideal / zero-parasitic fcm)
  int snap_e;  // grid exponent e
  double snap_scale;  // 2^e
  // sigma != 0: the variation multipliers m(s, p, device) are fixed for the
  // life of the core (mapping.cpp:28-35 keys them by seed and position only),
  // so they are computed once at create and read back: [s][p][Kp][Np] fp64
  const double* varm;
  uint64_t kpnp;  // Kp * Np
};

// update.cpp:43-88 + implied weights (mapping.cpp:70-81)
struct UpdP {
  double v, gamma, lr, factor;  // factor = (g_max-g_min)/layer_scale
  double wfactor;               // implied-weight factor
  uint64_t seed, iteration;
  int linear;
};

// ADC (converters.cpp:70-88) on the snapped grid: I = n * 2^sh exactly.
struct AdcP {
  int passthrough;  // adc.bits == 0
  int maxc;         // 2^bits - 1
  int sh;           // log2(v_fs) - e
  double i_fs;
  double maxc_d;
};

// General converters (multi-bit DAC streams, DAC / ADC transfer tables, ADC
// above 16 bits, non-power-of-two DAC full scale): exact fp64 CUDA-core path.
struct VoltsP {
  const double* lut;            // dac_encode of every digit (converters.cpp:28-35), device
  int sb;                       // dac.stream_bits
  int passthrough;              // adc.bits == 0
  const double* adc_tr;         // ADC thresholds (converters.cpp:76-82), device, or null
  int tr_len;
  unsigned long long maxcode;   // 2^bits - 1 (bits <= 32)
  double maxc_d, i_fs;          // i_fs: forward full scale
  double i_fs_b;                // backward full scale (differs after auto-calibration)
};

// Device scalars (one struct per core, in HBM).
struct DevScalars {
  double se;                 // max|dy|
  unsigned long long dwmax;  // bits of max|dW| (non-negative doubles order as u64)
  unsigned long long wmax;   // bits of max|implied W|
  unsigned long long wmax_in;// bits of max|W0| (layer scale)
  int err_flag;              // bit 0: nonlinear_update range violation, bit 1: update skipped on a
                             // non-finite gradient; sticky until the host reads it
  int dw_nonfinite;          // the last dW holds a non-finite value (update.cpp:18-19)
  unsigned long long exact_path, conversions;
  unsigned int fcm_fail;                 // FCM tiles without a fixed point in the last regeneration
  unsigned int pad2;
  unsigned long long fcm_residual;       // bits of the largest such residual (relative to v_fs)
  unsigned int wave_sync[2];             // CTA-pair arrival counters of the forward / backward VMM (wave alignment)
};

// FCM conversion parameters (fcm.hpp:9-16, tile geometry and parasitics of
// the mapped tile config, mapping.cpp:60-67)
struct FcmP {
  double r_row, r_col, r_source, r_sense, v_fs, tol;
  int max_iter;
  int use_fcm;  // 0: interp_fcm with the AAM base
};

}  // namespace xbs

struct xbs_core {
  xbs_layer_options opt{};
  std::vector<double> dac_tr, adc_tr;
  xbs::Geo g;
  xbs::RegenP rp{};
  xbs::AdcP adc{};    // forward ADC (adc_fwd_)
  xbs::AdcP adc_b{};  // backward ADC (adc_bwd_); differs from adc only after auto-calibration
  bool volts_mode = false;  // general converters: exact fp64 CUDA-core VMMs (k_fwd_volts / k_bwd_volts)
  bool out_host = false;    // the VMM being enqueued stores into a mapped host buffer (set per call)
  bool big_tiles = false;   // tiles above 256 x 256: exact integer CUDA-core VMMs (k_fwd_simt / k_bwd_simt)
  xbs::VoltsP volts{};
  double* d_dac_lut = nullptr;
  double* d_adc_tr = nullptr;
  xbs::FcmP fcm{};
  bool tile_engine = false;     // fcm / interp_fcm with parasitics: per-tile regeneration kernels
  uint64_t update_count = 0;    // layers.cpp:389 (interp refresh schedule)
  cudaStream_t stream = nullptr;
  // Update statistics are folded lazily: every apply_updates records an event
  // pair around its kernels and marks the device scalars pending; the next
  // observing call (synchronize, getters, a host call's final sync) reads
  // them once: running |dW| / |W| maxima, sticky error bits (read and
  // cleared), update time into conversion_seconds (layers.cpp:176-177).
  bool stats_pending = false;
  bool upd_async = false;  // host apply_updates returned before its kernels finished
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> upd_timing;
  int64_t tc_fallbacks = 0;  // VMM calls whose tcgen05 kernel refused the shape (SIMT ran)
  cudaStream_t copy_stream = nullptr;  // host->device input copies overlapping a pending update
  cudaEvent_t copy_ev = nullptr;
  bool own_stream = true;  // false after xbs_core_set_stream(caller's stream)
  int kernel = 0;  // 0 tcgen05, 1 SIMT
  bool weights_only = false;  // a mapping::TiledLayerWeights (xbs_weights.cu): master only, no conductances
  bool fully_ideal = false;
  bool adc_scaled = false;  // k_out includes i_fs/(2^bits-1)
  double layer_scale = 1.0, level_step = 0.0;
  double k_out_fwd = 0.0;     // layers.cpp:272-281
  double kb_F_over_vu = 0.0;  // backward: k = step_e * F / vu (* ifs_fac)
  double F = 0.0, vu = 0.0, ifs_fac = 1.0, sx = 0.0, lev_e = 0.0, lev_a = 0.0;
  double ifs_fac_b = 1.0;  // backward i_fs / (2^bits - 1)
  // ADC auto-calibration (layers.cpp:74, 189-213): pass-through VMMs that
  // record every sensed current (as n, units 2^sh) until adc_cal_batches
  // training forwards, then the nearest-rank quantile fixes i_fs
  bool adc_auto = false, adc_frozen = false;
  int64_t training_batches = 0;
  unsigned long long* d_obs[2] = {nullptr, nullptr};  // observed n [fwd, bwd]
  int64_t obs_cap[2] = {0, 0}, obs_used[2] = {0, 0};  // host upper bound of the device count
  unsigned long long* d_obs_count = nullptr;          // device counts [2]
  // device buffers
  uint8_t* d_digits = nullptr;
  uint32_t* d_qmin = nullptr;  // sigma == 0: snapped q of g_min per tile position
  double* d_varm = nullptr;    // sigma != 0: variation multipliers [s][p][Kp][Np]
  double* d_fcm_scratch = nullptr;  // FCM per-CTA node voltages / coefficients
  size_t fcm_scratch_bytes = 0;
  double* d_cache_d = nullptr;      // interp_fcm: distortion profile, g and converted g at refresh [s][p][Kp][Np]
  double* d_cache_g = nullptr;
  double* d_cache_gn = nullptr;
  unsigned long long* d_adc_tab = nullptr;  // T[k] = min column current n (units 2^-e) with code >= k
  unsigned long long* d_adc_tab_b = nullptr;  // same for the backward ADC
  double* d_master = nullptr;
  double* d_dW = nullptr;
  double* d_wimp = nullptr;  // implied weights (fully-ideal fast path), K x N row-major
  xbs::DevScalars* d_sc = nullptr;
  xbs::DevScalars* h_sc = nullptr;  // pinned mirror
  // batch-dependent
  int64_t M_cap = 0;
  uint8_t* d_Af = nullptr;   // 2 * rowsF * KI
  uint8_t* d_Ab = nullptr;   // 2 * rowsB * NI
  uint16_t* d_xcodes = nullptr;
  uint32_t* d_xcodes32 = nullptr;  // volts mode: u32 codes (act_bits up to 24), no bit planes
  int32_t* d_ecodes = nullptr;  // signed error codes: 16-bit magnitudes need more than int16
  // u8 operands of the tcgen05 dW GEMM (act/error bits <= 8): x codes
  // [Mcap8][KA], error magnitudes [plus | minus][Mcap8][NA]; K, N padded to
  // 128 (zero), batch padded to 128 (rows >= M zeroed per call)
  uint8_t* d_xc8 = nullptr;
  uint8_t* d_e8 = nullptr;
  int KA = 0, NA = 0;
  unsigned long long* d_S64 = nullptr;  // split-batch dW: int64 partial sums [KA][NA]
  size_t S64_bytes = 0;
  void* d_acc32 = nullptr;  // split-K VMMs (small or very deep / wide layers): exact int32 or int64 partial totals [cols][M], kept zero
  size_t acc32_bytes = 0;
  int64_t M_cap8 = 0;
  double* d_io_in = nullptr;   // host-API staging (M x max(K,N))
  double* d_io_out = nullptr;
  int64_t io_cap = 0;
  // state
  int64_t M_fwd = 0;
  bool have_forward = false, have_grad = false;
  int64_t refreshes = 0;
  double conversion_seconds = 0.0;
  double wmax_seen = 0.0, dwmax_seen = 0.0;
  int64_t exact_path = 0, conversions = 0;
  // host mirrors for readback
  std::vector<double> h_tmp;
  // profiling: pending (stage, start, stop) event pairs, accumulated totals
  bool profile = false;
  // CUDA graphs of the forward / backward launch sequences (xbs_core.cu):
  // a call whose key repeats is captured once and replayed as one launch.
  // gen changes whenever a kernel argument the key does not cover changes
  // (buffers reallocated, ADC re-armed, kernel / stream switched).
  bool use_graphs = true;
  uint64_t gen = 0;
  struct GraphSlot {
    uint64_t key[8] = {};
    bool seen = false, ready = false;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
    int64_t fallbacks = 0;
  } gfwd, gbwd;
  std::vector<cudaEvent_t> ev_pool;
  struct Pending { int stage; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  double stage_ms[XBS_NUM_STAGES] = {};
  int64_t stage_n[XBS_NUM_STAGES] = {};
  int64_t launches = 0;
};

namespace xbs {
// kernels (launchers), all enqueue on `st`
void launch_map_weights(const xbs_core* c, const double* d_W, cudaStream_t st);
void launch_absmax(const double* d_x, int64_t n, unsigned long long* out_bits, cudaStream_t st);
void launch_regen_all(const xbs_core* c, cudaStream_t st);
// Convolution input read in place of the patch matrix (CrossbarConv2d,
// layers.cpp:442-458): patch row (img, oy, ox), column (c, ky, kx) is the
// image element (c, oy*stride - pad + ky, ox*stride - pad + kx), or 0 in the
// padding.  The image is batch x (in_c*h*w) column-major.
struct ConvSrc {
  int in_c, h, w, k, stride, pad, oh, ow;
  int64_t batch;
};
void launch_prep_x(const xbs_core* c, const double* d_x, int64_t M, cudaStream_t st, const ConvSrc* conv = nullptr);
// forward of a core whose input is the im2col lowering of an image (no patch
// matrix is materialised); y is the rows x out_c column-major flat output
void core_forward_conv(xbs_core* c, const double* d_img, const ConvSrc& cs, bool training, double* d_y);
void launch_prep_dy(const xbs_core* c, const double* d_dy, int64_t M, cudaStream_t st);
void launch_fwd_simt(const xbs_core* c, int64_t M, double* d_y, cudaStream_t st);
void launch_fwd_volts(const xbs_core* c, int64_t M, double* d_y, cudaStream_t st);
void launch_bwd_volts(const xbs_core* c, int64_t M, double* d_dx, cudaStream_t st);
void launch_bwd_simt(const xbs_core* c, int64_t M, double* d_dx, cudaStream_t st);
void launch_fwd_ideal(const xbs_core* c, int64_t M, double* d_y, cudaStream_t st);
void launch_bwd_ideal(const xbs_core* c, const double* d_dy, int64_t M, double* d_dx, cudaStream_t st);
void launch_dw(const xbs_core* c, int64_t M, double grad_divisor, cudaStream_t st);
void launch_update(const xbs_core* c, const UpdP& up, cudaStream_t st, bool master_only = false);
void launch_fcm_regen(xbs_core* c, bool refresh_interp, cudaStream_t st);
void launch_interp_apply(const xbs_core* c, cudaStream_t st);
void ck_cuda(cudaError_t e, const char* what);  // throws the C-ABI error
int set_error(int code, const std::string& m);   // sets xbs_last_error, returns code
[[noreturn]] void fail_conv(int code, const std::string& m);
void check_rc(int rc);                            // rethrows a C-ABI status
int guard_conv(const std::function<void()>& f);   // runs f, mapping exceptions to statuses
void launch_qmin(const xbs_core* c, cudaStream_t st);
void launch_varm(const xbs_core* c, cudaStream_t st);
void launch_implied(const xbs_core* c, double* d_out, cudaStream_t st);
void launch_digits_to_g(const xbs_core* c, int s, int p, int tr, int tc, double* d_out, cudaStream_t st);
// tcgen05 kernels (xbs_vmm_tc.cu); return false if the shape is not covered
bool launch_fwd_tc(xbs_core* c, int64_t M, double* d_y, int64_t ldy, cudaStream_t st);
bool launch_bwd_tc(xbs_core* c, int64_t M, double* d_dx, int64_t ldx, cudaStream_t st);
bool launch_dw_tc(xbs_core* c, int64_t M, double grad_divisor, cudaStream_t st);
// TiledLayerWeights objects (xbs_weights.cu) share the core's geometry,
// master layout and kernels
xbs_core* create_weights_core(const xbs_layer_options* opt, const double* W, int64_t K, int64_t N, int64_t ldw);
void core_settle(xbs_core* c);
void core_h2d_rowmajor(xbs_core* c, const double* h, int64_t rows, int64_t cols, int64_t ld, double* d);
void core_d2h_rowmajor(xbs_core* c, const double* d, int64_t rows, int64_t cols, double* h, int64_t ld);
// ADC auto-calibration (xbs_calib.cu)
void calib_observe_fwd(xbs_core* c, int64_t M, cudaStream_t st);
void calib_observe_bwd(xbs_core* c, int64_t M, cudaStream_t st);
bool calib_select(xbs_core* c, int dir, double pct, uint64_t* n_out);  // false: no observations
void calib_release(xbs_core* c);
}  // namespace xbs
