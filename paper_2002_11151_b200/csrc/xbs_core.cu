// C-ABI implementation: the CrossbarCore state machine (layers.cpp:68-391)
// over device-resident state.  Host code validates exactly like the reference
// (same order, same exception classes mapped to status codes), computes the
// fp64 scale constants with the reference's expressions, and enqueues the
// kernels on the core's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <functional>
#include <string>
#include <vector>

#include "xbs_internal.cuh"

namespace {

thread_local std::string g_err;

struct XbsError : std::runtime_error {
  int code;
  XbsError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& m) { throw XbsError(code, m); }
void ck(cudaError_t e, const char* what);
}  // namespace
namespace xbs {
void ck_cuda(cudaError_t e, const char* what) { ck(e, what); }
}  // namespace xbs
namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(XBS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return XBS_OK;
  } catch (const XbsError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return XBS_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return XBS_INTERNAL;
  }
}

bool is_pow2_double(double v) {
  int e;
  return v > 0 && std::frexp(v, &e) == 0.5;
}
int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// ---- validation, in the reference's order and with its exception classes
void validate_crossbar(const xbs_layer_options& o) {  // crossbar.hpp:31-39
  if (o.xbar_rows < 1 || o.xbar_cols < 1) fail(XBS_INVALID_ARGUMENT, "CrossbarConfig: rows and cols must be >= 1");
  if (o.r_row < 0 || o.r_col < 0 || o.r_source < 0 || o.r_sense < 0)
    fail(XBS_INVALID_ARGUMENT, "CrossbarConfig: resistances must be >= 0");
  if (!(o.g_min > 0) || !(o.g_max > o.g_min)) fail(XBS_INVALID_ARGUMENT, "CrossbarConfig: need 0 < g_min < g_max");
  if (!(o.v_fs > 0)) fail(XBS_INVALID_ARGUMENT, "CrossbarConfig: v_fs must be > 0");
}
void validate_mapping(const xbs_layer_options& o) {  // mapping.cpp:10-24
  if (o.weight_bits < 1 || o.weight_bits > 24) fail(XBS_INVALID_ARGUMENT, "MappingSpec: weight_bits must be in [1, 24]");
  if (o.device_bits < 1 || o.device_bits > o.weight_bits)
    fail(XBS_INVALID_ARGUMENT, "MappingSpec: device_bits must be in [1, weight_bits]");
  if (o.weight_bits % o.device_bits != 0)
    fail(XBS_INVALID_ARGUMENT, "MappingSpec: weight_bits must be divisible by device_bits");
  if (o.tile_rows < 1 || o.tile_cols < 1) fail(XBS_INVALID_ARGUMENT, "MappingSpec: tile dims must be >= 1");
  if (o.tile_rows > o.xbar_rows || o.tile_cols > o.xbar_cols)
    fail(XBS_INVALID_ARGUMENT, "MappingSpec: tile dims exceed crossbar dims");
  if (o.variation_sigma < 0) fail(XBS_INVALID_ARGUMENT, "MappingSpec: variation_sigma must be >= 0");
}
void validate_options(const xbs_layer_options& o, const std::vector<double>& dac_tr,
                      const std::vector<double>& adc_tr) {  // layers.cpp:17-47
  validate_crossbar(o);
  validate_mapping(o);
  // DacSpec::validate (converters.cpp:11-26)
  if (o.dac_bits < 1 || o.dac_bits > 32) fail(XBS_INVALID_ARGUMENT, "DacSpec: bits must be in [1, 32]");
  if (!(o.dac_v_fs > 0)) fail(XBS_INVALID_ARGUMENT, "DacSpec: v_fs must be > 0");
  if (o.dac_stream_bits < 1) fail(XBS_INVALID_ARGUMENT, "DacSpec: stream_bits must be >= 1");
  if (!dac_tr.empty()) {
    if (dac_tr.size() != (size_t{1} << o.dac_bits))
      fail(XBS_INVALID_ARGUMENT, "DacSpec: transfer table must have 2^bits entries");
    if (dac_tr.front() != 0.0) fail(XBS_INVALID_ARGUMENT, "DacSpec: transfer[0] must be 0");
    if (dac_tr.back() > o.dac_v_fs) fail(XBS_INVALID_ARGUMENT, "DacSpec: transfer must not exceed v_fs");
    if (!std::is_sorted(dac_tr.begin(), dac_tr.end()))
      fail(XBS_INVALID_ARGUMENT, "DacSpec: transfer table must be monotone");
  }
  // AdcSpec::validate (converters.cpp:57-68)
  if (o.adc_bits < 0 || o.adc_bits > 32) fail(XBS_INVALID_ARGUMENT, "AdcSpec: bits must be in [0, 32]");
  if (!(o.adc_clip_percentile > 0.0) || o.adc_clip_percentile > 1.0)
    fail(XBS_INVALID_ARGUMENT, "AdcSpec: clip_percentile must be in (0, 1]");
  if (!adc_tr.empty()) {
    if (o.adc_bits == 0) fail(XBS_INVALID_ARGUMENT, "AdcSpec: transfer table with pass-through ADC");
    if (!std::is_sorted(adc_tr.begin(), adc_tr.end()))
      fail(XBS_INVALID_ARGUMENT, "AdcSpec: transfer thresholds must be monotone");
  }
  // UpdateSpec::validate (update.cpp:10-14)
  if (o.upd_v < 0) fail(XBS_INVALID_ARGUMENT, "UpdateSpec: v must be >= 0");
  if (o.upd_gamma < 0) fail(XBS_INVALID_ARGUMENT, "UpdateSpec: gamma must be >= 0");
  if (!(o.upd_lr > 0)) fail(XBS_INVALID_ARGUMENT, "UpdateSpec: lr must be > 0");
  if (o.dac_bits != o.dac_stream_bits)
    fail(XBS_CONFIG_ERROR, "dac.bits (" + std::to_string(o.dac_bits) + ") must equal dac.stream_bits (" +
                               std::to_string(o.dac_stream_bits) + "): the streamed slice is the physical converter");
  if (o.act_bits < 1 || o.act_bits > 24) fail(XBS_CONFIG_ERROR, "act_bits must be in [1, 24]");
  if (o.error_bits < 1 || o.error_bits > 24) fail(XBS_CONFIG_ERROR, "error_bits must be in [1, 24]");
  if (o.act_bits % o.dac_stream_bits != 0) fail(XBS_CONFIG_ERROR, "activation_bits must be divisible by dac.stream_bits");
  if (o.error_bits % o.dac_stream_bits != 0) fail(XBS_CONFIG_ERROR, "error_bits must be divisible by dac.stream_bits");
  if (!(o.act_full_scale > 0)) fail(XBS_CONFIG_ERROR, "act_full_scale must be > 0");
  if (o.interp_interval < 1) fail(XBS_CONFIG_ERROR, "interp_interval must be >= 1");
  if (o.engine == XBS_ENGINE_INTERP_FCM && o.interp_base != XBS_ENGINE_FCM && o.interp_base != XBS_ENGINE_AAM)
    fail(XBS_CONFIG_ERROR, "interp_base must be fcm or aam");
  if (o.adc_cal_batches < 1) fail(XBS_CONFIG_ERROR, "adc_cal_batches must be >= 1");
  if (o.threads < 1) fail(XBS_CONFIG_ERROR, "threads must be >= 1");
}

// Converters off the tensor-core contract (1-bit DAC streams at a power-of-
// two full scale, linear ADC of <= 16 bits, activation / error codes of <= 16
// bits): multi-bit DAC streams, DAC / ADC transfer tables, wider ADCs, other
// DAC full scales, 17- to 24-bit codes (layers.cpp:28-31).
bool volts_mode(const xbs_layer_options& o, const std::vector<double>& dac_tr, const std::vector<double>& adc_tr) {
  return !dac_tr.empty() || !adc_tr.empty() || o.adc_bits > 16 || o.dac_bits != 1 || !is_pow2_double(o.dac_v_fs) ||
         o.act_bits > 16 || o.error_bits > 16;
}

// Path scope: valid reference configurations this
// B200 path does not evaluate are refused loudly, never approximated.
void check_scope(const xbs_layer_options& o, const std::vector<double>& dac_tr, const std::vector<double>& adc_tr) {
  const bool zero_par = o.r_row == 0.0 && o.r_col == 0.0 && o.r_source == 0.0 && o.r_sense == 0.0;
  if (o.engine == XBS_ENGINE_ORACLE && !zero_par)
    fail(XBS_UNSUPPORTED, "engine oracle (dense nodal solve) with parasitics is not on this path (SURVEY §8f-4)");
  if ((o.engine == XBS_ENGINE_FCM || (o.engine == XBS_ENGINE_INTERP_FCM && o.interp_base == XBS_ENGINE_FCM)) &&
      !zero_par) {  // fcm.cpp:170-173, checked when the first tile is converted
    if (!(o.fcm_tol > 0.0) || !std::isfinite(o.fcm_tol))
      fail(XBS_INVALID_ARGUMENT, "fcm_convert: tol must be positive and finite");
    if (o.fcm_max_iter < 1) fail(XBS_INVALID_ARGUMENT, "fcm_convert: max_iter must be >= 1");
  }
  if (o.engine < 0 || o.engine > 4) fail(XBS_INVALID_ARGUMENT, "unknown engine");
  // general converters run the exact fp64 CUDA-core VMMs (volts mode)
  if (volts_mode(o, dac_tr, adc_tr) && o.dac_bits > 16)
    fail(XBS_UNSUPPORTED, "DAC streams wider than 16 bits are not on this path");
  // tiles above 256 x 256 run the exact integer CUDA-core VMMs (a 256-row
  // crossbar is the most one TMEM accumulator pair sums exactly); the integer
  // currents and the ADC table are sized for <= 1024 rows
  if (o.tile_rows > 1024 || o.tile_cols > 1024)
    fail(XBS_UNSUPPORTED, "tiles larger than 1024 x 1024 are not on this path");
  const bool circuit_tiles = (o.engine == XBS_ENGINE_FCM || o.engine == XBS_ENGINE_INTERP_FCM) && !zero_par;
  if (circuit_tiles && (o.tile_rows > 256 || o.tile_cols > 256))  // one thread per crossbar line, <= 256 per CTA
    fail(XBS_UNSUPPORTED, "fcm / interp_fcm on tiles larger than 256 x 256 is not on this path");
}

int snap_exponent(double g_max) {  // largest e with g_max * 2^e <= Q_MAX
  int e;
  (void)std::frexp(xbs::kQMax / g_max, &e);
  e += 2;
  while (std::ldexp(g_max, e) > xbs::kQMax) --e;
  return e;
}

void ensure_batch(xbs_core* c, int64_t M) {
  if (M <= c->M_cap) return;
  ++c->gen;  // buffers move: captured graphs are stale
  const int64_t cap = std::max<int64_t>(M, 2 * c->M_cap);
  cudaFree(c->d_Af);
  cudaFree(c->d_Ab);
  cudaFree(c->d_xcodes);
  cudaFree(c->d_xcodes32);
  cudaFree(c->d_ecodes);
  c->d_Af = nullptr;
  c->d_Ab = nullptr;
  c->d_xcodes = nullptr;
  c->d_xcodes32 = nullptr;
  c->d_ecodes = nullptr;
  if (c->volts_mode) {
    // the exact fp64 kernels read the codes themselves: u32 activation
    // codes (up to 24 bits), no bit planes
    ck(cudaMalloc(&c->d_xcodes32, size_t(cap) * c->g.K * sizeof(uint32_t)), "cudaMalloc xcodes");
  } else {
    const int64_t rowsF = xbs::rows_fwd(cap, c->g.TPi);
    const int64_t rowsB = xbs::rows_bwd(cap, c->g.TPe);
    ck(cudaMalloc(&c->d_Af, size_t(2 * rowsF) * c->g.KI), "cudaMalloc A_fwd");
    ck(cudaMalloc(&c->d_Ab, size_t(2 * rowsB) * c->g.NB), "cudaMalloc A_bwd");
    // the prep kernels never write 16-column groups that hold only tile
    // padding: those plane bytes stay the zeros written here
    ck(cudaMemsetAsync(c->d_Af, 0, size_t(2 * rowsF) * c->g.KI, c->stream), "memset A_fwd");
    ck(cudaMemsetAsync(c->d_Ab, 0, size_t(2 * rowsB) * c->g.NB, c->stream), "memset A_bwd");
    ck(cudaMalloc(&c->d_xcodes, size_t(cap) * c->g.K * sizeof(uint16_t)), "cudaMalloc xcodes");
  }
  ck(cudaMalloc(&c->d_ecodes, size_t(cap) * c->g.N * sizeof(int32_t)), "cudaMalloc ecodes");
  cudaFree(c->d_xc8);
  cudaFree(c->d_e8);
  c->d_xc8 = c->d_e8 = nullptr;
  if (c->opt.act_bits <= 8 && c->opt.error_bits <= 8) {
    c->KA = ((c->g.K + 127) / 128) * 128;
    c->NA = ((c->g.N + 127) / 128) * 128;
    c->M_cap8 = ((cap + 127) / 128) * 128;
    ck(cudaMalloc(&c->d_xc8, size_t(c->M_cap8) * c->KA), "cudaMalloc xc8");
    ck(cudaMalloc(&c->d_e8, 2 * size_t(c->M_cap8) * c->NA), "cudaMalloc e8");
    ck(cudaMemsetAsync(c->d_xc8, 0, size_t(c->M_cap8) * c->KA, c->stream), "memset");
    ck(cudaMemsetAsync(c->d_e8, 0, 2 * size_t(c->M_cap8) * c->NA, c->stream), "memset");
  }
  c->M_cap = cap;
}

void ensure_io(xbs_core* c, int64_t elems) {
  if (elems <= c->io_cap) return;
  cudaFree(c->d_io_in);
  cudaFree(c->d_io_out);
  c->d_io_in = c->d_io_out = nullptr;
  ck(cudaMalloc(&c->d_io_in, size_t(elems) * 8), "cudaMalloc io_in");
  ck(cudaMalloc(&c->d_io_out, size_t(elems) * 8), "cudaMalloc io_out");
  c->io_cap = elems;
}

void check_fcm(xbs_core* c);
cudaEvent_t take_event(xbs_core* c);

// Folds the statistics of the updates enqueued since the last fold, once
// their kernels are complete: update time from CUDA events into
// conversion_seconds (the reference times regenerate(), layers.cpp:176-177),
// the running |dW| / |W| maxima the device keeps across updates
// (layers.cpp:384-386), and the sticky error bits, which are cleared once
// read so an error surfaces exactly once.  Every entry point that observes
// core state calls this (directly or through sync) before reading; the
// *_device calls never do, so device-path steps queue back to back.
void settle(xbs_core* c) {
  if (!c->stats_pending) return;
  c->stats_pending = false;
  c->upd_async = false;
  ck(cudaMemcpyAsync(c->h_sc, c->d_sc, sizeof(xbs::DevScalars), cudaMemcpyDeviceToHost, c->stream), "D2H scalars");
  ck(cudaStreamSynchronize(c->stream), "kernel execution");
  for (auto& e : c->upd_timing) {
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, e.first, e.second), "update timing");
    c->conversion_seconds += 1e-3 * ms;
    c->ev_pool.push_back(e.first);
    c->ev_pool.push_back(e.second);
  }
  c->upd_timing.clear();
  c->dwmax_seen = std::max(c->dwmax_seen, __builtin_bit_cast(double, c->h_sc->dwmax));
  c->wmax_seen = std::max(c->wmax_seen, __builtin_bit_cast(double, c->h_sc->wmax));
  const int err = c->h_sc->err_flag;
  if (err || (c->tile_engine && c->h_sc->fcm_fail)) {
    ck(cudaMemsetAsync(&c->d_sc->err_flag, 0, sizeof(int), c->stream), "memset");
    ck(cudaMemsetAsync(&c->d_sc->fcm_fail, 0, sizeof(unsigned), c->stream), "memset");
    ck(cudaStreamSynchronize(c->stream), "kernel execution");
  }
  if (err & 2) fail(XBS_INVALID_ARGUMENT, "scale_gradient: gradient must be finite");
  if (err & 1) fail(XBS_INVALID_ARGUMENT, "nonlinear_update: g outside device range");
  check_fcm(c);
}

void sync(xbs_core* c) {
  ck(cudaStreamSynchronize(c->stream), "kernel execution");
  ck(cudaGetLastError(), "kernel launch");
  settle(c);
}

void regenerate_bookkeeping(xbs_core* c) {
  if (c->opt.engine == XBS_ENGINE_IDEAL) xbs::launch_implied(c, c->d_wimp, c->stream);
  const bool refresh_now = c->opt.engine != XBS_ENGINE_INTERP_FCM ||
                           c->update_count % uint64_t(c->opt.interp_interval) == 0;  // layers.cpp:145-147
  if (c->opt.engine != XBS_ENGINE_IDEAL && refresh_now) ++c->refreshes;           // layers.cpp:176
}

// Per-tile regeneration for the circuit engines (layers.cpp:129-179 with
// convert_tile 90-127): fcm every time, interp_fcm refreshing its distortion
// profile every interp_interval updates and applying it in between.
void regenerate_tiles(xbs_core* c) {
  ck(cudaMemsetAsync(&c->d_sc->fcm_fail, 0, sizeof(unsigned) * 2 + sizeof(unsigned long long), c->stream),
     "memset");
  if (c->opt.engine == XBS_ENGINE_INTERP_FCM && c->update_count % uint64_t(c->opt.interp_interval) != 0)
    xbs::launch_interp_apply(c, c->stream);
  else
    xbs::launch_fcm_regen(c, c->opt.engine == XBS_ENGINE_INTERP_FCM, c->stream);
  c->launches += 1;
}

void regenerate_all(xbs_core* c) {
  if (c->fully_ideal) return;
  if (c->tile_engine) regenerate_tiles(c);
  else xbs::launch_regen_all(c, c->stream);
}

// fcm.cpp:186-190: a tile without a fixed point raises ConvergenceError
void check_fcm(xbs_core* c) {
  if (!c->tile_engine || c->h_sc->fcm_fail == 0) return;
  const double r = __builtin_bit_cast(double, c->h_sc->fcm_residual);
  fail(XBS_CONVERGENCE_ERROR, "fcm_convert: no fixed point after " + std::to_string(c->opt.fcm_max_iter) +
                                  " sweeps (residual " + std::to_string(r) + ")");
}

// host col-major (ld) <-> device row-major (rows x cols)
void h2d_colmajor_to_rowmajor(xbs_core* c, const double* h, int64_t rows, int64_t cols, int64_t ld, double* d) {
  c->h_tmp.assign(size_t(rows * cols), 0.0);
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) c->h_tmp[size_t(i * cols + j)] = h[j * ld + i];
  // stream-ordered with the kernels that consume it (the core's stream is
  // non-blocking, so a legacy-stream copy would not order against it)
  ck(cudaMemcpyAsync(d, c->h_tmp.data(), size_t(rows * cols) * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaStreamSynchronize(c->stream), "H2D");  // h_tmp is reused by the next call
}
void d2h_rowmajor_to_colmajor(xbs_core* c, const double* d, int64_t rows, int64_t cols, double* h, int64_t ld) {
  c->h_tmp.resize(size_t(rows * cols));
  ck(cudaMemcpyAsync(c->h_tmp.data(), d, size_t(rows * cols) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "D2H");
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) h[j * ld + i] = c->h_tmp[size_t(i * cols + j)];
}

// CUDA-event bracket around one stage (only while profiling is enabled).
cudaEvent_t take_event(xbs_core* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  ck(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

struct StageScope {
  xbs_core* c;
  int stage;
  cudaEvent_t a = nullptr;
  static cudaEvent_t take(xbs_core* c) { return take_event(c); }
  StageScope(xbs_core* cc, int s) : c(cc), stage(s) {
    if (c->profile) {
      a = take(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~StageScope() {
    if (a) {
      cudaEvent_t b = take(c);
      cudaEventRecord(b, c->stream);
      c->pending.push_back({stage, a, b});
    }
  }
};

void collect_stage_times(xbs_core* c) {
  if (c->pending.empty()) return;
  sync(c);
  for (auto& p : c->pending) {
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, p.a, p.b), "cudaEventElapsedTime");
    c->stage_ms[p.stage] += ms;
    c->stage_n[p.stage] += 1;
    c->ev_pool.push_back(p.a);
    c->ev_pool.push_back(p.b);
  }
  c->pending.clear();
}

// Quantising ADC with full scale i_fs for one direction (0 forward, 1
// backward): converters.cpp:79-87 on the snapped current I = n 2^sh is
// monotone in n, so T[k] = min{n : code(n) >= k} decides every code exactly;
// the tcgen05 epilogues use it for the boundary cases.
void set_adc(xbs_core* c, int dir, double i_fs) {
  xbs::AdcP& a = dir == 0 ? c->adc : c->adc_b;
  unsigned long long*& tab = dir == 0 ? c->d_adc_tab : c->d_adc_tab_b;
  ++c->gen;
  a.passthrough = 0;
  a.i_fs = i_fs;
  const double fac = i_fs / (std::pow(2.0, c->opt.adc_bits) - 1.0);
  (dir == 0 ? c->ifs_fac : c->ifs_fac_b) = fac;
  if (tab) {
    sync(c);
    cudaFree(tab);
    tab = nullptr;
  }
  if (!(i_fs > 0)) return;  // calibrated without observations: adc_quantize throws on use
  auto code = [&](uint64_t n) {
    const double scaled = std::ldexp(double(n), a.sh) / a.i_fs * a.maxc_d;
    return scaled >= a.maxc_d ? int64_t(a.maxc) : int64_t(std::llround(scaled));
  };
  std::vector<unsigned long long> T(size_t(a.maxc) + 1, 0ull);
  const uint64_t top = uint64_t(1) << 44;  // > 65025^2 * 256 >= any column current
  for (int k = 1; k <= a.maxc; ++k) {
    uint64_t lo = k > 1 ? T[size_t(k) - 1] : 0, hi = top;
    if (code(hi) < k) {
      T[size_t(k)] = top;
      continue;
    }
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      if (code(mid) >= k) hi = mid;
      else lo = mid + 1;
    }
    T[size_t(k)] = lo;
  }
  ck(cudaMalloc(&tab, T.size() * 8), "cudaMalloc adc table");
  ck(cudaMemcpyAsync(tab, T.data(), T.size() * 8, cudaMemcpyHostToDevice, c->stream), "H2D adc table");
  ck(cudaStreamSynchronize(c->stream), "H2D adc table");  // T is local
}

// layers.cpp:189-197: after adc_cal_batches training forwards, each
// direction's i_fs becomes the nearest-rank clip_percentile quantile of the
// currents it observed (converters.cpp:96-107), chosen on the device by an
// exact radix select over the recorded n.
void maybe_freeze_adc(xbs_core* c) {
  if (!c->adc_auto || c->adc_frozen) return;
  if (c->training_batches < c->opt.adc_cal_batches) return;
  double ifs[2] = {0.0, 0.0};  // adc.i_fs as configured (<= 0) stays "unset"
  for (int dir = 0; dir < 2; ++dir) {
    uint64_t n = 0;  // the selected integer current, or (volts mode) the fp64 current's bit pattern
    if (!xbs::calib_select(c, dir, c->opt.adc_clip_percentile, &n)) ifs[dir] = c->opt.adc_i_fs;
    else ifs[dir] = c->volts_mode ? __builtin_bit_cast(double, n) : std::ldexp(double(n), c->adc.sh);
  }
  xbs::calib_release(c);
  c->adc_frozen = true;
  if (c->volts_mode) {  // the fp64 kernels quantise with adc_quantize itself: no threshold table
    ++c->gen;
    const double maxc = std::pow(2.0, c->opt.adc_bits) - 1.0;
    c->adc.i_fs = c->volts.i_fs = ifs[0];
    c->adc_b.i_fs = c->volts.i_fs_b = ifs[1];
    c->adc.passthrough = c->adc_b.passthrough = 0;
    c->volts.passthrough = 0;
    c->ifs_fac = ifs[0] / maxc;
    c->ifs_fac_b = ifs[1] / maxc;
  } else {
    set_adc(c, 0, ifs[0]);
    set_adc(c, 1, ifs[1]);
  }
  c->adc_scaled = true;
  c->k_out_fwd = c->sx * c->F / c->vu * c->ifs_fac;  // layers.cpp:278-281
}

bool calibrating(const xbs_core* c) { return c->adc_auto && !c->adc_frozen; }

// Output of a VMM call: a device buffer (column stride M), or the device
// alias of the caller's pinned host buffer (stride ld).  The tcgen05 kernels
// store straight into a host buffer from their epilogues, so the D2H
// transfer overlaps the VMM; the other kernels write d_io_out, copied after.
struct Out {
  double* p;
  int64_t ld;  // 0: M
  bool host;
};

// Device alias of a pinned, mapped host buffer; nullptr for pageable memory.
double* mapped_alias(const double* h) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr) return nullptr;
  return static_cast<double*>(at.devicePointer);
}

void finish_out(xbs_core* c, const Out& o, int64_t M, int64_t cols, bool direct) {
  if (o.host && !direct)
    ck(cudaMemcpy2DAsync(o.p, size_t(o.ld) * 8, c->d_io_out, size_t(M) * 8, size_t(M) * 8, size_t(cols),
                         cudaMemcpyDefault, c->stream),
       "D2H");
}

void enqueue_fwd_vmm(xbs_core* c, int64_t M, const Out& out) {
  const int64_t ld = out.ld ? out.ld : M;
  double* stage = out.host ? c->d_io_out : out.p;  // written with stride M
  bool direct = false;
  c->out_host = out.host;
  if (c->fully_ideal) {
    xbs::launch_fwd_ideal(c, M, stage, c->stream);
  } else if (c->volts_mode) {
    xbs::launch_fwd_volts(c, M, stage, c->stream);
  } else if (c->kernel == 1 || c->big_tiles || c->adc.passthrough ||
             !(direct = xbs::launch_fwd_tc(c, M, out.p, ld, c->stream))) {
    // shape outside the tcgen05 kernel's exact bounds (tiles above 256 x 256 are SIMT by design)
    if (c->kernel == 0 && !c->big_tiles && !c->adc.passthrough) ++c->tc_fallbacks;
    xbs::launch_fwd_simt(c, M, stage, c->stream);
  }
  finish_out(c, Out{out.p, ld, out.host}, M, c->g.N, direct);
}

void enqueue_bwd_vmm(xbs_core* c, const double* d_dy, int64_t M, const Out& out) {
  const int64_t ld = out.ld ? out.ld : M;
  double* stage = out.host ? c->d_io_out : out.p;
  bool direct = false;
  c->out_host = out.host;
  if (c->fully_ideal) {
    xbs::launch_bwd_ideal(c, d_dy, M, stage, c->stream);
  } else if (c->volts_mode) {
    xbs::launch_bwd_volts(c, M, stage, c->stream);
  } else if (c->kernel == 1 || c->big_tiles || c->adc.passthrough ||
             !(direct = xbs::launch_bwd_tc(c, M, out.p, ld, c->stream))) {
    if (c->kernel == 0 && !c->big_tiles && !c->adc.passthrough) ++c->tc_fallbacks;
    xbs::launch_bwd_simt(c, M, stage, c->stream);
  }
  finish_out(c, Out{out.p, ld, out.host}, M, c->g.K, direct);
}

// Replays `enqueue` (pure stream work on c->stream) from a CUDA graph when
// the same call repeats: the first call with a key runs eagerly, the second
// is captured and instantiated, later ones launch the executable graph (one
// launch instead of ~5-12 kernels and memsets).  Host-side state is updated
// by the caller on every call, outside the graph.
template <class F>
void run_graphed(xbs_core* c, xbs_core::GraphSlot& g, const uint64_t (&key)[8], F&& enqueue) {
  uint64_t k[8];
  std::memcpy(k, key, sizeof k);
  k[7] = c->gen;
  const bool same = std::memcmp(k, g.key, sizeof k) == 0;
  if (same && g.ready) {
    ck(cudaGraphLaunch(g.exec, c->stream), "cudaGraphLaunch");
    c->launches += g.kernels;
    c->tc_fallbacks += g.fallbacks;
    return;
  }
  if (!same || !g.seen) {  // new key: run eagerly, capture on the next identical call
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    g.ready = false;
    std::memcpy(g.key, k, sizeof k);
    g.seen = true;
    enqueue();
    return;
  }
  const int64_t l0 = c->launches, f0 = c->tc_fallbacks;
  ck(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  cudaGraph_t graph = nullptr;
  try {
    enqueue();
  } catch (...) {
    cudaStreamEndCapture(c->stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    (void)cudaGetLastError();
    g.seen = false;
    throw;
  }
  ck(cudaStreamEndCapture(c->stream, &graph), "cudaStreamEndCapture");
  const cudaError_t e = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  ck(e, "cudaGraphInstantiate");
  g.kernels = c->launches - l0;
  g.fallbacks = c->tc_fallbacks - f0;
  c->launches = l0;
  c->tc_fallbacks = f0;
  g.ready = true;
  ck(cudaGraphLaunch(g.exec, c->stream), "cudaGraphLaunch");
  c->launches += g.kernels;
  c->tc_fallbacks += g.fallbacks;
}

bool graphable(const xbs_core* c, int64_t M) { return c->use_graphs && !c->profile && !c->adc_auto && M > 0; }

uint64_t u64(const void* p) { return uint64_t(reinterpret_cast<uintptr_t>(p)); }
uint64_t u64(double v) { return __builtin_bit_cast(uint64_t, v); }

void forward_device(xbs_core* c, const double* d_x, int64_t M, bool training, Out out,
                    const xbs::ConvSrc* conv = nullptr) {
  if (M < 0) fail(XBS_INVALID_ARGUMENT, "CrossbarCore::forward: negative batch");
  maybe_freeze_adc(c);
  if (c->adc_auto && c->adc_frozen && !(c->adc.i_fs > 0) && M > 0)
    fail(XBS_STATE_ERROR, "adc_quantize: i_fs not set (calibrate first)");  // converters.cpp:83-84
  ensure_batch(c, std::max<int64_t>(M, 1));
  if (graphable(c, M)) {
    uint64_t key[8] = {u64(d_x), uint64_t(M), u64(out.p), uint64_t(out.ld), uint64_t(out.host), 0, 0, 0};
    if (conv) {
      key[5] = uint64_t(conv->batch) ^ (uint64_t(conv->h) << 32) ^ (uint64_t(conv->w) << 48);
      key[6] = uint64_t(conv->in_c) ^ (uint64_t(conv->k) << 16) ^ (uint64_t(conv->stride) << 24) ^
               (uint64_t(conv->pad) << 32) ^ (uint64_t(1) << 63);
    }
    run_graphed(c, c->gfwd, key, [&] {
      xbs::launch_prep_x(c, d_x, M, c->stream, conv);
      c->launches += 2;
      enqueue_fwd_vmm(c, M, out);
    });
    c->have_forward = true;
    c->M_fwd = M;
    if (training) ++c->training_batches;  // layers.cpp:224
    return;
  }
  {
    StageScope st(c, XBS_STAGE_PREP_X);
    xbs::launch_prep_x(c, d_x, M, c->stream, conv);
    c->launches += M > 0 ? 1 : 0;
  }
  c->have_forward = true;
  c->M_fwd = M;
  if (training) ++c->training_batches;  // layers.cpp:224
  if (M == 0) return;
  if (calibrating(c) && training) xbs::calib_observe_fwd(c, M, c->stream);
  StageScope st(c, XBS_STAGE_FWD);
  c->launches += 1;
  enqueue_fwd_vmm(c, M, out);
}

// dW (layers.cpp:304) with its finiteness flag: cleared, raised by the dW
// kernels, and copied to the pinned host mirror so a host apply_updates can
// refuse a non-finite gradient synchronously (update.cpp:18-19).
void enqueue_dw(xbs_core* c, int64_t M, double gd) {
  ck(cudaMemsetAsync(&c->d_sc->dw_nonfinite, 0, sizeof(int), c->stream), "memset");
  if (c->kernel == 1 || !xbs::launch_dw_tc(c, M, gd, c->stream)) xbs::launch_dw(c, M, gd, c->stream);
  ck(cudaMemcpyAsync(&c->h_sc->dw_nonfinite, &c->d_sc->dw_nonfinite, sizeof(int), cudaMemcpyDeviceToHost, c->stream),
     "D2H flag");
}

void backward_device(xbs_core* c, const double* d_dy, int64_t M, double gd, Out out) {
  if (!c->have_forward) fail(XBS_STATE_ERROR, "CrossbarCore::backward: no cached forward activations");
  if (M != c->M_fwd) fail(XBS_INVALID_ARGUMENT, "CrossbarCore::backward: gradient shape mismatch");
  maybe_freeze_adc(c);
  if (graphable(c, M)) {
    const uint64_t key[8] = {u64(d_dy), uint64_t(M), u64(out.p), uint64_t(out.ld), uint64_t(out.host), u64(gd), 0, 0};
    run_graphed(c, c->gbwd, key, [&] {
      xbs::launch_prep_dy(c, d_dy, M, c->stream);
      c->launches += 3;
      enqueue_dw(c, M, gd);
      c->launches += 2;
      enqueue_bwd_vmm(c, d_dy, M, out);
    });
    c->have_grad = true;
    return;
  }
  {
    StageScope st(c, XBS_STAGE_PREP_DY);
    xbs::launch_prep_dy(c, d_dy, M, c->stream);
    c->launches += M > 0 ? 3 : 2;
  }
  {
    StageScope st(c, XBS_STAGE_DW);
    enqueue_dw(c, M, gd);
    c->launches += 1;
  }
  c->have_grad = true;
  if (M == 0) return;
  if (c->adc_auto && c->adc_frozen && !(c->adc_b.i_fs > 0)) {
    double se = 0.0;  // layers.cpp:308: a zero error never reaches the ADC
    ck(cudaMemcpyAsync(&c->h_sc->se, &c->d_sc->se, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H se");
    sync(c);
    se = c->h_sc->se;
    if (se > 0) fail(XBS_STATE_ERROR, "adc_quantize: i_fs not set (calibrate first)");
  }
  if (calibrating(c)) xbs::calib_observe_bwd(c, M, c->stream);
  StageScope st(c, XBS_STAGE_BWD);
  c->launches += 1;
  enqueue_bwd_vmm(c, d_dy, M, out);
}

void apply_updates_device(xbs_core* c, uint64_t iteration) {
  if (!c->have_grad) return;  // layers.cpp:383
  // dwmax / wmax are running maxima on the device and err_flag is sticky:
  // nothing is reset here, so device-path steps lose no statistic
  xbs::UpdP up{};
  up.v = c->opt.upd_v;
  up.gamma = c->opt.upd_gamma;
  up.lr = c->opt.upd_lr;
  const double ls = c->opt.upd_layer_scale == 0.0 ? c->layer_scale : c->opt.upd_layer_scale;  // update.cpp:52
  up.factor = (c->opt.g_max - c->opt.g_min) / ls;
  const double levels = double((uint64_t{1} << c->g.wb) - 1), sl = double((uint64_t{1} << c->g.db) - 1);
  up.wfactor = (c->layer_scale / (c->opt.g_max - c->opt.g_min)) * (sl / levels);
  up.seed = c->opt.upd_seed;
  up.iteration = iteration;
  up.linear = c->opt.upd_v == 0.0;
  cudaEvent_t e0 = take_event(c), e1 = take_event(c);
  ck(cudaEventRecord(e0, c->stream), "event record");
  {
    StageScope st(c, XBS_STAGE_UPDATE);
    xbs::launch_update(c, up, c->stream, c->tile_engine);  // tile engines: master only, then per-tile regeneration
    ++c->update_count;                                     // layers.cpp:389
    if (c->tile_engine) regenerate_tiles(c);
    regenerate_bookkeeping(c);
  }
  ck(cudaEventRecord(e1, c->stream), "event record");
  c->upd_timing.emplace_back(e0, e1);
  c->stats_pending = true;
  c->launches += c->opt.engine == XBS_ENGINE_IDEAL ? 2 : 1;
  c->have_grad = false;
  c->have_forward = false;
}


}  // namespace

namespace xbs {
void core_forward_conv(xbs_core* c, const double* d_img, const ConvSrc& cs, bool training, double* d_y) {
  const int64_t rows = cs.batch * cs.oh * cs.ow;
  if (rows >= (int64_t(1) << 31)) fail(XBS_UNSUPPORTED, "CrossbarConv2d: more than 2^31 patch rows");
  forward_device(c, d_img, rows, training, Out{d_y, 0, false}, &cs);
}
}  // namespace xbs

namespace xbs {  // error plumbing shared with the conv layer (xbs_conv.cu)
int set_error(int code, const std::string& m) {
  g_err = m;
  return code;
}
void fail_conv(int code, const std::string& m) { fail(code, m); }
void check_rc(int rc) {
  if (rc != XBS_OK) throw XbsError(rc, g_err);
}
int guard_conv(const std::function<void()>& f) { return guard(f); }
}  // namespace xbs

extern "C" {

int32_t xbs_abi_version(void) { return XBS_ABI_VERSION; }
const char* xbs_last_error(void) { return g_err.c_str(); }

void xbs_options_init(xbs_layer_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->weight_bits = 8;  // MappingSpec defaults (mapping.hpp:15-21)
  o->device_bits = 2;
  o->tile_rows = 64;
  o->tile_cols = 64;
  o->variation_sigma = 0.0;
  o->variation_seed = 0;
  o->w_max = 0.0;
  o->xbar_rows = 64;  // CrossbarConfig defaults (crossbar.hpp:18-26)
  o->xbar_cols = 64;
  o->r_row = 1.0;
  o->r_col = 4.6;
  o->r_source = 0.0;
  o->r_sense = 0.0;
  o->g_min = 1e-6;
  o->g_max = 1e-5;
  o->v_fs = 1.0;
  o->dac_bits = 1;  // DacSpec (converters.hpp:15-18)
  o->dac_stream_bits = 1;
  o->dac_v_fs = 1.0;
  o->adc_bits = 8;  // AdcSpec (converters.hpp:38-41)
  o->adc_i_fs = 0.0;
  o->adc_clip_percentile = 0.999;
  o->upd_v = 0.0;  // UpdateSpec (update.hpp:14-20)
  o->upd_gamma = 0.0;
  o->upd_lr = 0.01;
  o->upd_seed = 0;
  o->upd_layer_scale = 0.0;
  o->engine = XBS_ENGINE_FCM;  // CrossbarLayerOptions (layers.hpp:25-34)
  o->interp_base = XBS_ENGINE_FCM;
  o->interp_interval = 10;
  o->fcm_tol = 1e-6;
  o->fcm_max_iter = 1000;
  o->act_bits = 8;
  o->act_full_scale = 1.0;
  o->error_bits = 8;
  o->adc_cal_batches = 20;
  o->threads = 1;
}

}  // extern "C"

namespace {
// CrossbarCore::CrossbarCore (layers.cpp:68-83).  weights_only: just
// mapping::map_weights (mapping.cpp:83-131) -- geometry, layer scale and the
// device master, for the free-function TiledLayerWeights (xbs_weights.cu).
xbs_core* create_core(const xbs_layer_options* opt, const double* W0, int64_t K, int64_t N, int64_t ldw,
                      bool weights_only) {
    if (!opt) fail(XBS_INVALID_ARGUMENT, "xbs_core_create: null argument");
    auto c = std::make_unique<xbs_core>();
    c->weights_only = weights_only;
    c->opt = *opt;
    if (opt->dac_transfer && opt->dac_transfer_len > 0)
      c->dac_tr.assign(opt->dac_transfer, opt->dac_transfer + opt->dac_transfer_len);
    if (opt->adc_transfer && opt->adc_transfer_len > 0)
      c->adc_tr.assign(opt->adc_transfer, opt->adc_transfer + opt->adc_transfer_len);
    c->opt.dac_transfer = nullptr;
    c->opt.adc_transfer = nullptr;
    const xbs_layer_options& o = c->opt;
    // map_weights validates first (layers.cpp:69 -> mapping.cpp:85-90)
    validate_crossbar(o);
    validate_mapping(o);
    if (K == 0 || N == 0) fail(XBS_INVALID_ARGUMENT, "map_weights: empty weight matrix");
    if (K < 0 || N < 0 || ldw < K || !W0) fail(XBS_INVALID_ARGUMENT, "map_weights: bad weight matrix");
    double wabs = 0.0;
    for (int64_t j = 0; j < N; ++j)
      for (int64_t i = 0; i < K; ++i) {
        const double w = W0[j * ldw + i];
        if (!std::isfinite(w)) fail(XBS_INVALID_ARGUMENT, "map_weights: weights must be finite");
        wabs = std::max(wabs, std::abs(w));
      }
    if (!weights_only) {
      validate_options(o, c->dac_tr, c->adc_tr);  // layers.cpp:70
      check_scope(o, c->dac_tr, c->adc_tr);
    }

    xbs::Geo& g = c->g;
    g.K = int(K);
    g.N = int(N);
    g.tile_rows = o.tile_rows;
    g.tile_cols = o.tile_cols;
    g.GR = (g.K + o.tile_rows - 1) / o.tile_rows;
    g.GC = (g.N + o.tile_cols - 1) / o.tile_cols;
    g.Kp = g.GR * o.tile_rows;
    g.Np = g.GC * o.tile_cols;
    g.R = ((o.tile_rows + 127) / 128) * 128;
    g.C = ((o.tile_cols + 127) / 128) * 128;
    g.KI = g.GR * g.R;
    g.NI = g.GC * g.C;
    // narrow layers (one 128-column tile, N <= 64): the error planes keep only
    // the 32 / 64 columns the backward MMA's K = 32 steps can touch, so the
    // prep writes and the tcgen05 operand loads skip the padding
    g.NB = (g.GC == 1 && g.C == 128 && g.N <= 64) ? (g.N <= 32 ? 32 : 64) : g.NI;
    g.S = o.weight_bits / o.device_bits;
    g.db = o.device_bits;
    g.wb = o.weight_bits;
    g.Ti = o.act_bits;
    g.TPi = next_pow2(o.act_bits);
    g.Te = o.error_bits;
    g.TPe = next_pow2(o.error_bits);

    double scale = o.w_max > 0 ? o.w_max : wabs;  // mapping.cpp:104-105
    if (scale == 0.0) scale = 1.0;
    c->layer_scale = scale;
    c->level_step = (o.g_max - o.g_min) / double((uint64_t{1} << o.device_bits) - 1);

    c->fully_ideal = o.engine == XBS_ENGINE_IDEAL && o.variation_sigma == 0.0 && c->dac_tr.empty() && o.adc_bits == 0;
    const bool zero_par = o.r_row == 0.0 && o.r_col == 0.0 && o.r_source == 0.0 && o.r_sense == 0.0;
    xbs::RegenP& rp = c->rp;
    rp.g_min = o.g_min;
    rp.g_max = o.g_max;
    rp.range = o.g_max - o.g_min;
    rp.sigma = o.variation_sigma;
    rp.vseed = o.variation_seed;
    rp.r_row = o.r_row;
    rp.r_col = o.r_col;
    rp.r_source = o.r_source;
    rp.r_sense = o.r_sense;
    rp.aam = (o.engine == XBS_ENGINE_AAM && !zero_par) ? 1 : 0;
    c->tile_engine = (o.engine == XBS_ENGINE_FCM || o.engine == XBS_ENGINE_INTERP_FCM) && !zero_par;
    c->fcm = xbs::FcmP{o.r_row, o.r_col, o.r_source, o.r_sense, o.v_fs, o.fcm_tol, o.fcm_max_iter, 1};
    rp.snap_e = snap_exponent(o.g_max);
    rp.snap_scale = std::ldexp(1.0, rp.snap_e);
    rp.kpnp = uint64_t(g.Kp) * g.Np;
    rp.varm = nullptr;

    // scale constants, same expressions as layers.cpp:272-281 / 369-377
    const double vu = o.dac_v_fs / (std::pow(2.0, o.dac_bits) - 1.0);
    const double sx = o.act_full_scale / (std::pow(2.0, o.act_bits) - 1.0);
    const double levels = std::pow(2.0, o.weight_bits) - 1.0;
    const double slice_levels = std::pow(2.0, o.device_bits) - 1.0;
    const double F = (scale / (o.g_max - o.g_min)) * (slice_levels / levels);
    c->vu = vu;
    c->F = F;
    c->sx = o.act_full_scale / double((1 << o.act_bits) - 1);  // tensor.cpp:29 (codes_to_values)
    c->lev_e = std::pow(2.0, o.error_bits) - 1.0;
    c->adc_auto = o.adc_bits > 0 && !(o.adc_i_fs > 0) && c->adc_tr.empty();  // layers.cpp:74
    c->adc_scaled = o.adc_bits > 0 && c->adc_tr.empty() && !c->adc_auto;      // layers.cpp:280
    c->ifs_fac = c->adc_scaled ? o.adc_i_fs / (std::pow(2.0, o.adc_bits) - 1.0) : 1.0;
    c->ifs_fac_b = c->ifs_fac;
    double k_out = sx * F / vu;
    if (c->adc_scaled) k_out *= c->ifs_fac;
    c->k_out_fwd = k_out;

    xbs::AdcP& a = c->adc;
    a.passthrough = o.adc_bits == 0 || c->adc_auto;  // calibration batches pass currents through
    a.maxc = o.adc_bits > 0 && o.adc_bits <= 16 ? int((1u << o.adc_bits) - 1) : 0;
    a.maxc_d = double(a.maxc);
    a.i_fs = o.adc_i_fs;
    int lv;
    (void)std::frexp(o.dac_v_fs, &lv);
    a.sh = (lv - 1) - rp.snap_e;
    c->adc_b = a;

    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    if (weights_only) {
      ck(cudaMalloc(&c->d_master, size_t(g.S) * g.Kp * g.Np * 8), "cudaMalloc master");
      ck(cudaMalloc(&c->d_dW, size_t(g.K) * g.N * 8), "cudaMalloc dW");
      ck(cudaMalloc(&c->d_sc, sizeof(xbs::DevScalars)), "cudaMalloc scalars");
      ck(cudaMemsetAsync(c->d_sc, 0, sizeof(xbs::DevScalars), c->stream), "memset scalars");
      ck(cudaMallocHost(&c->h_sc, sizeof(xbs::DevScalars)), "cudaMallocHost");
      double* d_W = nullptr;
      ck(cudaMalloc(&d_W, size_t(K) * N * 8), "cudaMalloc W");
      ck(cudaMemcpy2DAsync(d_W, size_t(K) * 8, W0, size_t(ldw) * 8, size_t(K) * 8, size_t(N), cudaMemcpyHostToDevice,
                           c->stream),
         "H2D W");
      xbs::launch_map_weights(c.get(), d_W, c->stream);
      ck(cudaStreamSynchronize(c->stream), "map_weights");
      cudaFree(d_W);
      return c.release();
    }
    c->volts_mode = volts_mode(o, c->dac_tr, c->adc_tr);
    c->big_tiles = o.tile_rows > 256 || o.tile_cols > 256;
    if (c->volts_mode) {
      // dac_encode of every digit (converters.cpp:28-35) and the ADC spec
      const uint64_t levels = (uint64_t{1} << o.dac_bits) - 1;
      std::vector<double> lut(size_t(levels) + 1);
      for (uint64_t d = 0; d <= levels; ++d)
        lut[d] = !c->dac_tr.empty() ? c->dac_tr[d] : d == 0 ? 0.0 : double(d) / double(levels) * o.dac_v_fs;
      ck(cudaMalloc(&c->d_dac_lut, lut.size() * 8), "cudaMalloc dac lut");
      ck(cudaMemcpy(c->d_dac_lut, lut.data(), lut.size() * 8, cudaMemcpyHostToDevice), "H2D dac lut");
      if (!c->adc_tr.empty()) {
        ck(cudaMalloc(&c->d_adc_tr, c->adc_tr.size() * 8), "cudaMalloc adc table");
        ck(cudaMemcpy(c->d_adc_tr, c->adc_tr.data(), c->adc_tr.size() * 8, cudaMemcpyHostToDevice), "H2D adc table");
      }
      xbs::VoltsP& v = c->volts;
      v.lut = c->d_dac_lut;
      v.sb = o.dac_stream_bits;
      v.passthrough = o.adc_bits == 0 || c->adc_auto;  // calibration batches pass currents through
      v.adc_tr = c->d_adc_tr;
      v.tr_len = int(c->adc_tr.size());
      v.maxcode = o.adc_bits > 0 ? (uint64_t{1} << o.adc_bits) - 1 : 0;
      v.maxc_d = double(v.maxcode);
      v.i_fs = v.i_fs_b = o.adc_i_fs;
    } else if (!a.passthrough) {
      set_adc(c.get(), 0, o.adc_i_fs);
      set_adc(c.get(), 1, o.adc_i_fs);
    }
    if (c->adc_auto) {
      ck(cudaMalloc(&c->d_obs_count, 2 * sizeof(unsigned long long)), "cudaMalloc calibration counters");
      ck(cudaMemsetAsync(c->d_obs_count, 0, 2 * sizeof(unsigned long long), c->stream), "memset");
    }
    ck(cudaMalloc(&c->d_master, size_t(g.S) * g.Kp * g.Np * 8), "cudaMalloc master");
    ck(cudaMalloc(&c->d_digits, g.digits_bytes()), "cudaMalloc digits");
    ck(cudaMemsetAsync(c->d_digits, 0, g.digits_bytes(), c->stream), "memset digits");
    ck(cudaMalloc(&c->d_dW, size_t(g.K) * g.N * 8), "cudaMalloc dW");
    ck(cudaMemsetAsync(c->d_dW, 0, size_t(g.K) * g.N * 8, c->stream), "memset dW");
    if (o.engine == XBS_ENGINE_IDEAL) ck(cudaMalloc(&c->d_wimp, size_t(g.K) * g.N * 8), "cudaMalloc wimp");
    ck(cudaMalloc(&c->d_sc, sizeof(xbs::DevScalars)), "cudaMalloc scalars");
    ck(cudaMemsetAsync(c->d_sc, 0, sizeof(xbs::DevScalars), c->stream), "memset scalars");
    ck(cudaMallocHost(&c->h_sc, sizeof(xbs::DevScalars)), "cudaMallocHost");

    // W0 -> device (contiguous column-major K x N) -> master
    double* d_W = nullptr;
    ck(cudaMalloc(&d_W, size_t(K) * N * 8), "cudaMalloc W");
    ck(cudaMemcpy2DAsync(d_W, size_t(K) * 8, W0, size_t(ldw) * 8, size_t(K) * 8, size_t(N), cudaMemcpyHostToDevice,
                         c->stream),
       "H2D W");
    xbs::launch_map_weights(c.get(), d_W, c->stream);
    if (o.variation_sigma == 0.0 && !c->fully_ideal) {
      ck(cudaMalloc(&c->d_qmin, size_t(o.tile_rows) * o.tile_cols * sizeof(uint32_t)), "cudaMalloc qmin");
      xbs::launch_qmin(c.get(), c->stream);
    }
    if (o.variation_sigma != 0.0 && !c->fully_ideal) {
      ck(cudaMalloc(&c->d_varm, size_t(g.S) * 2 * size_t(g.Kp) * g.Np * sizeof(double)), "cudaMalloc variation");
      c->rp.varm = c->d_varm;
      xbs::launch_varm(c.get(), c->stream);
    }
    if (c->tile_engine && o.engine == XBS_ENGINE_INTERP_FCM) {
      const size_t n = size_t(g.S) * 2 * size_t(g.Kp) * g.Np * sizeof(double);
      ck(cudaMalloc(&c->d_cache_d, n), "cudaMalloc distortion cache");
      ck(cudaMalloc(&c->d_cache_g, n), "cudaMalloc distortion cache");
      ck(cudaMalloc(&c->d_cache_gn, n), "cudaMalloc distortion cache");
    }
    const auto t0 = std::chrono::steady_clock::now();
    regenerate_all(c.get());
    regenerate_bookkeeping(c.get());
    sync(c.get());
    ck(cudaMemcpyAsync(c->h_sc, c->d_sc, sizeof(xbs::DevScalars), cudaMemcpyDeviceToHost, c->stream), "D2H scalars");
    ck(cudaStreamSynchronize(c->stream), "D2H scalars");
    check_fcm(c.get());
    c->conversion_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    cudaFree(d_W);
    return c.release();
}
}  // namespace

namespace xbs {
xbs_core* create_weights_core(const xbs_layer_options* opt, const double* W, int64_t K, int64_t N, int64_t ldw) {
  return create_core(opt, W, K, N, ldw, true);
}
void core_settle(xbs_core* c) { sync(c); }
void core_h2d_rowmajor(xbs_core* c, const double* h, int64_t rows, int64_t cols, int64_t ld, double* d) {
  h2d_colmajor_to_rowmajor(c, h, rows, cols, ld, d);
}
void core_d2h_rowmajor(xbs_core* c, const double* d, int64_t rows, int64_t cols, double* h, int64_t ld) {
  d2h_rowmajor_to_colmajor(c, d, rows, cols, h, ld);
}
}  // namespace xbs

extern "C" {

int xbs_options_validate(const xbs_layer_options* opt) {
  return guard([&] {
    if (!opt) fail(XBS_INVALID_ARGUMENT, "xbs_options_validate: null argument");
    std::vector<double> dac_tr, adc_tr;
    if (opt->dac_transfer && opt->dac_transfer_len > 0)
      dac_tr.assign(opt->dac_transfer, opt->dac_transfer + opt->dac_transfer_len);
    if (opt->adc_transfer && opt->adc_transfer_len > 0)
      adc_tr.assign(opt->adc_transfer, opt->adc_transfer + opt->adc_transfer_len);
    validate_options(*opt, dac_tr, adc_tr);  // layers.cpp:17-47
  });
}

int xbs_core_create(const xbs_layer_options* opt, const double* W0, int64_t K, int64_t N, int64_t ldw,
                    xbs_core** out) {
  return guard([&] {
    if (!out) fail(XBS_INVALID_ARGUMENT, "xbs_core_create: null argument");
    *out = nullptr;
    *out = create_core(opt, W0, K, N, ldw, false);
  });
}

void xbs_core_destroy(xbs_core* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  if (c->copy_ev) cudaEventDestroy(c->copy_ev);
  for (auto& e : c->upd_timing) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  cudaFree(c->d_digits);
  cudaFree(c->d_adc_tab);
  cudaFree(c->d_adc_tab_b);
  xbs::calib_release(c);
  cudaFree(c->d_obs_count);
  cudaFree(c->d_qmin);
  cudaFree(c->d_dac_lut);
  cudaFree(c->d_adc_tr);
  cudaFree(c->d_varm);
  cudaFree(c->d_fcm_scratch);
  cudaFree(c->d_cache_d);
  cudaFree(c->d_cache_g);
  cudaFree(c->d_cache_gn);
  cudaFree(c->d_master);
  cudaFree(c->d_dW);
  cudaFree(c->d_wimp);
  cudaFree(c->d_sc);
  cudaFreeHost(c->h_sc);
  cudaFree(c->d_Af);
  cudaFree(c->d_Ab);
  cudaFree(c->d_xcodes);
  cudaFree(c->d_xcodes32);
  cudaFree(c->d_ecodes);
  cudaFree(c->d_xc8);
  cudaFree(c->d_e8);
  cudaFree(c->d_S64);
  cudaFree(c->d_acc32);
  if (c->gfwd.exec) cudaGraphExecDestroy(c->gfwd.exec);
  if (c->gbwd.exec) cudaGraphExecDestroy(c->gbwd.exec);
  cudaFree(c->d_io_in);
  cudaFree(c->d_io_out);
  for (auto& p : c->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->stream && c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int xbs_core_forward(xbs_core* c, const double* x, int64_t M, int64_t K, int64_t ldx, int32_t training, double* y,
                     int64_t ldy) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    if (K != c->g.K) fail(XBS_INVALID_ARGUMENT, "CrossbarCore::forward: feature count mismatch");  // layers.cpp:216-217
    if (M < 0 || (M > 0 && (ldx < M || ldy < M || !x || !y))) fail(XBS_INVALID_ARGUMENT, "CrossbarCore::forward: bad buffers");
    ensure_io(c, std::max<int64_t>(1, M * std::max(c->g.K, c->g.N)));
    if (M > 0 && c->upd_async) {
      // the pending update does not touch the staging buffer: copy x on the
      // side stream while it runs, and order the forward after both
      if (!c->copy_stream) {
        ck(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaEventCreateWithFlags(&c->copy_ev, cudaEventDisableTiming), "cudaEventCreate");
      }
      ck(cudaMemcpy2DAsync(c->d_io_in, size_t(M) * 8, x, size_t(ldx) * 8, size_t(M) * 8, size_t(c->g.K),
                           cudaMemcpyHostToDevice, c->copy_stream),
         "H2D x");
      ck(cudaEventRecord(c->copy_ev, c->copy_stream), "event record");
      ck(cudaStreamWaitEvent(c->stream, c->copy_ev, 0), "stream wait");
    } else if (M > 0) {
      ck(cudaMemcpy2DAsync(c->d_io_in, size_t(M) * 8, x, size_t(ldx) * 8, size_t(M) * 8, size_t(c->g.K),
                           cudaMemcpyHostToDevice, c->stream),
         "H2D x");
    }
    double* ym = M > 0 ? mapped_alias(y) : nullptr;  // pinned: the kernel stores y into it
    forward_device(c, c->d_io_in, M, training != 0, ym ? Out{ym, ldy, true} : Out{c->d_io_out, 0, false});
    if (M > 0 && !ym)
      ck(cudaMemcpy2DAsync(y, size_t(ldy) * 8, c->d_io_out, size_t(M) * 8, size_t(M) * 8, size_t(c->g.N),
                           cudaMemcpyDeviceToHost, c->stream),
         "D2H y");
    sync(c);
  });
}

int xbs_core_backward(xbs_core* c, const double* dy, int64_t M, int64_t N, int64_t lddy, double gd, double* dx,
                      int64_t lddx) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    if (!c->have_forward) fail(XBS_STATE_ERROR, "CrossbarCore::backward: no cached forward activations");
    if (N != c->g.N || M != c->M_fwd) fail(XBS_INVALID_ARGUMENT, "CrossbarCore::backward: gradient shape mismatch");
    if (M > 0 && (lddy < M || lddx < M || !dy || !dx)) fail(XBS_INVALID_ARGUMENT, "CrossbarCore::backward: bad buffers");
    ensure_io(c, std::max<int64_t>(1, M * std::max(c->g.K, c->g.N)));
    if (M > 0)
      ck(cudaMemcpy2DAsync(c->d_io_in, size_t(M) * 8, dy, size_t(lddy) * 8, size_t(M) * 8, size_t(c->g.N),
                           cudaMemcpyHostToDevice, c->stream),
         "H2D dy");
    double* dxm = M > 0 ? mapped_alias(dx) : nullptr;
    backward_device(c, c->d_io_in, M, gd, dxm ? Out{dxm, lddx, true} : Out{c->d_io_out, 0, false});
    if (M > 0 && !dxm)
      ck(cudaMemcpy2DAsync(dx, size_t(lddx) * 8, c->d_io_out, size_t(M) * 8, size_t(M) * 8, size_t(c->g.K),
                           cudaMemcpyDeviceToHost, c->stream),
         "D2H dx");
    sync(c);
  });
}

int xbs_core_apply_updates(xbs_core* c, uint64_t iteration) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    if (!c->have_grad) return;
    sync(c);  // the dW producer is complete and the previous update folded
    // scale_gradient (update.cpp:18-19): a non-finite gradient throws before
    // anything changes (the dW kernels raised the flag, or set_gradient did)
    if (c->h_sc->dw_nonfinite) fail(XBS_INVALID_ARGUMENT, "scale_gradient: gradient must be finite");
    // Engines whose update cannot raise (AAM / ideal regeneration, linear
    // update: no range check, update.cpp:28-29, no FCM convergence; the
    // gradient was checked above) return before the kernels finish; the next
    // call settles timing and statistics and a forward overlaps its input
    // copy with them.  Others stay synchronous so their exceptions surface
    // here, as in the reference.
    const bool defer = (c->opt.engine == XBS_ENGINE_AAM || c->opt.engine == XBS_ENGINE_IDEAL) &&
                       c->opt.upd_v == 0.0 && !c->profile;
    apply_updates_device(c, iteration);
    ck(cudaGetLastError(), "kernel launch");
    if (defer) {
      c->upd_async = true;
      return;
    }
    sync(c);
  });
}

int xbs_core_forward_device(xbs_core* c, const double* d_x, int64_t M, int32_t training, double* d_y) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    forward_device(c, d_x, M, training != 0, Out{d_y, 0, false});
  });
}
int xbs_core_backward_device(xbs_core* c, const double* d_dy, int64_t M, double gd, double* d_dx) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    backward_device(c, d_dy, M, gd, Out{d_dx, 0, false});
  });
}
int xbs_core_apply_updates_device(xbs_core* c, uint64_t iteration) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    apply_updates_device(c, iteration);
  });
}
int xbs_core_synchronize(xbs_core* c) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    sync(c);
  });
}

int xbs_core_get_info(xbs_core* c, xbs_core_info* info) {
  return guard([&] {
    if (!c || !info) fail(XBS_INVALID_ARGUMENT, "null argument");
    settle(c);
    std::memset(info, 0, sizeof(*info));
    info->in_features = c->g.K;
    info->out_features = c->g.N;
    info->grid_rows = c->g.GR;
    info->grid_cols = c->g.GC;
    info->padded_rows = c->g.Kp;
    info->padded_cols = c->g.Np;
    info->num_slices = c->g.S;
    info->snap_exponent = c->rp.snap_e;
    info->layer_scale = c->layer_scale;
    info->level_step = c->level_step;
    info->refresh_count = c->refreshes;
    info->conversion_seconds = c->conversion_seconds;
    info->weight_abs_max_seen = c->wmax_seen;
    info->grad_abs_max_seen = c->dwmax_seen;
    info->forward_adc_full_scale = c->adc_auto && c->adc_frozen ? c->adc.i_fs : c->opt.adc_i_fs;
    info->fully_ideal = c->fully_ideal ? 1 : 0;
    info->kernel = c->kernel;
    info->tc_fallbacks = c->tc_fallbacks;
  });
}

int xbs_core_gradient(xbs_core* c, double* dW, int64_t ld) {
  return guard([&] {
    if (!c || !dW || ld < c->g.K) fail(XBS_INVALID_ARGUMENT, "bad gradient buffer");
    sync(c);
    d2h_rowmajor_to_colmajor(c, c->d_dW, c->g.K, c->g.N, dW, ld);
  });
}

int xbs_core_set_gradient(xbs_core* c, const double* dW, int64_t ld) {
  return guard([&] {
    if (!c || !dW || ld < c->g.K) fail(XBS_INVALID_ARGUMENT, "bad gradient buffer");
    sync(c);
    h2d_colmajor_to_rowmajor(c, dW, c->g.K, c->g.N, ld, c->d_dW);
    bool finite = true;  // checked when the update runs (update.cpp:18-19), like a backward's dW
    for (double v : c->h_tmp) finite = finite && std::isfinite(v);
    c->h_sc->dw_nonfinite = finite ? 0 : 1;
    ck(cudaMemcpyAsync(&c->d_sc->dw_nonfinite, &c->h_sc->dw_nonfinite, sizeof(int), cudaMemcpyHostToDevice, c->stream),
       "H2D flag");
    ck(cudaStreamSynchronize(c->stream), "H2D flag");
    c->have_grad = true;
  });
}

int xbs_core_nonideal(xbs_core* c, int32_t s, int32_t p, int32_t t, double* out, int64_t ld) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    if (c->fully_ideal) fail(XBS_STATE_ERROR, "CrossbarCore: no non-ideal state for the ideal fast path");
    if (s < 0 || s >= c->g.S || p < 0 || p > 1 || t < 0 || t >= c->g.GR * c->g.GC)
      fail(XBS_INVALID_ARGUMENT, "nonideal: index out of range");  // std::vector::at -> out_of_range
    if (!out || ld < c->g.tile_rows) fail(XBS_INVALID_ARGUMENT, "bad output buffer");
    const int n = c->g.tile_rows * c->g.tile_cols;
    double* d = nullptr;
    ck(cudaMalloc(&d, size_t(n) * 8), "cudaMalloc");
    xbs::launch_digits_to_g(c, s, p, t / c->g.GC, t % c->g.GC, d, c->stream);
    sync(c);
    std::vector<double> h(static_cast<size_t>(n));
    ck(cudaMemcpyAsync(h.data(), d, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "D2H");
    cudaFree(d);
    for (int j = 0; j < c->g.tile_cols; ++j)
      for (int i = 0; i < c->g.tile_rows; ++i) out[int64_t(j) * ld + i] = h[size_t(j) * c->g.tile_rows + i];
  });
}

int xbs_core_master(xbs_core* c, int32_t s, double* u, int64_t ld) {
  return guard([&] {
    if (!c || s < 0 || s >= c->g.S || !u || ld < c->g.Kp) fail(XBS_INVALID_ARGUMENT, "master: bad arguments");
    sync(c);
    d2h_rowmajor_to_colmajor(c, c->d_master + size_t(s) * c->g.Kp * c->g.Np, c->g.Kp, c->g.Np, u, ld);
  });
}

int xbs_core_set_master(xbs_core* c, int32_t s, const double* u, int64_t ld) {
  return guard([&] {
    if (!c || s < 0 || s >= c->g.S || !u || ld < c->g.Kp) fail(XBS_INVALID_ARGUMENT, "set_master: bad arguments");
    sync(c);
    h2d_colmajor_to_rowmajor(c, u, c->g.Kp, c->g.Np, ld, c->d_master + size_t(s) * c->g.Kp * c->g.Np);
    regenerate_all(c);
    if (c->opt.engine == XBS_ENGINE_IDEAL) xbs::launch_implied(c, c->d_wimp, c->stream);
    sync(c);
    ck(cudaMemcpyAsync(c->h_sc, c->d_sc, sizeof(xbs::DevScalars), cudaMemcpyDeviceToHost, c->stream), "D2H scalars");
    ck(cudaStreamSynchronize(c->stream), "D2H scalars");
    check_fcm(c);
  });
}

int xbs_core_implied_weights(xbs_core* c, double* w, int64_t ld) {
  return guard([&] {
    if (!c || !w || ld < c->g.K) fail(XBS_INVALID_ARGUMENT, "implied_weights: bad arguments");
    double* d = nullptr;
    ck(cudaMalloc(&d, size_t(c->g.K) * c->g.N * 8), "cudaMalloc");
    xbs::launch_implied(c, d, c->stream);
    sync(c);
    d2h_rowmajor_to_colmajor(c, d, c->g.K, c->g.N, w, ld);
    cudaFree(d);
  });
}

int xbs_core_adc_counters(xbs_core* c, int64_t* exact_path, int64_t* conversions) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    sync(c);
    ck(cudaMemcpyAsync(c->h_sc, c->d_sc, sizeof(xbs::DevScalars), cudaMemcpyDeviceToHost, c->stream), "D2H scalars");
    ck(cudaStreamSynchronize(c->stream), "D2H scalars");
    if (exact_path) *exact_path = int64_t(c->h_sc->exact_path);
    if (conversions) *conversions = int64_t(c->h_sc->conversions);
  });
}

int xbs_core_select_kernel(xbs_core* c, int32_t kernel) {
  return guard([&] {
    if (!c || kernel < 0 || kernel > 1) fail(XBS_INVALID_ARGUMENT, "select_kernel: 0 (tcgen05) or 1 (SIMT)");
    settle(c);
    c->kernel = kernel;
    ++c->gen;
  });
}

void* xbs_core_stream(xbs_core* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int xbs_core_set_stream(xbs_core* c, void* stream) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    sync(c);  // work already queued on the old stream completes first
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
      ++c->gen;
      c->own_stream = false;
    } else {
      ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
      c->own_stream = true;
    }
  });
}

int xbs_core_use_graphs(xbs_core* c, int32_t enable) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    settle(c);
    c->use_graphs = enable != 0;
  });
}

int xbs_core_profile(xbs_core* c, int32_t enable) {
  return guard([&] {
    if (!c) fail(XBS_INVALID_ARGUMENT, "null core");
    settle(c);
    collect_stage_times(c);
    c->profile = enable != 0;
    for (int i = 0; i < XBS_NUM_STAGES; ++i) {
      c->stage_ms[i] = 0.0;
      c->stage_n[i] = 0;
    }
  });
}

int xbs_core_stage_times(xbs_core* c, double* ms, int64_t* count, int32_t n) {
  return guard([&] {
    if (!c || n < 0 || n > XBS_NUM_STAGES) fail(XBS_INVALID_ARGUMENT, "stage_times: bad arguments");
    settle(c);
    collect_stage_times(c);
    for (int i = 0; i < n; ++i) {
      if (ms) ms[i] = c->stage_ms[i];
      if (count) count[i] = c->stage_n[i];
    }
  });
}

int64_t xbs_core_launch_count(xbs_core* c) { return c ? c->launches : 0; }

}  // extern "C"
