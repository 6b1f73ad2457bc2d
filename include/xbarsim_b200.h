/*
 * xbarsim_b200.h — C ABI of the B200-native crossbar-evaluation hot path.
 *
 * Drop-in boundary for xbarsim::nn::CrossbarCore
 * (/root/reference/proj/core/include/xbarsim/layers.hpp:49-111).  Plain
 * pointers and sizes only; no CUDA, torch or C++ types cross this line, and no
 * exception crosses it: every entry point returns an xbs_status and leaves a
 * thread-local message in xbs_last_error().  The C++ classes in
 * include/xbarsim/ (and the Python mirror paper_2002_11151_b200.xbarsim) wrap
 * these calls and rethrow the reference's exception types.
 *
 * Host matrices follow the reference's storage: Eigen::MatrixXd is
 * column-major, so element (i, j) of an R x C matrix with leading dimension ld
 * lives at p[j * ld + i].
 *
 * Every call on a core is synchronous at return (like the reference), except
 * the *_device entry points, which enqueue on the core's CUDA stream and
 * return immediately (xbs_core_synchronize waits).
 */
#ifndef XBARSIM_B200_H_
#define XBARSIM_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XBS_ABI_VERSION 3

/* Status codes: one per reference exception class (errors.hpp:10-47). */
typedef enum xbs_status {
  XBS_OK = 0,
  XBS_INVALID_ARGUMENT = 1,        /* std::invalid_argument                 */
  XBS_STATE_ERROR = 2,             /* xbarsim::StateError                    */
  XBS_CONFIG_ERROR = 3,            /* xbarsim::ConfigError                   */
  XBS_CONVERGENCE_ERROR = 4,       /* xbarsim::ConvergenceError              */
  XBS_STALE_CACHE_ERROR = 5,       /* xbarsim::StaleCacheError               */
  XBS_DEGENERATE_CIRCUIT_ERROR = 6,/* xbarsim::DegenerateCircuitError        */
  XBS_UNSUPPORTED = 7,             /* valid reference config outside this
                                      path's scope (the oracle engine with
                                      parasitics, DAC streams above 16 bits,
                                      tiles above 1024 x 1024, fcm on tiles
                                      above 256 x 256, an auto-calibration
                                      sample larger than the device); maps
                                      to ConfigError in the C++ wrapper      */
  XBS_CUDA_ERROR = 8,              /* device fault; StateError + CUDA string */
  XBS_INTERNAL = 9
} xbs_status;

/* EngineKind (engine.hpp:15-35). */
enum { XBS_ENGINE_IDEAL = 0, XBS_ENGINE_ORACLE = 1, XBS_ENGINE_FCM = 2, XBS_ENGINE_AAM = 3,
       XBS_ENGINE_INTERP_FCM = 4 };

/* Flat POD mirroring CrossbarLayerOptions (layers.hpp:19-37) and the specs
 * it aggregates.  xbs_options_init() fills the reference defaults. */
typedef struct xbs_layer_options {
  /* MappingSpec (mapping.hpp:14-25) */
  int32_t weight_bits, device_bits, tile_rows, tile_cols;
  double variation_sigma;
  uint64_t variation_seed;
  double w_max;
  /* CrossbarConfig (crossbar.hpp:17-40) */
  int32_t xbar_rows, xbar_cols;
  double r_row, r_col, r_source, r_sense, g_min, g_max, v_fs;
  /* DacSpec (converters.hpp:14-22) */
  int32_t dac_bits, dac_stream_bits;
  double dac_v_fs;
  const double* dac_transfer; /* NULL: ideal linear */
  int32_t dac_transfer_len;
  /* AdcSpec (converters.hpp:37-45) */
  int32_t adc_bits;
  double adc_i_fs;
  const double* adc_transfer; /* NULL: linear */
  int32_t adc_transfer_len;
  double adc_clip_percentile;
  /* UpdateSpec (update.hpp:13-23) */
  double upd_v, upd_gamma, upd_lr;
  uint64_t upd_seed;
  double upd_layer_scale;
  /* CrossbarLayerOptions proper */
  int32_t engine, interp_base, interp_interval;
  double fcm_tol;
  int32_t fcm_max_iter;
  int32_t act_bits;
  double act_full_scale;
  int32_t error_bits, adc_cal_batches, threads;
} xbs_layer_options;

/* Reference statistics getters (layers.hpp:64-68) plus geometry. */
typedef struct xbs_core_info {
  int32_t in_features, out_features;          /* K, N                        */
  int32_t grid_rows, grid_cols;               /* TiledLayerWeights grid      */
  int32_t padded_rows, padded_cols;           /* Kp, Np                      */
  int32_t num_slices;
  int32_t snap_exponent;                      /* e of the 2^-e grid          */
  double layer_scale, level_step;
  int64_t refresh_count;                      /* refresh_count()             */
  double conversion_seconds;                  /* conversion_seconds()        */
  double weight_abs_max_seen;                 /* weight_abs_max_seen()       */
  double grad_abs_max_seen;                   /* grad_abs_max_seen()         */
  double forward_adc_full_scale;              /* forward_adc_full_scale()    */
  int32_t fully_ideal;                        /* fully_ideal() fast path     */
  int32_t kernel;                             /* 0 = tcgen05, 1 = SIMT check */
  int64_t tc_fallbacks;                       /* forward / backward VMM calls whose
                                                 shape left the tcgen05 kernels'
                                                 exact int32 / fp32 bounds, so the
                                                 exact SIMT kernel ran instead  */
} xbs_core_info;

typedef struct xbs_core xbs_core;

int32_t xbs_abi_version(void);
const char* xbs_last_error(void);
void xbs_options_init(xbs_layer_options* opt);

/* CrossbarCore::CrossbarCore(W0, opt) — layers.cpp:68-83.  W0 is K x N,
 * column-major with leading dimension ldw >= K. */
int xbs_core_create(const xbs_layer_options* opt, const double* W0, int64_t K, int64_t N, int64_t ldw,
                    xbs_core** out);
void xbs_core_destroy(xbs_core* core);

/* CrossbarCore::forward(x, training) — layers.cpp:215-284.  x: M x K
 * (K must equal in_features, else XBS_INVALID_ARGUMENT as layers.cpp:216-217),
 * y: M x N, column-major host buffers. */
int xbs_core_forward(xbs_core* core, const double* x, int64_t M, int64_t K, int64_t ldx, int32_t training,
                     double* y, int64_t ldy);
/* CrossbarCore::backward(dy, grad_divisor) — layers.cpp:286-380.  dy: M x N,
 * dx: M x K, column-major host buffers.  Checks in the reference's order:
 * no cached forward -> XBS_STATE_ERROR, then N != out_features or M != the
 * forward batch -> XBS_INVALID_ARGUMENT (layers.cpp:287-290). */
int xbs_core_backward(xbs_core* core, const double* dy, int64_t M, int64_t N, int64_t lddy, double grad_divisor,
                      double* dx, int64_t lddx);
/* CrossbarCore::apply_updates(iteration) — layers.cpp:382-391.  When the
 * update cannot raise (engine AAM or ideal, update.v == 0, profiling off) the
 * call returns once the update is queued on the core's stream; every later
 * call on the core settles it (statistics, conversion_seconds) before it
 * reads state, so results are those of the synchronous call.  Other engines
 * return after completion, so ConvergenceError / range errors surface here. */
int xbs_core_apply_updates(xbs_core* core, uint64_t iteration);

/* Device-resident variants (HBM pointers, column-major, ld = M): enqueue on
 * the core's stream, return at once.  Same semantics as the host calls. */
int xbs_core_forward_device(xbs_core* core, const double* d_x, int64_t M, int32_t training, double* d_y);
int xbs_core_backward_device(xbs_core* core, const double* d_dy, int64_t M, double grad_divisor,
                             double* d_dx);
int xbs_core_apply_updates_device(xbs_core* core, uint64_t iteration);
int xbs_core_synchronize(xbs_core* core);

/* Accessors (layers.hpp:59-71).  Host copies. */
int xbs_core_get_info(xbs_core* core, xbs_core_info* info);
int xbs_core_gradient(xbs_core* core, double* dW, int64_t ld);             /* K x N */
int xbs_core_set_gradient(xbs_core* core, const double* dW, int64_t ld);   /* feeds apply_update
                                                                               (update.hpp:51-52) */
int xbs_core_nonideal(xbs_core* core, int32_t slice, int32_t polarity, int32_t tile, double* g,
                      int64_t ld);                                         /* tile_rows x tile_cols */
int xbs_core_master(xbs_core* core, int32_t slice, double* u, int64_t ld);  /* Kp x Np */
int xbs_core_set_master(xbs_core* core, int32_t slice, const double* u, int64_t ld);
int xbs_core_implied_weights(xbs_core* core, double* w, int64_t ld);       /* K x N */

/* Diagnostics for the parity harness: ADC conversions that took the exact
 * fp64 boundary path in the last forward/backward, and total conversions. */
int xbs_core_adc_counters(xbs_core* core, int64_t* exact_path, int64_t* conversions);
/* Select the VMM kernel: 0 = tcgen05 (default), 1 = exact SIMT cross-check. */
int xbs_core_select_kernel(xbs_core* core, int32_t kernel);
/* CUDA stream (cudaStream_t) the core enqueues on, as an opaque pointer. */
void* xbs_core_stream(xbs_core* core);
/* Enqueue on the caller's stream from now on (e.g. all layers of a network
 * on one stream); the core never destroys a caller's stream.  NULL returns
 * to a private stream.  Waits for work queued on the previous stream. */
int xbs_core_set_stream(xbs_core* core, void* stream);

/* CrossbarConv2d (layers.hpp:136-152, layers.cpp:415-505): im2col lowering
 * onto one core, on the device.  W0 is (in_c*kernel*kernel) x out_c
 * column-major; tensors are batch x features column-major with features
 * ordered (c, y, x).  Backward uses grad_divisor 1.0 and the reference's
 * col2im summation order. */
typedef struct xbs_conv2d xbs_conv2d;
int xbs_conv2d_create(const xbs_layer_options* opt, const double* W0, int64_t ldw, int32_t in_c, int32_t out_c,
                      int32_t kernel, int32_t stride, int32_t padding, xbs_conv2d** out);
void xbs_conv2d_destroy(xbs_conv2d* conv);
xbs_core* xbs_conv2d_core(xbs_conv2d* conv);  /* borrowed; owned by the conv */
int xbs_conv2d_output_dims(xbs_conv2d* conv, int32_t h, int32_t w, int32_t* out_h, int32_t* out_w);
int xbs_conv2d_forward(xbs_conv2d* conv, const double* x, int64_t batch, int32_t c, int32_t h, int32_t w, int64_t ldx,
                       int32_t training, double* y, int64_t ldy);
int xbs_conv2d_backward(xbs_conv2d* conv, const double* dy, int64_t batch, int64_t lddy, double* dx, int64_t lddx);
int xbs_conv2d_forward_device(xbs_conv2d* conv, const double* d_x, int64_t batch, int32_t c, int32_t h, int32_t w,
                              int32_t training, double* d_y);
int xbs_conv2d_backward_device(xbs_conv2d* conv, const double* d_dy, int64_t batch, double* d_dx);
int xbs_conv2d_apply_updates(xbs_conv2d* conv, uint64_t iteration);

/* ---- Free functions of the operator API (mapping.hpp:92-109, update.hpp:25-52)
 *
 * mapping::TiledLayerWeights (mapping.hpp:39-90) as a device-resident
 * object: the per-slice signed master in HBM, mutated only by
 * xbs_apply_update / xbs_weights_set_master.  A view of a core's weights
 * (xbs_core_weights) reads the live core; setting its master regenerates
 * the core's conductances like xbs_core_set_master. */
typedef struct xbs_weights xbs_weights;
typedef struct xbs_weights_info {
  int32_t rows, cols;                 /* K, N                                 */
  int32_t padded_rows, padded_cols;   /* grid * tile dims                     */
  int32_t grid_rows, grid_cols;
  int32_t num_slices;
  int32_t tile_rows, tile_cols;
  int32_t weight_bits, device_bits;
  double layer_scale, level_step;
  double variation_sigma;
  uint64_t variation_seed;
  double g_min, g_max;                /* tile_config() conductance range      */
} xbs_weights_info;

/* mapping::map_weights(W, spec, cfg) (mapping.cpp:83-131): reads the
 * MappingSpec (weight_bits, device_bits, tile_rows/cols, variation_sigma /
 * seed, w_max) and CrossbarConfig fields of opt; the others are ignored.
 * Errors as the reference: CrossbarConfig / MappingSpec validation, then
 * non-finite and empty W -> XBS_INVALID_ARGUMENT. */
int xbs_map_weights(const xbs_layer_options* opt, const double* W, int64_t K, int64_t N, int64_t ldw,
                    xbs_weights** out);
/* mapping::apply_variation(t, sigma, seed) (mapping.cpp:133-140): a copy
 * carrying new variation parameters; the master is copied unchanged. */
int xbs_weights_apply_variation(const xbs_weights* w, double sigma, uint64_t seed, xbs_weights** out);
/* View of a core's weights (CrossbarCore::weights(), layers.hpp:59); owned by
 * the core, valid until xbs_core_destroy; destroy the view with
 * xbs_weights_destroy (the core is untouched). */
int xbs_core_weights(xbs_core* core, xbs_weights** out);
void xbs_weights_destroy(xbs_weights* w);
int xbs_weights_get_info(const xbs_weights* w, xbs_weights_info* info);
/* master_diff(slice) / mutable_master_diff(slice) write-back (padded dims). */
int xbs_weights_master(const xbs_weights* w, int32_t slice, double* u, int64_t ld);
int xbs_weights_set_master(xbs_weights* w, int32_t slice, const double* u, int64_t ld);
/* master_polarity(slice, p) (mapping.cpp:39-45) and ideal_working(slice, p)
 * (mapping.cpp:47-58, variation from the counter RNG): padded dims. */
int xbs_weights_master_polarity(const xbs_weights* w, int32_t slice, int32_t polarity, double* g, int64_t ld);
int xbs_weights_ideal_working(const xbs_weights* w, int32_t slice, int32_t polarity, double* g, int64_t ld);
/* implied_weights() (mapping.cpp:70-81): K x N. */
int xbs_weights_implied(const xbs_weights* w, double* W, int64_t ld);

/* UpdateSpec (update.hpp:13-23) */
typedef struct xbs_update_spec {
  double v, gamma, lr;
  uint64_t seed;
  double layer_scale; /* 0: the weights' mapping scale */
} xbs_update_spec;
/* update::apply_update(t, dW, spec, iteration) (update.cpp:43-88): the
 * master only, on the device; the caller regenerates (a core view refuses:
 * CrossbarCore::apply_updates does update + regeneration).  UpdateSpec
 * validation, shape mismatch and a non-finite dW -> XBS_INVALID_ARGUMENT
 * before anything changes; a device state outside [g_min, g_max] ->
 * XBS_INVALID_ARGUMENT (nonlinear_update, update.cpp:28-29). */
int xbs_apply_update(xbs_weights* w, const double* dW, int64_t K, int64_t N, int64_t ld, const xbs_update_spec* spec,
                     uint64_t iteration);
/* update::scale_gradient (update.cpp:16-24): out = dW * ((g_max - g_min) /
 * layer_scale), K x N column-major; layer_scale == 0 -> XBS_CONFIG_ERROR,
 * non-finite dW -> XBS_INVALID_ARGUMENT. */
int xbs_scale_gradient(const double* dW, int64_t K, int64_t N, int64_t ld, double layer_scale, double g_min,
                       double g_max, double* out, int64_t ldo);
/* update::nonlinear_update (update.cpp:26-33), elementwise over n devices;
 * any g outside [g_min, g_max] -> XBS_INVALID_ARGUMENT. */
int xbs_nonlinear_update(const double* g, const double* dg, int64_t n, double v, double g_min, double g_max,
                         double* out);
/* update::write_noise (update.cpp:35-41), elementwise: element i draws one
 * Gaussian from the counter RNG (rng.hpp) with key keys[i] at counters
 * counters[i] + 1 and + 2, unless its deviation is 0 (then out[i] = 0 and
 * nothing is drawn, as in the reference); drew[i] (nullable) = 1 if it drew.
 * The caller advances its CounterRng by 2 per drawing element. */
int xbs_write_noise(const double* dg, int64_t n, double gamma, double g_min, double g_max, const uint64_t* keys,
                    const uint64_t* counters, double* out, int32_t* drew);
/* mapping::reconstruct_output (mapping.cpp:142-160): codes_pos / codes_neg
 * are slices x n (slice-major, contiguous); out = scale * sum_s
 * 2^(s*device_bits) (pos_s - neg_s) in the reference's order. */
int xbs_reconstruct_output(const double* codes_pos, const double* codes_neg, int32_t slices, int64_t n,
                           int32_t device_bits, double scale, double* out);
/* CrossbarLayerOptions::validate (layers.cpp:17-47): the reference's checks
 * and exception classes, no device work. */
int xbs_options_validate(const xbs_layer_options* opt);

/* Per-stage device timing (CUDA events recorded on the core's stream around
 * each stage while enabled).  Stages: 0 prep_x (K0a), 1 forward VMM (K1),
 * 2 prep_dy (K0b), 3 dW (K3a), 4 backward VMM (K2), 5 update+regeneration
 * (K3b).  xbs_core_stage_times synchronizes and returns the accumulated
 * milliseconds and the number of timed instances per stage (n <= 6). */
enum { XBS_STAGE_PREP_X = 0, XBS_STAGE_FWD = 1, XBS_STAGE_PREP_DY = 2, XBS_STAGE_DW = 3, XBS_STAGE_BWD = 4,
       XBS_STAGE_UPDATE = 5, XBS_NUM_STAGES = 6 };
int xbs_core_profile(xbs_core* core, int32_t enable);
/* CUDA graphs (default on): a forward / backward call that repeats the
 * previous call's buffers and shape is replayed from a captured graph (one
 * launch); results are identical with graphs off.  Stage profiling and ADC
 * auto-calibration always run eagerly. */
int xbs_core_use_graphs(xbs_core* core, int32_t enable);
int xbs_core_stage_times(xbs_core* core, double* ms, int64_t* count, int32_t n);
/* Number of this library's kernels launched by the core so far. */
int64_t xbs_core_launch_count(xbs_core* core);

#ifdef __cplusplus
}
#endif
#endif /* XBARSIM_B200_H_ */
