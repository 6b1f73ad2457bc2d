// Free functions of the operator API on the device (mapping.hpp:92-109,
// update.hpp:25-52): mapping::TiledLayerWeights as an HBM-resident object
// (a weights-only core: geometry, layer scale, per-slice master), the
// master-only update::apply_update, and the elementwise helpers the
// reference exposes (scale_gradient, nonlinear_update, write_noise,
// reconstruct_output).  The fused core update (xbs_kernels.cu k_update) is
// the hot path; these entry points reuse its kernels and arithmetic.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "xbs_internal.cuh"
#include "xbs_rng.cuh"

struct xbs_weights {
  xbs_core* c = nullptr;
  bool view = false;  // a core's weights (CrossbarCore::weights()): the core owns c
};

namespace xbs {
namespace {

int blocks(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16))); }

// mapping.cpp:39-58: g = max(+-u, 0) + g_min, then (sigma != 0) the
// variation multiplier m = max(1 + sigma N(0,1), 1e-12) keyed (seed, 2 s + p,
// i * Np + j) and g = min(g * m, g_max).  Output row-major Kp x Np.
__global__ void k_ideal_working(Geo g, double g_min, double g_max, double sigma, uint64_t seed, int s, int p,
                                const double* __restrict__ u, double* __restrict__ out) {
  const int64_t n = int64_t(g.Kp) * g.Np;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const double v = p == 0 ? u[t] : -u[t];
    double gv = fmax(v, 0.0) + g_min;
    if (sigma != 0.0) {
      double m = 1.0 + sigma * rng_gaussian(rng_key(seed, uint64_t(s) * 2 + p, uint64_t(t), 0));
      m = m > 1e-12 ? m : 1e-12;
      gv = fmin(gv * m, g_max);
    }
    out[t] = gv;
  }
}

// update.cpp:16-24 on a column-major K x N matrix
__global__ void k_scale_gradient(const double* __restrict__ dW, int64_t K, int64_t N, int64_t ld, double factor,
                                 double* __restrict__ out, int64_t ldo, int* nonfinite) {
  const int64_t n = K * N;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = t / K, i = t - j * K;
    const double w = dW[j * ld + i];
    if (!isfinite(w)) *nonfinite = 1;
    out[j * ldo + i] = w * factor;
  }
}

// update.cpp:26-33
__global__ void k_nonlinear(const double* __restrict__ g, const double* __restrict__ dg, int64_t n, double v,
                            double g_min, double g_max, double* __restrict__ out, int* range_err) {
  const double range = g_max - g_min;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const double gg = g[t], d = dg[t];
    if (gg < g_min || gg > g_max) {
      *range_err = 1;
      out[t] = 0.0;
      continue;
    }
    const double x = d >= 0.0 ? (gg - g_min) / range : (g_max - gg) / range;
    out[t] = d * exp(-v * x);
  }
}

// update.cpp:35-41
__global__ void k_write_noise(const double* __restrict__ dg, int64_t n, double gamma, double range,
                              const uint64_t* __restrict__ keys, const uint64_t* __restrict__ ctr,
                              double* __restrict__ out, int32_t* __restrict__ drew) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    const double sigma = gamma * sqrt(range * fabs(dg[t]));
    const bool d = sigma != 0.0;
    out[t] = d ? sigma * rng_gaussian_at(keys[t], ctr[t]) : 0.0;
    if (drew) drew[t] = d ? 1 : 0;
  }
}

// mapping.cpp:142-160: acc += w * (pos_s - neg_s), w *= 2^db, in slice order
__global__ void k_reconstruct(const double* __restrict__ pos, const double* __restrict__ neg, int slices, int64_t n,
                              double base, double scale, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
    double acc = 0.0, w = 1.0;
    for (int s = 0; s < slices; ++s) {
      acc += w * (pos[s * n + t] - neg[s * n + t]);
      w *= base;
    }
    out[t] = scale * acc;
  }
}

// Device scratch of one call (freed on scope exit).
struct Scratch {
  std::vector<void*> p;
  template <class T>
  T* get(size_t count) {
    void* q = nullptr;
    ck_cuda(cudaMalloc(&q, std::max<size_t>(1, count) * sizeof(T)), "cudaMalloc");
    p.push_back(q);
    return static_cast<T*>(q);
  }
  ~Scratch() {
    for (void* q : p) cudaFree(q);
  }
};

int read_flag(const int* d, cudaStream_t st) {
  int h = 0;
  ck_cuda(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H flag");
  ck_cuda(cudaStreamSynchronize(st), "kernel execution");
  return h;
}

void check_slice(const xbs_weights* w, int32_t s) {
  if (!w || !w->c) fail_conv(XBS_INVALID_ARGUMENT, "null weights");
  if (s < 0 || s >= w->c->g.S) fail_conv(XBS_INVALID_ARGUMENT, "TiledLayerWeights: slice out of range");
}

}  // namespace
}  // namespace xbs

using xbs::ck_cuda;
using xbs::fail_conv;
using xbs::guard_conv;

extern "C" {

int xbs_map_weights(const xbs_layer_options* opt, const double* W, int64_t K, int64_t N, int64_t ldw,
                    xbs_weights** out) {
  return guard_conv([&] {
    if (!out) fail_conv(XBS_INVALID_ARGUMENT, "xbs_map_weights: null argument");
    *out = nullptr;
    auto* w = new xbs_weights;
    try {
      w->c = xbs::create_weights_core(opt, W, K, N, ldw);
    } catch (...) {
      delete w;
      throw;
    }
    *out = w;
  });
}

int xbs_weights_apply_variation(const xbs_weights* w, double sigma, uint64_t seed, xbs_weights** out) {
  return guard_conv([&] {
    if (!w || !w->c || !out) fail_conv(XBS_INVALID_ARGUMENT, "apply_variation: null argument");
    if (sigma < 0) fail_conv(XBS_INVALID_ARGUMENT, "apply_variation: sigma must be >= 0");  // mapping.cpp:135
    xbs::core_settle(w->c);
    const xbs_core* c = w->c;
    // a fresh weights object of the same geometry (map of a zero matrix),
    // then the master copied in and the variation parameters replaced
    xbs_layer_options o = c->opt;
    o.variation_sigma = sigma;
    o.variation_seed = seed;
    o.w_max = c->layer_scale;
    std::vector<double> zero(size_t(c->g.K) * c->g.N, 0.0);
    auto* r = new xbs_weights;
    try {
      r->c = xbs::create_weights_core(&o, zero.data(), c->g.K, c->g.N, c->g.K);
      r->c->layer_scale = c->layer_scale;
      ck_cuda(cudaMemcpyAsync(r->c->d_master, c->d_master, size_t(c->g.S) * c->g.Kp * c->g.Np * 8,
                              cudaMemcpyDeviceToDevice, r->c->stream),
              "D2D master");
      ck_cuda(cudaStreamSynchronize(r->c->stream), "D2D master");
    } catch (...) {
      if (r->c) xbs_core_destroy(r->c);
      delete r;
      throw;
    }
    *out = r;
  });
}

int xbs_core_weights(xbs_core* core, xbs_weights** out) {
  return guard_conv([&] {
    if (!core || !out) fail_conv(XBS_INVALID_ARGUMENT, "xbs_core_weights: null argument");
    auto* w = new xbs_weights;
    w->c = core;
    w->view = true;
    *out = w;
  });
}

void xbs_weights_destroy(xbs_weights* w) {
  if (!w) return;
  if (!w->view && w->c) xbs_core_destroy(w->c);
  delete w;
}

int xbs_weights_get_info(const xbs_weights* w, xbs_weights_info* info) {
  return guard_conv([&] {
    if (!w || !w->c || !info) fail_conv(XBS_INVALID_ARGUMENT, "null argument");
    const xbs_core* c = w->c;
    info->rows = c->g.K;
    info->cols = c->g.N;
    info->padded_rows = c->g.Kp;
    info->padded_cols = c->g.Np;
    info->grid_rows = c->g.GR;
    info->grid_cols = c->g.GC;
    info->num_slices = c->g.S;
    info->tile_rows = c->g.tile_rows;
    info->tile_cols = c->g.tile_cols;
    info->weight_bits = c->g.wb;
    info->device_bits = c->g.db;
    info->layer_scale = c->layer_scale;
    info->level_step = c->level_step;
    info->variation_sigma = c->rp.sigma;
    info->variation_seed = c->rp.vseed;
    info->g_min = c->rp.g_min;
    info->g_max = c->rp.g_max;
  });
}

int xbs_weights_master(const xbs_weights* w, int32_t s, double* u, int64_t ld) {
  return guard_conv([&] {
    xbs::check_slice(w, s);
    xbs_core* c = w->c;
    if (!u || ld < c->g.Kp) fail_conv(XBS_INVALID_ARGUMENT, "master: bad buffer");
    xbs::core_settle(c);
    xbs::core_d2h_rowmajor(c, c->d_master + size_t(s) * c->g.Kp * c->g.Np, c->g.Kp, c->g.Np, u, ld);
  });
}

int xbs_weights_set_master(xbs_weights* w, int32_t s, const double* u, int64_t ld) {
  if (w && w->view) return xbs_core_set_master(w->c, s, u, ld);  // regenerates the core's conductances
  return guard_conv([&] {
    xbs::check_slice(w, s);
    xbs_core* c = w->c;
    if (!u || ld < c->g.Kp) fail_conv(XBS_INVALID_ARGUMENT, "set_master: bad buffer");
    xbs::core_settle(c);
    xbs::core_h2d_rowmajor(c, u, c->g.Kp, c->g.Np, ld, c->d_master + size_t(s) * c->g.Kp * c->g.Np);
  });
}

static int polarity_or_working(const xbs_weights* w, int32_t s, int32_t p, double* g, int64_t ld, bool working) {
  return guard_conv([&] {
    xbs::check_slice(w, s);
    xbs_core* c = w->c;
    if (p < 0 || p > 1) fail_conv(XBS_INVALID_ARGUMENT, "polarity must be 0 (pos) or 1 (neg)");
    if (!g || ld < c->g.Kp) fail_conv(XBS_INVALID_ARGUMENT, "bad output buffer");
    xbs::core_settle(c);
    xbs::Scratch sc;
    double* d = sc.get<double>(size_t(c->g.Kp) * c->g.Np);
    const int64_t n = int64_t(c->g.Kp) * c->g.Np;
    xbs::k_ideal_working<<<xbs::blocks(n), 256, 0, c->stream>>>(c->g, c->rp.g_min, c->rp.g_max,
                                                                   working ? c->rp.sigma : 0.0, c->rp.vseed, s, p,
                                                                   c->d_master + size_t(s) * n, d);
    ck_cuda(cudaGetLastError(), "kernel launch");
    xbs::core_d2h_rowmajor(c, d, c->g.Kp, c->g.Np, g, ld);
  });
}

int xbs_weights_master_polarity(const xbs_weights* w, int32_t s, int32_t p, double* g, int64_t ld) {
  return polarity_or_working(w, s, p, g, ld, false);
}
int xbs_weights_ideal_working(const xbs_weights* w, int32_t s, int32_t p, double* g, int64_t ld) {
  return polarity_or_working(w, s, p, g, ld, true);
}

int xbs_weights_implied(const xbs_weights* w, double* W, int64_t ld) {
  if (w && w->view) return xbs_core_implied_weights(w->c, W, ld);
  return guard_conv([&] {
    if (!w || !w->c || !W || ld < w->c->g.K) fail_conv(XBS_INVALID_ARGUMENT, "implied_weights: bad arguments");
    xbs_core* c = w->c;
    xbs::core_settle(c);
    xbs::Scratch sc;
    double* d = sc.get<double>(size_t(c->g.K) * c->g.N);
    xbs::launch_implied(c, d, c->stream);
    xbs::core_d2h_rowmajor(c, d, c->g.K, c->g.N, W, ld);
  });
}

int xbs_apply_update(xbs_weights* w, const double* dW, int64_t K, int64_t N, int64_t ld, const xbs_update_spec* spec,
                     uint64_t iteration) {
  return guard_conv([&] {
    if (!w || !w->c || !spec) fail_conv(XBS_INVALID_ARGUMENT, "apply_update: null argument");
    if (w->view)
      fail_conv(XBS_INVALID_ARGUMENT,
                "apply_update: a core's weights change through CrossbarCore::apply_updates (update + regeneration)");
    // UpdateSpec::validate (update.cpp:10-14), then the shape (update.cpp:46-47)
    if (spec->v < 0) fail_conv(XBS_INVALID_ARGUMENT, "UpdateSpec: v must be >= 0");
    if (spec->gamma < 0) fail_conv(XBS_INVALID_ARGUMENT, "UpdateSpec: gamma must be >= 0");
    if (!(spec->lr > 0)) fail_conv(XBS_INVALID_ARGUMENT, "UpdateSpec: lr must be > 0");
    xbs_core* c = w->c;
    if (K != c->g.K || N != c->g.N) fail_conv(XBS_INVALID_ARGUMENT, "apply_update: gradient shape does not match layer");
    if (K > 0 && N > 0 && (!dW || ld < K)) fail_conv(XBS_INVALID_ARGUMENT, "apply_update: bad gradient buffer");
    xbs::core_settle(c);
    xbs::core_h2d_rowmajor(c, dW, K, N, ld, c->d_dW);
    for (int64_t j = 0; j < N; ++j)  // scale_gradient (update.cpp:18-19): nothing changes on a non-finite dW
      for (int64_t i = 0; i < K; ++i)
        if (!std::isfinite(dW[j * ld + i])) fail_conv(XBS_INVALID_ARGUMENT, "scale_gradient: gradient must be finite");
    const double ls = spec->layer_scale == 0.0 ? c->layer_scale : spec->layer_scale;  // update.cpp:52
    if (ls == 0.0) fail_conv(XBS_CONFIG_ERROR, "scale_gradient: layer_scale must be nonzero");
    xbs::UpdP up{};
    up.v = spec->v;
    up.gamma = spec->gamma;
    up.lr = spec->lr;
    up.factor = (c->rp.g_max - c->rp.g_min) / ls;
    up.wfactor = 0.0;
    up.seed = spec->seed;
    up.iteration = iteration;
    up.linear = spec->v == 0.0;
    ck_cuda(cudaMemsetAsync(c->d_sc, 0, sizeof(xbs::DevScalars), c->stream), "memset");
    xbs::launch_update(c, up, c->stream, true);
    ck_cuda(cudaGetLastError(), "kernel launch");
    if (xbs::read_flag(&c->d_sc->err_flag, c->stream) & 1)
      fail_conv(XBS_INVALID_ARGUMENT, "nonlinear_update: g outside device range");
  });
}

int xbs_scale_gradient(const double* dW, int64_t K, int64_t N, int64_t ld, double layer_scale, double g_min,
                       double g_max, double* out, int64_t ldo) {
  return guard_conv([&] {
    if (K < 0 || N < 0 || (K * N > 0 && (!dW || !out || ld < K || ldo < K)))
      fail_conv(XBS_INVALID_ARGUMENT, "scale_gradient: bad buffers");
    const int64_t n = K * N;
    xbs::Scratch sc;
    const double* d_in = nullptr;
    double* d_out = nullptr;
    int* flag = sc.get<int>(1);
    ck_cuda(cudaMemset(flag, 0, sizeof(int)), "memset");
    if (n > 0) {
      double* a = sc.get<double>(size_t(n));
      d_out = sc.get<double>(size_t(n));
      ck_cuda(cudaMemcpy2D(a, size_t(K) * 8, dW, size_t(ld) * 8, size_t(K) * 8, size_t(N), cudaMemcpyHostToDevice),
              "H2D");
      d_in = a;
      // the factor is applied only after the checks below pass; the kernel
      // runs with factor 1 when layer_scale is 0 so the finiteness check
      // still comes first (update.cpp:18-21)
      const double factor = layer_scale == 0.0 ? 1.0 : (g_max - g_min) / layer_scale;
      xbs::k_scale_gradient<<<xbs::blocks(n), 256>>>(d_in, K, N, K, factor, d_out, K, flag);
      ck_cuda(cudaGetLastError(), "kernel launch");
    }
    int nf = 0;
    ck_cuda(cudaMemcpy(&nf, flag, sizeof(int), cudaMemcpyDeviceToHost), "D2H flag");
    if (nf) fail_conv(XBS_INVALID_ARGUMENT, "scale_gradient: gradient must be finite");
    if (layer_scale == 0.0) fail_conv(XBS_CONFIG_ERROR, "scale_gradient: layer_scale must be nonzero");
    if (n > 0)
      ck_cuda(cudaMemcpy2D(out, size_t(ldo) * 8, d_out, size_t(K) * 8, size_t(K) * 8, size_t(N),
                           cudaMemcpyDeviceToHost),
              "D2H");
  });
}

int xbs_nonlinear_update(const double* g, const double* dg, int64_t n, double v, double g_min, double g_max,
                         double* out) {
  return guard_conv([&] {
    if (n < 0 || (n > 0 && (!g || !dg || !out))) fail_conv(XBS_INVALID_ARGUMENT, "nonlinear_update: bad buffers");
    xbs::Scratch sc;
    int* flag = sc.get<int>(1);
    ck_cuda(cudaMemset(flag, 0, sizeof(int)), "memset");
    if (n > 0) {
      double* a = sc.get<double>(size_t(n));
      double* b = sc.get<double>(size_t(n));
      double* o = sc.get<double>(size_t(n));
      ck_cuda(cudaMemcpy(a, g, size_t(n) * 8, cudaMemcpyHostToDevice), "H2D");
      ck_cuda(cudaMemcpy(b, dg, size_t(n) * 8, cudaMemcpyHostToDevice), "H2D");
      xbs::k_nonlinear<<<xbs::blocks(n), 256>>>(a, b, n, v, g_min, g_max, o, flag);
      ck_cuda(cudaGetLastError(), "kernel launch");
      ck_cuda(cudaMemcpy(out, o, size_t(n) * 8, cudaMemcpyDeviceToHost), "D2H");
    }
    int err = 0;
    ck_cuda(cudaMemcpy(&err, flag, sizeof(int), cudaMemcpyDeviceToHost), "D2H flag");
    if (err) fail_conv(XBS_INVALID_ARGUMENT, "nonlinear_update: g outside device range");
  });
}

int xbs_write_noise(const double* dg, int64_t n, double gamma, double g_min, double g_max, const uint64_t* keys,
                    const uint64_t* counters, double* out, int32_t* drew) {
  return guard_conv([&] {
    if (n < 0 || (n > 0 && (!dg || !keys || !counters || !out)))
      fail_conv(XBS_INVALID_ARGUMENT, "write_noise: bad buffers");
    if (n == 0) return;
    xbs::Scratch sc;
    double* a = sc.get<double>(size_t(n));
    uint64_t* k = sc.get<uint64_t>(size_t(n));
    uint64_t* c = sc.get<uint64_t>(size_t(n));
    double* o = sc.get<double>(size_t(n));
    int32_t* d = drew ? sc.get<int32_t>(size_t(n)) : nullptr;
    ck_cuda(cudaMemcpy(a, dg, size_t(n) * 8, cudaMemcpyHostToDevice), "H2D");
    ck_cuda(cudaMemcpy(k, keys, size_t(n) * 8, cudaMemcpyHostToDevice), "H2D");
    ck_cuda(cudaMemcpy(c, counters, size_t(n) * 8, cudaMemcpyHostToDevice), "H2D");
    xbs::k_write_noise<<<xbs::blocks(n), 256>>>(a, n, gamma, g_max - g_min, k, c, o, d);
    ck_cuda(cudaGetLastError(), "kernel launch");
    ck_cuda(cudaMemcpy(out, o, size_t(n) * 8, cudaMemcpyDeviceToHost), "D2H");
    if (drew) ck_cuda(cudaMemcpy(drew, d, size_t(n) * 4, cudaMemcpyDeviceToHost), "D2H");
  });
}

int xbs_reconstruct_output(const double* codes_pos, const double* codes_neg, int32_t slices, int64_t n,
                           int32_t device_bits, double scale, double* out) {
  return guard_conv([&] {
    if (slices < 0 || n < 0 || device_bits < 1 || device_bits > 62 ||
        (slices * n > 0 && (!codes_pos || !codes_neg)) || (n > 0 && !out))
      fail_conv(XBS_INVALID_ARGUMENT, "reconstruct_output: bad arguments");
    if (n == 0) return;
    xbs::Scratch sc;
    double* p = sc.get<double>(size_t(slices) * n);
    double* q = sc.get<double>(size_t(slices) * n);
    double* o = sc.get<double>(size_t(n));
    if (slices > 0) {
      ck_cuda(cudaMemcpy(p, codes_pos, size_t(slices) * n * 8, cudaMemcpyHostToDevice), "H2D");
      ck_cuda(cudaMemcpy(q, codes_neg, size_t(slices) * n * 8, cudaMemcpyHostToDevice), "H2D");
    }
    xbs::k_reconstruct<<<xbs::blocks(n), 256>>>(p, q, slices, n, double(uint64_t{1} << device_bits), scale, o);
    ck_cuda(cudaGetLastError(), "kernel launch");
    ck_cuda(cudaMemcpy(out, o, size_t(n) * 8, cudaMemcpyDeviceToHost), "D2H");
  });
}

}  // extern "C"
