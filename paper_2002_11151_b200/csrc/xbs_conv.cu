// CrossbarConv2d (layers.cpp:415-505) on the device: im2col fused into the
// core's input quantisation (the patch matrix is never written), the crossbar
// core, and the inverse layouts.  Tensors follow
// the reference: values are batch x features, column-major (Eigen), features
// ordered (c, y, x); the patch matrix is (batch * oh * ow) x (in_c * k * k)
// with rows (b, oy, ox) and columns (c, ky, kx).
//
// col2im is written as a gather: each input element sums its patch entries
// in increasing (oy, ox) order, which is the order the reference's scatter
// loop adds them in, so dx is bit-identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "xbs_internal.cuh"

struct xbs_conv2d {
  xbs_core* core = nullptr;
  int in_c = 0, out_c = 0, k = 0, stride = 1, pad = 0;
  int in_h = 0, in_w = 0, out_h = 0, out_w = 0;
  int64_t batch = 0;
  bool have_forward = false;
  double *d_x = nullptr, *d_patch = nullptr, *d_flat = nullptr, *d_y = nullptr;
  int64_t cap_x = 0, cap_patch = 0, cap_flat = 0, cap_y = 0;
};

namespace xbs {
namespace {

// flat (rows x out_c) <-> tensor (batch x out_c*oh*ow), both column-major.
// Thread order follows the flat matrix (r fastest) so its side is coalesced.
template <typename I>  // index type: int when every index fits, else int64_t
__global__ void k_flat_to_tensor(const double* __restrict__ flat, I batch, int out_c, int oh, int ow,
                                 double* __restrict__ y, int to_tensor) {
  const I hw = I(oh) * ow, rows = batch * hw, n = rows * out_c;
  for (I e = I(blockIdx.x) * I(blockDim.x) + I(threadIdx.x); e < n; e += I(gridDim.x) * I(blockDim.x)) {
    const I oc = e / rows, r = e - oc * rows;  // flat element (r, oc), r = (b, oy, ox)
    const I b = r / hw, pos = r - b * hw;
    const I t = (oc * hw + pos) * batch + b;  // tensor element (b, f), f = (oc, oy, ox)
    if (to_tensor) y[t] = flat[e];
    else y[e] = flat[t];  // (here `flat` is the tensor and `y` the flat matrix)
  }
}

// col2im as a gather: each input element sums its patch entries in
// increasing (oy, ox) order -- the reference's scatter order
// (layers.cpp:486-502) -- visiting only the (oy, ox) whose window covers it.
template <typename I>
__global__ void k_col2im(const double* __restrict__ dpatch, I batch, int c_in, int h, int w, int k, int stride,
                         int pad, int oh, int ow, double* __restrict__ dx) {
  const I rows = batch * oh * ow, n = batch * I(c_in) * h * w;
  for (I e = I(blockIdx.x) * I(blockDim.x) + I(threadIdx.x); e < n; e += I(gridDim.x) * I(blockDim.x)) {
    // ix fastest: neighbouring threads read neighbouring patch rows
    const int ix = int(e % w);
    const I e2 = e / w;
    const int iy = int(e2 % h);
    const I e3 = e2 / h;
    const int c = int(e3 % c_in);
    const I b = e3 / c_in;
    const int ny = iy + pad - k + 1, nx = ix + pad - k + 1;
    const int oy0 = ny <= 0 ? 0 : (ny + stride - 1) / stride, oy1 = min(oh - 1, (iy + pad) / stride);
    const int ox0 = nx <= 0 ? 0 : (nx + stride - 1) / stride, ox1 = min(ow - 1, (ix + pad) / stride);
    double acc = 0.0;
    for (int oy = oy0; oy <= oy1; ++oy) {
      const int ky = iy + pad - oy * stride;
      for (int ox = ox0; ox <= ox1; ++ox) {
        const int kx = ix + pad - ox * stride;
        const int64_t r = (int64_t(b) * oh + oy) * ow + ox;
        acc += dpatch[((int64_t(c) * k + ky) * k + kx) * int64_t(rows) + r];
      }
    }
    dx[((int64_t(c) * h + iy) * w + ix) * int64_t(batch) + b] = acc;
  }
}

int blocks_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16))); }

void flat_to_tensor(const double* src, int64_t batch, int out_c, int oh, int ow, double* dst, int to_tensor,
                    cudaStream_t st) {
  const int64_t n = batch * oh * ow * out_c;
  if (n <= 0) return;
  if (n < (int64_t(1) << 31))
    k_flat_to_tensor<int><<<blocks_for(n), 256, 0, st>>>(src, int(batch), out_c, oh, ow, dst, to_tensor);
  else
    k_flat_to_tensor<int64_t><<<blocks_for(n), 256, 0, st>>>(src, batch, out_c, oh, ow, dst, to_tensor);
}

void grow(double*& p, int64_t& cap, int64_t n) {
  if (cap >= n) return;
  cudaFree(p);
  p = nullptr;
  ck_cuda(cudaMalloc(&p, size_t(std::max<int64_t>(n, 1)) * sizeof(double)), "cudaMalloc conv buffer");
  cap = n;
}

}  // namespace
}  // namespace xbs

extern "C" {

int xbs_conv2d_create(const xbs_layer_options* opt, const double* W0, int64_t ldw, int32_t in_c, int32_t out_c,
                      int32_t kernel, int32_t stride, int32_t padding, xbs_conv2d** out) {
  if (!out) return XBS_INVALID_ARGUMENT;
  *out = nullptr;
  xbs_core* core = nullptr;
  // layers.cpp:418-428: the core is built first (its validation comes first), then the geometry
  const int rc = xbs_core_create(opt, W0, int64_t(in_c) * kernel * kernel, out_c, ldw, &core);
  if (rc != XBS_OK) return rc;
  if (stride < 1 || kernel < 1 || padding < 0 || in_c < 1 || out_c < 1) {
    xbs_core_destroy(core);
    return xbs::set_error(XBS_INVALID_ARGUMENT, "CrossbarConv2d: bad geometry");
  }
  auto* c = new xbs_conv2d;
  c->core = core;
  c->in_c = in_c;
  c->out_c = out_c;
  c->k = kernel;
  c->stride = stride;
  c->pad = padding;
  *out = c;
  return XBS_OK;
}

void xbs_conv2d_destroy(xbs_conv2d* c) {
  if (!c) return;
  cudaFree(c->d_x);
  cudaFree(c->d_patch);
  cudaFree(c->d_flat);
  cudaFree(c->d_y);
  xbs_core_destroy(c->core);
  delete c;
}

xbs_core* xbs_conv2d_core(xbs_conv2d* c) { return c ? c->core : nullptr; }

int xbs_conv2d_output_dims(xbs_conv2d* c, int32_t h, int32_t w, int32_t* oh, int32_t* ow) {
  if (!c || !oh || !ow) return xbs::set_error(XBS_INVALID_ARGUMENT, "null argument");
  *oh = (h + 2 * c->pad - c->k) / c->stride + 1;
  *ow = (w + 2 * c->pad - c->k) / c->stride + 1;
  if (*oh < 1 || *ow < 1) return xbs::set_error(XBS_INVALID_ARGUMENT, "CrossbarConv2d: kernel does not fit the input");
  return XBS_OK;
}

int xbs_conv2d_forward_device(xbs_conv2d* c, const double* d_x, int64_t batch, int32_t ch, int32_t h, int32_t w,
                              int32_t training, double* d_y) {
  return xbs::guard_conv([&] {
    if (!c) xbs::fail_conv(XBS_INVALID_ARGUMENT, "null conv");
    if (ch != c->in_c) xbs::fail_conv(XBS_INVALID_ARGUMENT, "CrossbarConv2d: expected (c, h, w) input");
    int oh = 0, ow = 0;
    xbs::check_rc(xbs_conv2d_output_dims(c, h, w, &oh, &ow));
    c->in_h = h;
    c->in_w = w;
    c->out_h = oh;
    c->out_w = ow;
    c->batch = batch;
    cudaStream_t st = static_cast<cudaStream_t>(xbs_core_stream(c->core));
    const int64_t rows = batch * oh * ow;
    xbs::grow(c->d_flat, c->cap_flat, rows * c->out_c);
    // im2col fused into the core's input quantisation: the patch matrix is
    // never written (xbs_kernels.cu k_prep_x<true>)
    const xbs::ConvSrc cs{c->in_c, h, w, c->k, c->stride, c->pad, oh, ow, batch};
    xbs::core_forward_conv(c->core, d_x, cs, training != 0, c->d_flat);
    xbs::flat_to_tensor(c->d_flat, batch, c->out_c, oh, ow, d_y, 1, st);
    c->have_forward = true;
  });
}

int xbs_conv2d_backward_device(xbs_conv2d* c, const double* d_dy, int64_t batch, double* d_dx) {
  return xbs::guard_conv([&] {
    if (!c) xbs::fail_conv(XBS_INVALID_ARGUMENT, "null conv");
    cudaStream_t st = static_cast<cudaStream_t>(xbs_core_stream(c->core));
    if (batch != c->batch && c->have_forward)
      xbs::fail_conv(XBS_INVALID_ARGUMENT, "CrossbarCore::backward: gradient shape mismatch");
    const int64_t rows = c->batch * c->out_h * c->out_w, kk = int64_t(c->in_c) * c->k * c->k;
    xbs::grow(c->d_flat, c->cap_flat, rows * c->out_c);
    xbs::grow(c->d_patch, c->cap_patch, rows * kk);
    xbs::flat_to_tensor(d_dy, c->batch, c->out_c, c->out_h, c->out_w, c->d_flat, 0, st);
    // layers.cpp:483: grad_divisor 1.0
    xbs::check_rc(xbs_core_backward_device(c->core, c->d_flat, rows, 1.0, c->d_patch));
    const int64_t n = c->batch * int64_t(c->in_c) * c->in_h * c->in_w;
    if (n > 0) {
      if (n < (int64_t(1) << 31))
        xbs::k_col2im<int><<<xbs::blocks_for(n), 256, 0, st>>>(c->d_patch, int(c->batch), c->in_c, c->in_h, c->in_w,
                                                               c->k, c->stride, c->pad, c->out_h, c->out_w, d_dx);
      else
        xbs::k_col2im<int64_t><<<xbs::blocks_for(n), 256, 0, st>>>(c->d_patch, c->batch, c->in_c, c->in_h, c->in_w,
                                                                   c->k, c->stride, c->pad, c->out_h, c->out_w, d_dx);
    }
  });
}

int xbs_conv2d_forward(xbs_conv2d* c, const double* x, int64_t batch, int32_t ch, int32_t h, int32_t w, int64_t ldx,
                       int32_t training, double* y, int64_t ldy) {
  return xbs::guard_conv([&] {
    if (!c) xbs::fail_conv(XBS_INVALID_ARGUMENT, "null conv");
    if (ch != c->in_c) xbs::fail_conv(XBS_INVALID_ARGUMENT, "CrossbarConv2d: expected (c, h, w) input");
    int oh = 0, ow = 0;
    xbs::check_rc(xbs_conv2d_output_dims(c, h, w, &oh, &ow));
    const int64_t fin = int64_t(ch) * h * w, fout = int64_t(c->out_c) * oh * ow;
    if (batch > 0 && (!x || !y || ldx < batch || ldy < batch))
      xbs::fail_conv(XBS_INVALID_ARGUMENT, "CrossbarConv2d::forward: bad buffers");
    cudaStream_t st = static_cast<cudaStream_t>(xbs_core_stream(c->core));
    xbs::grow(c->d_x, c->cap_x, batch * fin);
    xbs::grow(c->d_y, c->cap_y, batch * fout);
    if (batch > 0)
      xbs::ck_cuda(cudaMemcpy2DAsync(c->d_x, size_t(batch) * 8, x, size_t(ldx) * 8, size_t(batch) * 8, size_t(fin),
                                     cudaMemcpyHostToDevice, st),
                   "H2D x");
    xbs::check_rc(xbs_conv2d_forward_device(c, c->d_x, batch, ch, h, w, training, c->d_y));
    if (batch > 0)
      xbs::ck_cuda(cudaMemcpy2DAsync(y, size_t(ldy) * 8, c->d_y, size_t(batch) * 8, size_t(batch) * 8, size_t(fout),
                                     cudaMemcpyDeviceToHost, st),
                   "D2H y");
    xbs::check_rc(xbs_core_synchronize(c->core));
  });
}

int xbs_conv2d_backward(xbs_conv2d* c, const double* dy, int64_t batch, int64_t lddy, double* dx, int64_t lddx) {
  return xbs::guard_conv([&] {
    if (!c) xbs::fail_conv(XBS_INVALID_ARGUMENT, "null conv");
    if (!c->have_forward) xbs::fail_conv(XBS_STATE_ERROR, "CrossbarCore::backward: no cached forward activations");
    if (batch != c->batch) xbs::fail_conv(XBS_INVALID_ARGUMENT, "CrossbarCore::backward: gradient shape mismatch");
    const int64_t fin = int64_t(c->in_c) * c->in_h * c->in_w, fout = int64_t(c->out_c) * c->out_h * c->out_w;
    if (batch > 0 && (!dy || !dx || lddy < batch || lddx < batch))
      xbs::fail_conv(XBS_INVALID_ARGUMENT, "CrossbarConv2d::backward: bad buffers");
    cudaStream_t st = static_cast<cudaStream_t>(xbs_core_stream(c->core));
    xbs::grow(c->d_y, c->cap_y, batch * fout);
    xbs::grow(c->d_x, c->cap_x, batch * fin);
    if (batch > 0)
      xbs::ck_cuda(cudaMemcpy2DAsync(c->d_y, size_t(batch) * 8, dy, size_t(lddy) * 8, size_t(batch) * 8,
                                     size_t(fout), cudaMemcpyHostToDevice, st),
                   "H2D dy");
    xbs::check_rc(xbs_conv2d_backward_device(c, c->d_y, batch, c->d_x));
    if (batch > 0)
      xbs::ck_cuda(cudaMemcpy2DAsync(dx, size_t(lddx) * 8, c->d_x, size_t(batch) * 8, size_t(batch) * 8, size_t(fin),
                                     cudaMemcpyDeviceToHost, st),
                   "D2H dx");
    xbs::check_rc(xbs_core_synchronize(c->core));
  });
}

int xbs_conv2d_apply_updates(xbs_conv2d* c, uint64_t iteration) {
  if (!c) return xbs::set_error(XBS_INVALID_ARGUMENT, "null conv");
  c->have_forward = false;
  return xbs_core_apply_updates(c->core, iteration);
}

}  // extern "C"
