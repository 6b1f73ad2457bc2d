"""ctypes binding of the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product.
The options POD is the product's xbs_layer_options layout (same fields, same
order), filled from the same CrossbarLayerOptions dataclass.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")

_D = ctypes.POINTER(ctypes.c_double)
_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
        L = _lib
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_core_create.argtypes = [ctypes.c_void_p, ctypes.c_int, _D, ctypes.c_long, ctypes.c_long,
                                      ctypes.POINTER(ctypes.c_void_p)]
        L.orc_core_create_tiles.argtypes = [ctypes.c_void_p, ctypes.c_int, _D, ctypes.c_long, ctypes.c_long,
                                            ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        L.orc_core_destroy.argtypes = [ctypes.c_void_p]
        L.orc_core_forward.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_long, ctypes.c_int, _D]
        L.orc_core_forward_tiles.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_long, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int), ctypes.c_int, _D]
        L.orc_core_backward.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_long, ctypes.c_double, _D]
        L.orc_core_backward_tiles.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_long, ctypes.c_double,
                                              ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int, _D]
        L.orc_core_apply_updates.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        for n in ("orc_core_gradient", "orc_core_implied_weights", "orc_core_set_gradient"):
            getattr(L, n).argtypes = [ctypes.c_void_p, _D]
        L.orc_core_nonideal.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.orc_core_set_nonideal.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.orc_core_master.argtypes = [ctypes.c_void_p, ctypes.c_int, _D]
        L.orc_core_set_master.argtypes = [ctypes.c_void_p, ctypes.c_int, _D]
        L.orc_core_regenerate.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.c_int]
        L.orc_core_geometry.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_long)]
        L.orc_core_stats.argtypes = [ctypes.c_void_p, _D]
        L.orc_core_record_codes.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc_core_last_codes.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint16), ctypes.c_long]
        L.orc_core_last_codes.restype = ctypes.c_long
        L.orc_rng_draws.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_long, ctypes.POINTER(ctypes.c_uint64)]
        L.orc_rng_gaussian.argtypes = [ctypes.c_uint64] * 4
        L.orc_rng_gaussian.restype = ctypes.c_double
        L.orc_snap_exponent.argtypes = [ctypes.c_double]
        L.orc_adc_quantize.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_uint64)]
        L.orc_aam_convert.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_double] * 4 + [_D, _D]
        L.orc_calibrate.argtypes = [_D, ctypes.c_long, ctypes.c_double]
        L.orc_calibrate.restype = ctypes.c_double
        L.orc_conv2d_create.argtypes = [ctypes.c_void_p, ctypes.c_int, _D, ctypes.c_long, ctypes.c_long] + \
            [ctypes.c_int] * 5 + [ctypes.POINTER(ctypes.c_void_p)]
        L.orc_conv2d_destroy.argtypes = [ctypes.c_void_p]
        L.orc_conv2d_forward.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, _D, ctypes.POINTER(ctypes.c_int)]
        L.orc_conv2d_backward.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_long, _D]
        L.orc_conv2d_apply_updates.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.orc_softmax_ce.argtypes = [_D, ctypes.c_long, ctypes.c_long, ctypes.POINTER(ctypes.c_int), ctypes.c_long, _D, _D]
        L.orc_relu.argtypes = [_D, ctypes.c_long, ctypes.c_long, _D, _D, _D]
        L.orc_maxpool2d.argtypes = [_D, ctypes.c_long] + [ctypes.c_int] * 5 + [_D, _D, _D]
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(_D)


class OracleCore:
    """CPU restatement of CrossbarCore; snapped=True is the GPU's exactness contract."""

    def __init__(self, W0, opt, snapped: bool = True, tiles=None):
        """tiles: convert only these tiles (tr * grid_cols + tc) -- sampled
        parity on layers too large to convert whole; forward_tiles /
        backward_tiles must then stay inside them."""
        W = _f(W0)
        self._copt = opt.to_c()
        h = ctypes.c_void_p()
        if tiles is None:
            _check(lib().orc_core_create(ctypes.byref(self._copt), int(snapped), _p(W), W.shape[0], W.shape[1],
                                         ctypes.byref(h)))
        else:
            arr = (ctypes.c_int * max(1, len(tiles)))(*tiles)
            _check(lib().orc_core_create_tiles(ctypes.byref(self._copt), int(snapped), _p(W), W.shape[0], W.shape[1],
                                               arr, len(tiles), ctypes.byref(h)))
        self._h = h
        self.K, self.N = W.shape
        self.opt = opt
        g = (ctypes.c_long * 8)()
        _check(lib().orc_core_geometry(self._h, g))
        (self.rows, self.cols, self.grid_rows, self.grid_cols, self.padded_rows, self.padded_cols, self.slices,
         self.snap_e) = list(g)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_core_destroy(self._h)
            self._h = None

    def forward(self, x, training=False):
        x = _f(x)
        y = np.zeros((x.shape[0], self.N), order="F")
        _check(lib().orc_core_forward(self._h, _p(x), x.shape[0], x.shape[1], int(training), _p(y)))
        return y

    def forward_tiles(self, x, tcs, training=False):
        x = _f(x)
        y = np.zeros((x.shape[0], self.N), order="F")
        arr = (ctypes.c_int * len(tcs))(*tcs)
        _check(lib().orc_core_forward_tiles(self._h, _p(x), x.shape[0], x.shape[1], int(training), arr, len(tcs),
                                            _p(y)))
        return y

    def backward(self, dy, grad_divisor=1.0):
        dy = _f(dy)
        dx = np.zeros((dy.shape[0], self.K), order="F")
        _check(lib().orc_core_backward(self._h, _p(dy), dy.shape[0], dy.shape[1], grad_divisor, _p(dx)))
        return dx

    def backward_tiles(self, dy, trs, grad_divisor=1.0, compute_dw=False):
        dy = _f(dy)
        dx = np.zeros((dy.shape[0], self.K), order="F")
        arr = (ctypes.c_int * len(trs))(*trs)
        _check(lib().orc_core_backward_tiles(self._h, _p(dy), dy.shape[0], dy.shape[1], grad_divisor, arr, len(trs),
                                             int(compute_dw), _p(dx)))
        return dx

    def apply_updates(self, iteration):
        _check(lib().orc_core_apply_updates(self._h, iteration))

    def gradient(self):
        g = np.zeros((self.K, self.N), order="F")
        _check(lib().orc_core_gradient(self._h, _p(g)))
        return g

    def set_gradient(self, dW):
        dW = _f(dW)
        _check(lib().orc_core_set_gradient(self._h, _p(dW)))

    def implied_weights(self):
        g = np.zeros((self.K, self.N), order="F")
        _check(lib().orc_core_implied_weights(self._h, _p(g)))
        return g

    def nonideal(self, s, p, t):
        g = np.zeros((self.opt.map.tile_rows, self.opt.map.tile_cols), order="F")
        _check(lib().orc_core_nonideal(self._h, s, int(p), t, _p(g)))
        return g

    def set_nonideal(self, s, p, t, g):
        g = _f(g)
        _check(lib().orc_core_set_nonideal(self._h, s, int(p), t, _p(g)))

    def master(self, s):
        u = np.zeros((self.padded_rows, self.padded_cols), order="F")
        _check(lib().orc_core_master(self._h, s, _p(u)))
        return u

    def set_master(self, s, u):
        u = _f(u)
        _check(lib().orc_core_set_master(self._h, s, _p(u)))

    def regenerate(self, tiles=()):
        arr = (ctypes.c_int * max(1, len(tiles)))(*tiles)
        _check(lib().orc_core_regenerate(self._h, arr, len(tiles)))

    def stats(self):
        s = (ctypes.c_double * 7)()
        _check(lib().orc_core_stats(self._h, s))
        keys = ("layer_scale", "wmax_seen", "dwmax_seen", "fwd_i_fs", "bwd_i_fs", "refresh_count", "level_step")
        return dict(zip(keys, list(s)))

    def record_codes(self, on=True):
        lib().orc_core_record_codes(self._h, int(on))

    def last_codes(self):
        n = lib().orc_core_last_codes(self._h, None, 0)
        out = np.zeros(n, dtype=np.uint16)
        lib().orc_core_last_codes(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)), n)
        return out


class OracleConv2d:
    """CrossbarConv2d restated (layers.cpp:415-505); x: batch x (c*h*w)."""

    def __init__(self, W0, in_c, out_c, kernel, stride, padding, opt, snapped: bool = True):
        W = _f(W0)
        self._copt = opt.to_c()
        h = ctypes.c_void_p()
        _check(lib().orc_conv2d_create(ctypes.byref(self._copt), int(snapped), _p(W), W.shape[0], W.shape[1], in_c,
                                       out_c, kernel, stride, padding, ctypes.byref(h)))
        self._h = h
        self._feat_in = None

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_conv2d_destroy(self._h)
            self._h = None

    def forward(self, x, c, h, w, training=False):
        x = _f(x)
        dims = (ctypes.c_int * 3)()
        _check(lib().orc_conv2d_forward(self._h, _p(x), x.shape[0], c, h, w, int(training), None, dims))
        y = np.zeros((x.shape[0], dims[0] * dims[1] * dims[2]), order="F")
        _check(lib().orc_conv2d_forward(self._h, _p(x), x.shape[0], c, h, w, int(training), _p(y), dims))
        self._feat_in = c * h * w
        return y, tuple(dims)

    def backward(self, dy):
        dy = _f(dy)
        dx = np.zeros((dy.shape[0], self._feat_in), order="F")
        _check(lib().orc_conv2d_backward(self._h, _p(dy), dy.shape[0], dy.shape[1], _p(dx)))
        return dx

    def apply_updates(self, it):
        _check(lib().orc_conv2d_apply_updates(self._h, it))


def rng_draws(seed, a, b, c, n):
    out = (ctypes.c_uint64 * n)()
    lib().orc_rng_draws(seed, a, b, c, n, out)
    return np.array(list(out), dtype=np.uint64)


def rng_gaussian(seed, a, b=0, c=0):
    return lib().orc_rng_gaussian(seed, a, b, c)


def calibrate(samples, pct=0.999):
    s = np.ascontiguousarray(samples, dtype=np.float64)
    return lib().orc_calibrate(_p(s), s.size, pct)


# ---------------------------------------------------------------- step glue
def softmax_cross_entropy(logits, labels):
    """train.cpp:11-33 restated in the oracle: (mean loss, dlogits)."""
    lg = _f(logits)
    n, c = lg.shape
    lab = (ctypes.c_int * max(1, len(labels)))(*[int(v) for v in labels])
    d = np.zeros((n, c), order="F")
    loss = ctypes.c_double()
    _check(lib().orc_softmax_ce(_p(lg), n, c, lab, len(labels), _p(d), ctypes.byref(loss)))
    return loss.value, np.ascontiguousarray(d)


def relu(x, dy):
    """layers.cpp:510-522: forward of x and backward of dy through its mask."""
    xf, dyf = _f(x), _f(dy)
    y, dx = np.zeros(xf.shape, order="F"), np.zeros(dyf.shape, order="F")
    _check(lib().orc_relu(_p(xf), xf.shape[0], xf.shape[1], _p(dyf), _p(y), _p(dx)))
    return np.ascontiguousarray(y), np.ascontiguousarray(dx)


def maxpool2d(x, c, h, w, kernel, stride, dy):
    """layers.cpp:524-575: (y, dx) of a MaxPool2d over (c, h, w) rows."""
    xf, dyf = _f(x), _f(dy)
    oh, ow = (h - kernel) // stride + 1, (w - kernel) // stride + 1
    y = np.zeros((xf.shape[0], c * oh * ow), order="F")
    dx = np.zeros(xf.shape, order="F")
    _check(lib().orc_maxpool2d(_p(xf), xf.shape[0], c, h, w, kernel, stride, _p(dyf), _p(y), _p(dx)))
    return np.ascontiguousarray(y), np.ascontiguousarray(dx)
