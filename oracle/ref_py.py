"""TEST INFRASTRUCTURE ONLY — ctypes access to the reference's OWN core
sources compiled in place (oracle/ref/Makefile -> oracle/_ref/libxbsref.so,
Eigen API supplied by oracle/eigen_shim).  Used by tests/test_ref_pin_cpu.py
to pin the restated oracle (oracle_py, literal mode) to the reference code.
Absent where /root/reference is not (the GPU box): callers skip."""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libxbsref.so")
_D = ctypes.POINTER(ctypes.c_double)
_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_core_create.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_long, ctypes.POINTER(ctypes.c_void_p)]
        L.ref_core_destroy.argtypes = [ctypes.c_void_p]
        L.ref_core_forward.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_long, ctypes.c_int, _D]
        L.ref_core_backward.argtypes = [ctypes.c_void_p, _D, ctypes.c_long, ctypes.c_long, ctypes.c_double, _D]
        L.ref_core_apply_updates.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.ref_core_gradient.argtypes = [ctypes.c_void_p, _D]
        L.ref_core_nonideal.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.ref_core_master.argtypes = [ctypes.c_void_p, ctypes.c_int, _D]
        L.ref_core_stats.argtypes = [ctypes.c_void_p, _D]
        L.ref_softmax_ce.argtypes = [_D, ctypes.c_long, ctypes.c_long, ctypes.POINTER(ctypes.c_int), ctypes.c_long,
                                     _D, _D]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(_D)


class RefCore:
    """xbarsim::nn::CrossbarCore of the reference sources."""

    def __init__(self, W0, opt, tile_rows_padded, tile_cols_padded, slices, tiles):
        W = _f(W0)
        self._copt = opt.to_c()  # the same POD layout as the oracle's options
        h = ctypes.c_void_p()
        _check(lib().ref_core_create(ctypes.byref(self._copt), _p(W), W.shape[0], W.shape[1], ctypes.byref(h)))
        self._h = h
        self.K, self.N = W.shape
        self.tr, self.tc, self.S, self.T = tile_rows_padded, tile_cols_padded, slices, tiles

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_core_destroy(self._h)
            self._h = None

    def forward(self, x, training=False):
        x = _f(x)
        y = np.zeros((x.shape[0], self.N), order="F")
        _check(lib().ref_core_forward(self._h, _p(x), x.shape[0], x.shape[1], int(training), _p(y)))
        return np.ascontiguousarray(y)

    def backward(self, dy, grad_divisor=1.0):
        dy = _f(dy)
        dx = np.zeros((dy.shape[0], self.K), order="F")
        _check(lib().ref_core_backward(self._h, _p(dy), dy.shape[0], dy.shape[1], grad_divisor, _p(dx)))
        return np.ascontiguousarray(dx)

    def apply_updates(self, it):
        _check(lib().ref_core_apply_updates(self._h, it))

    def gradient(self):
        g = np.zeros((self.K, self.N), order="F")
        _check(lib().ref_core_gradient(self._h, _p(g)))
        return np.ascontiguousarray(g)

    def nonideal(self, s, p, t):
        g = np.zeros((self.tr, self.tc), order="F")
        _check(lib().ref_core_nonideal(self._h, s, p, t, _p(g)))
        return np.ascontiguousarray(g)

    def master(self, s, rows, cols):
        u = np.zeros((rows, cols), order="F")
        _check(lib().ref_core_master(self._h, s, _p(u)))
        return np.ascontiguousarray(u)

    def stats(self):
        out = (ctypes.c_double * 4)()
        _check(lib().ref_core_stats(self._h, out))
        return {"refresh_count": out[0], "weight_abs_max_seen": out[1], "grad_abs_max_seen": out[2],
                "forward_adc_full_scale": out[3]}


def softmax_cross_entropy(logits, labels):
    lg = _f(logits)
    n, c = lg.shape
    lab = (ctypes.c_int * max(1, len(labels)))(*[int(v) for v in labels])
    d = np.zeros((n, c), order="F")
    loss = ctypes.c_double()
    _check(lib().ref_softmax_ce(_p(lg), n, c, lab, len(labels), _p(d), ctypes.byref(loss)))
    return loss.value, np.ascontiguousarray(d)
