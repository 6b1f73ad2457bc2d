"""Python mirror of the reference's crossbar-layer operator API over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/xbarsim/layers.hpp:19-152 (CrossbarLayerOptions,
CrossbarCore, Layer, CrossbarLinear) and the spec structs they aggregate
(mapping.hpp:14-25, crossbar.hpp:17-40, converters.hpp:14-45, update.hpp:13-23).
Matrices are numpy float64 arrays, logically (rows, cols) like Eigen::MatrixXd.

Every compute call goes through ``libxbarsim_b200.so`` (include/xbarsim_b200.h):
there is no CPU fallback; importing this module on a machine without the built
library, or calling it without a GPU, raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import enum
import os
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XBS_LIB_PATH") or os.path.join(_HERE, "_lib", "libxbarsim_b200.so")


# ----------------------------------------------------------------- errors.hpp
class XbarsimError(RuntimeError):
    pass


class StateError(XbarsimError):
    """errors.hpp:38-42"""


class ConfigError(XbarsimError):
    """errors.hpp:44-47 (also raised for configurations outside this path)"""


class ConvergenceError(XbarsimError):
    pass


class StaleCacheError(XbarsimError):
    pass


class DegenerateCircuitError(XbarsimError):
    pass


class UnsupportedConfigError(ConfigError):
    """A valid reference configuration this B200 path does not evaluate."""


class CudaError(StateError):
    pass


_STATUS = {
    1: ValueError,  # std::invalid_argument
    2: StateError,
    3: ConfigError,
    4: ConvergenceError,
    5: StaleCacheError,
    6: DegenerateCircuitError,
    7: UnsupportedConfigError,
    8: CudaError,
    9: XbarsimError,
}


class EngineKind(enum.IntEnum):
    """engine.hpp:15-21"""

    ideal = 0
    oracle = 1
    fcm = 2
    aam = 3
    interp_fcm = 4


class Polarity(enum.IntEnum):
    pos = 0
    neg = 1


# ------------------------------------------------------------- option specs
@dataclasses.dataclass
class MappingSpec:
    weight_bits: int = 8
    device_bits: int = 2
    tile_rows: int = 64
    tile_cols: int = 64
    variation_sigma: float = 0.0
    seed: int = 0
    w_max: float = 0.0

    def num_slices(self) -> int:
        return self.weight_bits // self.device_bits


@dataclasses.dataclass
class CrossbarConfig:
    rows: int = 64
    cols: int = 64
    r_row: float = 1.0
    r_col: float = 4.6
    r_source: float = 0.0
    r_sense: float = 0.0
    g_min: float = 1e-6
    g_max: float = 1e-5
    v_fs: float = 1.0


@dataclasses.dataclass
class DacSpec:
    bits: int = 1
    v_fs: float = 1.0
    transfer: List[float] = dataclasses.field(default_factory=list)
    stream_bits: int = 1


@dataclasses.dataclass
class AdcSpec:
    bits: int = 8
    i_fs: float = 0.0
    transfer: List[float] = dataclasses.field(default_factory=list)
    clip_percentile: float = 0.999


@dataclasses.dataclass
class UpdateSpec:
    v: float = 0.0
    gamma: float = 0.0
    lr: float = 0.01
    seed: int = 0
    layer_scale: float = 0.0


@dataclasses.dataclass
class CrossbarLayerOptions:
    map: MappingSpec = dataclasses.field(default_factory=MappingSpec)
    crossbar: CrossbarConfig = dataclasses.field(default_factory=CrossbarConfig)
    dac: DacSpec = dataclasses.field(default_factory=DacSpec)
    adc: AdcSpec = dataclasses.field(default_factory=AdcSpec)
    update: UpdateSpec = dataclasses.field(default_factory=UpdateSpec)
    engine: EngineKind = EngineKind.fcm
    interp_base: EngineKind = EngineKind.fcm
    interp_interval: int = 10
    fcm_tol: float = 1e-6
    fcm_max_iter: int = 1000
    act_bits: int = 8
    act_full_scale: float = 1.0
    error_bits: int = 8
    adc_cal_batches: int = 20
    threads: int = 1

    def validate(self) -> None:
        """layers.cpp:17-47 (through the C ABI: same checks and exception classes)."""
        o = self.to_c()
        _check(load_library().xbs_options_validate(ctypes.byref(o)))

    def to_c(self) -> "CLayerOptions":
        """Flat POD (include/xbarsim_b200.h xbs_layer_options)."""
        o = CLayerOptions()
        m, x, d, a, u = self.map, self.crossbar, self.dac, self.adc, self.update
        o.weight_bits, o.device_bits, o.tile_rows, o.tile_cols = m.weight_bits, m.device_bits, m.tile_rows, m.tile_cols
        o.variation_sigma, o.variation_seed, o.w_max = m.variation_sigma, m.seed, m.w_max
        o.xbar_rows, o.xbar_cols = x.rows, x.cols
        o.r_row, o.r_col, o.r_source, o.r_sense = x.r_row, x.r_col, x.r_source, x.r_sense
        o.g_min, o.g_max, o.v_fs = x.g_min, x.g_max, x.v_fs
        o.dac_bits, o.dac_stream_bits, o.dac_v_fs = d.bits, d.stream_bits, d.v_fs
        o._keep = []
        if d.transfer:
            arr = (ctypes.c_double * len(d.transfer))(*d.transfer)
            o._keep.append(arr)
            o.dac_transfer, o.dac_transfer_len = ctypes.cast(arr, ctypes.POINTER(ctypes.c_double)), len(d.transfer)
        o.adc_bits, o.adc_i_fs, o.adc_clip_percentile = a.bits, a.i_fs, a.clip_percentile
        if a.transfer:
            arr = (ctypes.c_double * len(a.transfer))(*a.transfer)
            o._keep.append(arr)
            o.adc_transfer, o.adc_transfer_len = ctypes.cast(arr, ctypes.POINTER(ctypes.c_double)), len(a.transfer)
        o.upd_v, o.upd_gamma, o.upd_lr, o.upd_seed, o.upd_layer_scale = u.v, u.gamma, u.lr, u.seed, u.layer_scale
        o.engine, o.interp_base, o.interp_interval = int(self.engine), int(self.interp_base), self.interp_interval
        o.fcm_tol, o.fcm_max_iter = self.fcm_tol, self.fcm_max_iter
        o.act_bits, o.act_full_scale, o.error_bits = self.act_bits, self.act_full_scale, self.error_bits
        o.adc_cal_batches, o.threads = self.adc_cal_batches, self.threads
        return o


class CLayerOptions(ctypes.Structure):
    _fields_ = [
        ("weight_bits", ctypes.c_int32), ("device_bits", ctypes.c_int32),
        ("tile_rows", ctypes.c_int32), ("tile_cols", ctypes.c_int32),
        ("variation_sigma", ctypes.c_double), ("variation_seed", ctypes.c_uint64), ("w_max", ctypes.c_double),
        ("xbar_rows", ctypes.c_int32), ("xbar_cols", ctypes.c_int32),
        ("r_row", ctypes.c_double), ("r_col", ctypes.c_double), ("r_source", ctypes.c_double),
        ("r_sense", ctypes.c_double), ("g_min", ctypes.c_double), ("g_max", ctypes.c_double),
        ("v_fs", ctypes.c_double),
        ("dac_bits", ctypes.c_int32), ("dac_stream_bits", ctypes.c_int32), ("dac_v_fs", ctypes.c_double),
        ("dac_transfer", ctypes.POINTER(ctypes.c_double)), ("dac_transfer_len", ctypes.c_int32),
        ("adc_bits", ctypes.c_int32), ("adc_i_fs", ctypes.c_double),
        ("adc_transfer", ctypes.POINTER(ctypes.c_double)), ("adc_transfer_len", ctypes.c_int32),
        ("adc_clip_percentile", ctypes.c_double),
        ("upd_v", ctypes.c_double), ("upd_gamma", ctypes.c_double), ("upd_lr", ctypes.c_double),
        ("upd_seed", ctypes.c_uint64), ("upd_layer_scale", ctypes.c_double),
        ("engine", ctypes.c_int32), ("interp_base", ctypes.c_int32), ("interp_interval", ctypes.c_int32),
        ("fcm_tol", ctypes.c_double), ("fcm_max_iter", ctypes.c_int32),
        ("act_bits", ctypes.c_int32), ("act_full_scale", ctypes.c_double),
        ("error_bits", ctypes.c_int32), ("adc_cal_batches", ctypes.c_int32), ("threads", ctypes.c_int32),
    ]


class CoreInfo(ctypes.Structure):
    _fields_ = [
        ("in_features", ctypes.c_int32), ("out_features", ctypes.c_int32),
        ("grid_rows", ctypes.c_int32), ("grid_cols", ctypes.c_int32),
        ("padded_rows", ctypes.c_int32), ("padded_cols", ctypes.c_int32),
        ("num_slices", ctypes.c_int32), ("snap_exponent", ctypes.c_int32),
        ("layer_scale", ctypes.c_double), ("level_step", ctypes.c_double),
        ("refresh_count", ctypes.c_int64), ("conversion_seconds", ctypes.c_double),
        ("weight_abs_max_seen", ctypes.c_double), ("grad_abs_max_seen", ctypes.c_double),
        ("forward_adc_full_scale", ctypes.c_double), ("fully_ideal", ctypes.c_int32), ("kernel", ctypes.c_int32),
        ("tc_fallbacks", ctypes.c_int64),
    ]


class WeightsInfo(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
        ("padded_rows", ctypes.c_int32), ("padded_cols", ctypes.c_int32),
        ("grid_rows", ctypes.c_int32), ("grid_cols", ctypes.c_int32),
        ("num_slices", ctypes.c_int32), ("tile_rows", ctypes.c_int32), ("tile_cols", ctypes.c_int32),
        ("weight_bits", ctypes.c_int32), ("device_bits", ctypes.c_int32),
        ("layer_scale", ctypes.c_double), ("level_step", ctypes.c_double),
        ("variation_sigma", ctypes.c_double), ("variation_seed", ctypes.c_uint64),
        ("g_min", ctypes.c_double), ("g_max", ctypes.c_double),
    ]


class CUpdateSpec(ctypes.Structure):
    _fields_ = [("v", ctypes.c_double), ("gamma", ctypes.c_double), ("lr", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("layer_scale", ctypes.c_double)]


# Exported symbols (name -> (restype, argtypes)); tests check every one of
# them against include/xbarsim_b200.h.
_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64
SYMBOLS = {
    "xbs_abi_version": (ctypes.c_int32, []),
    "xbs_last_error": (ctypes.c_char_p, []),
    "xbs_options_init": (None, [ctypes.POINTER(CLayerOptions)]),
    "xbs_core_create": (ctypes.c_int, [ctypes.POINTER(CLayerOptions), _D, _I64, _I64, _I64, ctypes.POINTER(_P)]),
    "xbs_core_destroy": (None, [_P]),
    "xbs_core_forward": (ctypes.c_int, [_P, _D, _I64, _I64, _I64, ctypes.c_int32, _D, _I64]),
    "xbs_core_backward": (ctypes.c_int, [_P, _D, _I64, _I64, _I64, ctypes.c_double, _D, _I64]),
    "xbs_core_apply_updates": (ctypes.c_int, [_P, ctypes.c_uint64]),
    "xbs_core_forward_device": (ctypes.c_int, [_P, _P, _I64, ctypes.c_int32, _P]),
    "xbs_core_backward_device": (ctypes.c_int, [_P, _P, _I64, ctypes.c_double, _P]),
    "xbs_core_apply_updates_device": (ctypes.c_int, [_P, ctypes.c_uint64]),
    "xbs_core_synchronize": (ctypes.c_int, [_P]),
    "xbs_core_get_info": (ctypes.c_int, [_P, ctypes.POINTER(CoreInfo)]),
    "xbs_core_gradient": (ctypes.c_int, [_P, _D, _I64]),
    "xbs_core_set_gradient": (ctypes.c_int, [_P, _D, _I64]),
    "xbs_core_nonideal": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _D, _I64]),
    "xbs_core_master": (ctypes.c_int, [_P, ctypes.c_int32, _D, _I64]),
    "xbs_core_set_master": (ctypes.c_int, [_P, ctypes.c_int32, _D, _I64]),
    "xbs_core_implied_weights": (ctypes.c_int, [_P, _D, _I64]),
    "xbs_core_adc_counters": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "xbs_core_select_kernel": (ctypes.c_int, [_P, ctypes.c_int32]),
    "xbs_core_stream": (_P, [_P]),
    "xbs_core_set_stream": (ctypes.c_int, [_P, _P]),
    "xbs_conv2d_create": (ctypes.c_int, [_P, _D, _I64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_int32, _P]),
    "xbs_conv2d_destroy": (None, [_P]),
    "xbs_conv2d_core": (_P, [_P]),
    "xbs_conv2d_output_dims": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                              ctypes.POINTER(ctypes.c_int32)]),
    "xbs_conv2d_forward": (ctypes.c_int, [_P, _D, _I64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _I64,
                                          ctypes.c_int32, _D, _I64]),
    "xbs_conv2d_backward": (ctypes.c_int, [_P, _D, _I64, _I64, _D, _I64]),
    "xbs_conv2d_forward_device": (ctypes.c_int, [_P, _P, _I64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.c_int32, _P]),
    "xbs_conv2d_backward_device": (ctypes.c_int, [_P, _P, _I64, _P]),
    "xbs_conv2d_apply_updates": (ctypes.c_int, [_P, ctypes.c_uint64]),
    "xbs_core_profile": (ctypes.c_int, [_P, ctypes.c_int32]),
    "xbs_core_use_graphs": (ctypes.c_int, [_P, ctypes.c_int32]),
    "xbs_core_stage_times": (ctypes.c_int, [_P, _D, ctypes.POINTER(_I64), ctypes.c_int32]),
    "xbs_core_launch_count": (_I64, [_P]),
    "xbs_map_weights": (ctypes.c_int, [ctypes.POINTER(CLayerOptions), _D, _I64, _I64, _I64, ctypes.POINTER(_P)]),
    "xbs_weights_apply_variation": (ctypes.c_int, [_P, ctypes.c_double, ctypes.c_uint64, ctypes.POINTER(_P)]),
    "xbs_core_weights": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "xbs_weights_destroy": (None, [_P]),
    "xbs_weights_get_info": (ctypes.c_int, [_P, ctypes.POINTER(WeightsInfo)]),
    "xbs_weights_master": (ctypes.c_int, [_P, ctypes.c_int32, _D, _I64]),
    "xbs_weights_set_master": (ctypes.c_int, [_P, ctypes.c_int32, _D, _I64]),
    "xbs_weights_master_polarity": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, _D, _I64]),
    "xbs_weights_ideal_working": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, _D, _I64]),
    "xbs_weights_implied": (ctypes.c_int, [_P, _D, _I64]),
    "xbs_apply_update": (ctypes.c_int, [_P, _D, _I64, _I64, _I64, ctypes.POINTER(CUpdateSpec), ctypes.c_uint64]),
    "xbs_scale_gradient": (ctypes.c_int, [_D, _I64, _I64, _I64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                          _D, _I64]),
    "xbs_nonlinear_update": (ctypes.c_int, [_D, _D, _I64, ctypes.c_double, ctypes.c_double, ctypes.c_double, _D]),
    "xbs_write_noise": (ctypes.c_int, [_D, _I64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64), _D,
                                       ctypes.POINTER(ctypes.c_int32)]),
    "xbs_reconstruct_output": (ctypes.c_int, [_D, _D, ctypes.c_int32, _I64, ctypes.c_int32, ctypes.c_double, _D]),
    "xbs_options_validate": (ctypes.c_int, [ctypes.POINTER(CLayerOptions)]),
}

STAGES = ("prep_x", "fwd_vmm", "prep_dy", "dw", "bwd_vmm", "update")

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Loads the C-ABI library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"libxbarsim_b200.so not built ({path}); run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = load_library().xbs_last_error().decode(errors="replace")
        raise _STATUS.get(rc, XbarsimError)(msg)


def _fortran(a: np.ndarray) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


# --------------------------------------------------------------- operators
class CrossbarCore:
    """xbarsim::nn::CrossbarCore (layers.hpp:49-111) on one B200."""

    def __init__(self, W0: np.ndarray, opt: CrossbarLayerOptions):
        lib = load_library()
        W = _fortran(W0)
        if W.ndim != 2:
            raise ValueError("CrossbarCore: W0 must be a matrix")
        self._opt = opt
        self._copt = opt.to_c()
        h = ctypes.c_void_p()
        _check(lib.xbs_core_create(ctypes.byref(self._copt), _ptr(W), W.shape[0], W.shape[1], max(1, W.shape[0]),
                                   ctypes.byref(h)))
        self._h = h
        self._K, self._N = W.shape

    @classmethod
    def _view(cls, handle, K: int, N: int, opt: CrossbarLayerOptions, owner) -> "CrossbarCore":
        """Non-owning view of a core owned by another object (a conv layer)."""
        core = cls.__new__(cls)
        core._opt, core._copt = opt, opt.to_c()
        core._h, core._K, core._N = handle, K, N
        core._owner = owner  # keeps the owner (and the handle) alive
        return core

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(self, "_owner", None) is None:
            _lib.xbs_core_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def forward(self, x: np.ndarray, training: bool, out: Optional[np.ndarray] = None) -> np.ndarray:
        x = _fortran(x)
        if x.ndim != 2:
            raise ValueError("CrossbarCore::forward: feature count mismatch")
        M = x.shape[0]
        y = np.zeros((M, self._N), dtype=np.float64, order="F") if out is None else out
        assert y.shape == (M, self._N) and y.flags.f_contiguous
        _check(load_library().xbs_core_forward(self._h, _ptr(x), M, x.shape[1], max(1, M), int(bool(training)), _ptr(y),
                                               max(1, M)))
        return y

    def backward(self, dy: np.ndarray, grad_divisor: float, out: Optional[np.ndarray] = None) -> np.ndarray:
        dy = _fortran(dy)
        if dy.ndim != 2:
            raise ValueError("CrossbarCore::backward: gradient shape mismatch")
        M = dy.shape[0]
        dx = np.zeros((M, self._K), dtype=np.float64, order="F") if out is None else out
        assert dx.shape == (M, self._K) and dx.flags.f_contiguous
        _check(load_library().xbs_core_backward(self._h, _ptr(dy), M, dy.shape[1], max(1, M), float(grad_divisor),
                                                _ptr(dx),
                                                max(1, M)))
        return dx

    def apply_updates(self, iteration: int) -> None:
        _check(load_library().xbs_core_apply_updates(self._h, int(iteration)))

    def in_features(self) -> int:
        return self._K

    def out_features(self) -> int:
        return self._N

    def info(self) -> CoreInfo:
        inf = CoreInfo()
        _check(load_library().xbs_core_get_info(self._h, ctypes.byref(inf)))
        return inf

    def gradient(self) -> np.ndarray:
        g = np.zeros((self._K, self._N), order="F")
        _check(load_library().xbs_core_gradient(self._h, _ptr(g), self._K))
        return g

    def set_gradient(self, dW: np.ndarray) -> None:
        dW = _fortran(dW)
        _check(load_library().xbs_core_set_gradient(self._h, _ptr(dW), self._K))

    def weights(self) -> "TiledLayerWeights":
        """CrossbarCore::weights() (layers.hpp:59): a view of the core's state."""
        h = ctypes.c_void_p()
        _check(load_library().xbs_core_weights(self._h, ctypes.byref(h)))
        return TiledLayerWeights(h, owner=self)

    def refresh_count(self) -> int:
        return int(self.info().refresh_count)

    def conversion_seconds(self) -> float:
        return float(self.info().conversion_seconds)

    def weight_abs_max_seen(self) -> float:
        return float(self.info().weight_abs_max_seen)

    def grad_abs_max_seen(self) -> float:
        return float(self.info().grad_abs_max_seen)

    def forward_adc_full_scale(self) -> float:
        return float(self.info().forward_adc_full_scale)

    def nonideal(self, slice_: int, p: Polarity, tile: int) -> np.ndarray:
        o = self._opt.map
        g = np.zeros((o.tile_rows, o.tile_cols), order="F")
        _check(load_library().xbs_core_nonideal(self._h, slice_, int(p), tile, _ptr(g), o.tile_rows))
        return g

    def master_diff(self, slice_: int) -> np.ndarray:
        inf = self.info()
        u = np.zeros((inf.padded_rows, inf.padded_cols), order="F")
        _check(load_library().xbs_core_master(self._h, slice_, _ptr(u), inf.padded_rows))
        return u

    def set_master_diff(self, slice_: int, u: np.ndarray) -> None:
        u = _fortran(u)
        _check(load_library().xbs_core_set_master(self._h, slice_, _ptr(u), u.shape[0]))

    def implied_weights(self) -> np.ndarray:
        w = np.zeros((self._K, self._N), order="F")
        _check(load_library().xbs_core_implied_weights(self._h, _ptr(w), self._K))
        return w

    def adc_counters(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(load_library().xbs_core_adc_counters(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def select_kernel(self, kernel: int) -> None:
        _check(load_library().xbs_core_select_kernel(self._h, int(kernel)))

    # device-resident entry points (pointers are CUDA device addresses)
    def forward_device(self, d_x: int, M: int, training: bool, d_y: int) -> None:
        _check(load_library().xbs_core_forward_device(self._h, d_x, M, int(bool(training)), d_y))

    def backward_device(self, d_dy: int, M: int, grad_divisor: float, d_dx: int) -> None:
        _check(load_library().xbs_core_backward_device(self._h, d_dy, M, float(grad_divisor), d_dx))

    def apply_updates_device(self, iteration: int) -> None:
        _check(load_library().xbs_core_apply_updates_device(self._h, int(iteration)))

    def synchronize(self) -> None:
        _check(load_library().xbs_core_synchronize(self._h))

    def stream(self) -> int:
        return load_library().xbs_core_stream(self._h) or 0

    def set_stream(self, stream: int) -> None:
        """Enqueue on a caller-owned cudaStream_t (0: back to a private stream)."""
        _check(load_library().xbs_core_set_stream(self._h, stream or None))

    def profile(self, enable: bool) -> None:
        _check(load_library().xbs_core_profile(self._h, int(bool(enable))))

    def use_graphs(self, enable: bool) -> None:
        """CUDA-graph replay of repeated forward / backward calls (default on)."""
        _check(load_library().xbs_core_use_graphs(self._h, int(bool(enable))))

    def stage_times(self):
        """{stage: (total_ms, count)} accumulated while profiling."""
        ms = (ctypes.c_double * 6)()
        n = (ctypes.c_int64 * 6)()
        _check(load_library().xbs_core_stage_times(self._h, ms, n, 6))
        return {STAGES[i]: (ms[i], n[i]) for i in range(6)}

    def launch_count(self) -> int:
        return int(load_library().xbs_core_launch_count(self._h))




# ------------------------------------------- free functions (mapping / update)
class TiledLayerWeights:
    """mapping::TiledLayerWeights (mapping.hpp:39-90): device-resident master.
    From map_weights / apply_variation (owned) or CrossbarCore.weights()
    (a view of the core's live state)."""

    def __init__(self, handle, owner=None):
        self._h = handle
        self._owner = owner  # the core of a view (kept alive)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.xbs_weights_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self) -> WeightsInfo:
        i = WeightsInfo()
        _check(load_library().xbs_weights_get_info(self._h, ctypes.byref(i)))
        return i

    def rows(self):
        return self.info().rows

    def cols(self):
        return self.info().cols

    def padded_rows(self):
        return self.info().padded_rows

    def padded_cols(self):
        return self.info().padded_cols

    def grid_rows(self):
        return self.info().grid_rows

    def grid_cols(self):
        return self.info().grid_cols

    def num_slices(self):
        return self.info().num_slices

    def layer_scale(self):
        return self.info().layer_scale

    def level_step(self):
        return self.info().level_step

    def variation_sigma(self):
        return self.info().variation_sigma

    def variation_seed(self):
        return self.info().variation_seed

    def master_diff(self, s: int) -> np.ndarray:
        i = self.info()
        u = np.zeros((i.padded_rows, i.padded_cols), order="F")
        _check(load_library().xbs_weights_master(self._h, s, _ptr(u), max(1, i.padded_rows)))
        return u

    def set_master_diff(self, s: int, u: np.ndarray) -> None:
        u = _fortran(u)
        _check(load_library().xbs_weights_set_master(self._h, s, _ptr(u), max(1, u.shape[0])))

    def _padded(self, fn, s, p):
        i = self.info()
        g = np.zeros((i.padded_rows, i.padded_cols), order="F")
        _check(fn(self._h, s, int(p), _ptr(g), max(1, i.padded_rows)))
        return g

    def master_polarity(self, s: int, p: "Polarity") -> np.ndarray:
        return self._padded(load_library().xbs_weights_master_polarity, s, p)

    def ideal_working(self, s: int, p: "Polarity") -> np.ndarray:
        return self._padded(load_library().xbs_weights_ideal_working, s, p)

    def ideal_tile(self, s: int, p: "Polarity", tr: int, tc: int) -> np.ndarray:
        i = self.info()
        if not (0 <= tr < i.grid_rows and 0 <= tc < i.grid_cols):
            raise ValueError("TiledLayerWeights: tile index out of range")
        w = self.ideal_working(s, p)
        return np.asfortranarray(w[tr * i.tile_rows:(tr + 1) * i.tile_rows, tc * i.tile_cols:(tc + 1) * i.tile_cols])

    def implied_weights(self) -> np.ndarray:
        i = self.info()
        w = np.zeros((i.rows, i.cols), order="F")
        _check(load_library().xbs_weights_implied(self._h, _ptr(w), max(1, i.rows)))
        return w


def map_weights(W: np.ndarray, spec: "MappingSpec", cfg: "CrossbarConfig") -> TiledLayerWeights:
    """mapping::map_weights (mapping.cpp:83-131) on the device."""
    o = CrossbarLayerOptions(map=spec, crossbar=cfg).to_c()
    W = _fortran(W)
    if W.ndim != 2:
        raise ValueError("map_weights: W must be a matrix")
    h = ctypes.c_void_p()
    _check(load_library().xbs_map_weights(ctypes.byref(o), _ptr(W), W.shape[0], W.shape[1], max(1, W.shape[0]),
                                          ctypes.byref(h)))
    return TiledLayerWeights(h)


def apply_variation(t: TiledLayerWeights, sigma: float, seed: int) -> TiledLayerWeights:
    """mapping::apply_variation (mapping.cpp:133-140): a copy, new variation."""
    h = ctypes.c_void_p()
    _check(load_library().xbs_weights_apply_variation(t.handle, float(sigma), int(seed), ctypes.byref(h)))
    return TiledLayerWeights(h)


def reconstruct_output(codes_pos, codes_neg, spec: "MappingSpec", scale: float) -> np.ndarray:
    """mapping::reconstruct_output (mapping.cpp:142-160) on the device."""
    S = spec.num_slices()
    if len(codes_pos) != S or len(codes_neg) != S:
        raise ValueError("reconstruct_output: need codes for every slice")
    n = len(codes_pos[0]) if S else 0
    if any(len(c) != n for c in list(codes_pos) + list(codes_neg)):
        raise ValueError("reconstruct_output: inconsistent code lengths")
    pos = np.ascontiguousarray(np.asarray(codes_pos, dtype=np.float64).reshape(S, n))
    neg = np.ascontiguousarray(np.asarray(codes_neg, dtype=np.float64).reshape(S, n))
    out = np.zeros(n)
    _check(load_library().xbs_reconstruct_output(_ptr(pos), _ptr(neg), S, n, spec.device_bits, float(scale),
                                                 _ptr(out)))
    return out


def _cspec(spec: "UpdateSpec") -> CUpdateSpec:
    return CUpdateSpec(spec.v, spec.gamma, spec.lr, spec.seed, spec.layer_scale)


def apply_update(t: TiledLayerWeights, dW: np.ndarray, spec: "UpdateSpec", iteration: int) -> None:
    """update::apply_update (update.cpp:43-88): the master only, on the device."""
    dW = _fortran(dW)
    cs = _cspec(spec)
    _check(load_library().xbs_apply_update(t.handle, _ptr(dW), dW.shape[0], dW.shape[1], max(1, dW.shape[0]),
                                           ctypes.byref(cs), int(iteration)))


def scale_gradient(dW: np.ndarray, spec: "UpdateSpec", cfg: "CrossbarConfig") -> np.ndarray:
    """update::scale_gradient (update.cpp:16-24) on the device."""
    dW = _fortran(dW)
    out = np.zeros_like(dW, order="F")
    _check(load_library().xbs_scale_gradient(_ptr(dW), dW.shape[0], dW.shape[1], max(1, dW.shape[0]),
                                             spec.layer_scale, cfg.g_min, cfg.g_max, _ptr(out), max(1, dW.shape[0])))
    return out


def nonlinear_update(g, dg, spec: "UpdateSpec", cfg: "CrossbarConfig"):
    """update::nonlinear_update (update.cpp:26-33), elementwise on the device."""
    g_, dg_ = np.ascontiguousarray(np.atleast_1d(g), np.float64), np.ascontiguousarray(np.atleast_1d(dg), np.float64)
    g_, dg_ = np.broadcast_arrays(g_, dg_)
    g_, dg_ = np.ascontiguousarray(g_), np.ascontiguousarray(dg_)
    out = np.zeros(g_.size)
    _check(load_library().xbs_nonlinear_update(_ptr(g_), _ptr(dg_), g_.size, spec.v, cfg.g_min, cfg.g_max, _ptr(out)))
    return float(out[0]) if np.ndim(g) == 0 and np.ndim(dg) == 0 else out


_GOLDEN = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def _splitmix(h: int, v: int) -> int:
    h = (h + _GOLDEN + v) & _M64
    h = ((h ^ (h >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    h = ((h ^ (h >> 27)) * 0x94D049BB133111EB) & _M64
    return h ^ (h >> 31)


class CounterRng:
    """rng.hpp:12-48: stateless keyed counter generator (host utility; the
    update kernels draw the same stream on the device)."""

    def __init__(self, seed: int, a: int, b: int = 0, c: int = 0):
        self.key = _splitmix(_splitmix(_splitmix(_splitmix(_GOLDEN ^ (seed & _M64), a & _M64), b & _M64),
                                       c & _M64), 0)
        self.counter = 0

    def _next(self) -> int:
        self.counter += 1
        return _splitmix(self.key, self.counter)

    def uniform(self) -> float:
        return float(self._next() >> 11) * 2.0 ** -53

    def gaussian(self) -> float:
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        return float(np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586476925287 * u2))


def write_noise(dg: float, spec: "UpdateSpec", cfg: "CrossbarConfig", rng: CounterRng) -> float:
    """update::write_noise (update.cpp:35-41) on the device; advances rng by
    the two draws of a Gaussian unless the deviation is 0."""
    d = np.array([float(dg)])
    key, ctr = (ctypes.c_uint64 * 1)(rng.key), (ctypes.c_uint64 * 1)(rng.counter)
    out, drew = np.zeros(1), (ctypes.c_int32 * 1)()
    _check(load_library().xbs_write_noise(_ptr(d), 1, spec.gamma, cfg.g_min, cfg.g_max, key, ctr, _ptr(out), drew))
    if drew[0]:
        rng.counter += 2
    return float(out[0])


@dataclasses.dataclass
class Tensor:
    """tensor.hpp:13-21"""

    values: np.ndarray
    dims: List[int] = dataclasses.field(default_factory=list)
    bits: int = 0
    full_scale: float = 0.0


class Layer:
    """layers.hpp:113-121"""

    def forward(self, x: Tensor, training: bool) -> Tensor:
        raise NotImplementedError

    def backward(self, dy: Tensor) -> Tensor:
        raise NotImplementedError

    def apply_updates(self, iteration: int) -> None:
        pass

    def core(self) -> Optional[CrossbarCore]:
        return None

    def name(self) -> str:
        raise NotImplementedError


class CrossbarLinear(Layer):
    """layers.cpp:393-413"""

    def __init__(self, W0: np.ndarray, opt: CrossbarLayerOptions):
        self._core = CrossbarCore(W0, opt)

    def forward(self, x: Tensor, training: bool) -> Tensor:
        return Tensor(self._core.forward(x.values, training), [self._core.out_features()])

    def backward(self, dy: Tensor) -> Tensor:
        return Tensor(self._core.backward(dy.values, 1.0), [self._core.in_features()])

    def apply_updates(self, iteration: int) -> None:
        self._core.apply_updates(iteration)

    def core(self) -> CrossbarCore:
        return self._core

    def name(self) -> str:
        return "linear"


class CrossbarConv2d(Layer):
    """layers.hpp:136-152, layers.cpp:415-505: im2col lowering onto one core,
    on the device (xbs_conv2d_*).  W0 is (in_c*kernel*kernel) x out_c."""

    def __init__(self, W0: np.ndarray, in_c: int, out_c: int, kernel: int, stride: int, padding: int,
                 opt: CrossbarLayerOptions):
        lib = load_library()
        W = _fortran(W0)
        if W.ndim != 2 or W.shape[0] != in_c * kernel * kernel or W.shape[1] != out_c:
            raise ValueError("CrossbarConv2d: kernel matrix must be (in_c*k*k) x out_c")
        self._copt = opt.to_c()
        h = ctypes.c_void_p()
        _check(lib.xbs_conv2d_create(ctypes.byref(self._copt), _ptr(W), max(1, W.shape[0]), in_c, out_c, kernel, stride,
                                     padding, ctypes.byref(h)))
        self._h = h
        self.in_c, self.out_c = in_c, out_c
        self._core = CrossbarCore._view(lib.xbs_conv2d_core(h), W.shape[0], out_c, opt, self)
        self._in_dims = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.xbs_conv2d_destroy(h)
            self._h = None

    def forward(self, x: Tensor, training: bool, out: Optional[np.ndarray] = None) -> Tensor:
        """out: optional F-ordered (batch x out_c*oh*ow) float64 array to
        write into (e.g. pinned host memory, as CrossbarCore.forward)."""
        if len(x.dims) != 3 or x.dims[0] != self.in_c:
            raise ValueError("CrossbarConv2d: expected (c, h, w) input")
        c, hh, ww = x.dims
        oh, ow = ctypes.c_int32(), ctypes.c_int32()
        _check(load_library().xbs_conv2d_output_dims(self._h, hh, ww, ctypes.byref(oh), ctypes.byref(ow)))
        v = _fortran(x.values)
        b = v.shape[0]
        shape = (b, self.out_c * oh.value * ow.value)
        if out is not None and (out.shape != shape or out.dtype != np.float64 or not out.flags.f_contiguous):
            raise ValueError("CrossbarConv2d.forward: out must be an F-ordered float64 array of shape %s" % (shape,))
        y = out if out is not None else np.zeros(shape, order="F")
        _check(load_library().xbs_conv2d_forward(self._h, _ptr(v), b, c, hh, ww, max(1, b), int(bool(training)), _ptr(y),
                                                 max(1, b)))
        self._in_dims = list(x.dims)
        return Tensor(y, [self.out_c, oh.value, ow.value])

    def backward(self, dy: Tensor, out: Optional[np.ndarray] = None) -> Tensor:
        v = _fortran(dy.values)
        b = v.shape[0]
        c, hh, ww = self._in_dims if self._in_dims else (self.in_c, 0, 0)
        shape = (b, c * hh * ww)
        if out is not None and (out.shape != shape or out.dtype != np.float64 or not out.flags.f_contiguous):
            raise ValueError("CrossbarConv2d.backward: out must be an F-ordered float64 array of shape %s" % (shape,))
        dx = out if out is not None else np.zeros(shape, order="F")
        _check(load_library().xbs_conv2d_backward(self._h, _ptr(v), b, max(1, b), _ptr(dx), max(1, b)))
        return Tensor(dx, [c, hh, ww])

    def apply_updates(self, iteration: int) -> None:
        _check(load_library().xbs_conv2d_apply_updates(self._h, int(iteration)))

    # ---- B200 extensions: device tensors (batch x features column-major),
    # enqueued on the core's stream
    def forward_device(self, d_x: int, batch: int, c: int, h: int, w: int, training: bool, d_y: int) -> None:
        _check(load_library().xbs_conv2d_forward_device(self._h, d_x, batch, c, h, w, int(bool(training)), d_y))

    def backward_device(self, d_dy: int, batch: int, d_dx: int) -> None:
        _check(load_library().xbs_conv2d_backward_device(self._h, d_dy, batch, d_dx))

    def output_dims(self, h: int, w: int):
        oh, ow = ctypes.c_int32(), ctypes.c_int32()
        _check(load_library().xbs_conv2d_output_dims(self._h, h, w, ctypes.byref(oh), ctypes.byref(ow)))
        return oh.value, ow.value

    def core(self) -> CrossbarCore:
        return self._core

    def name(self) -> str:
        return "conv2d"


# ---- host-side step glue of the reference (layers.cpp:507-587, train.cpp:11-33);
# not on the crossbar path, kept with the reference's exact semantics so a
# Network of these layers steps like the reference's.
class ReLU(Layer):
    def forward(self, x: Tensor, training: bool) -> Tensor:
        self._mask = (x.values > 0.0).astype(np.float64)
        return Tensor(x.values * self._mask, list(x.dims), x.bits, x.full_scale)

    def backward(self, dy: Tensor) -> Tensor:
        return Tensor(dy.values * self._mask, list(dy.dims), dy.bits, dy.full_scale)

    def name(self) -> str:
        return "relu"


class MaxPool2d(Layer):
    def __init__(self, kernel: int, stride: int):
        if kernel < 1 or stride < 1:
            raise ValueError("MaxPool2d: bad kernel/stride")
        self.kernel, self.stride = kernel, stride

    def forward(self, x: Tensor, training: bool) -> Tensor:
        if len(x.dims) != 3:
            raise ValueError("MaxPool2d: expected (c, h, w)")
        c, h, w = x.dims
        k, s = self.kernel, self.stride
        oh, ow = (h - k) // s + 1, (w - k) // s + 1
        v = x.values.reshape(x.values.shape[0], c, h, w)
        best = np.full((v.shape[0], c, oh, ow), -np.inf)
        arg = np.zeros((v.shape[0], c, oh, ow), dtype=np.int64)
        for ky in range(k):  # strict '>' keeps the first maximum in (ky, kx) order
            for kx in range(k):
                cand = v[:, :, ky:ky + s * (oh - 1) + 1:s, kx:kx + s * (ow - 1) + 1:s]
                idx = (np.arange(c)[None, :, None, None] * h + (np.arange(oh)[None, None, :, None] * s + ky)) * w + \
                      (np.arange(ow)[None, None, None, :] * s + kx)
                upd = cand > best
                best = np.where(upd, cand, best)
                arg = np.where(upd, idx, arg)
        self._arg, self._in = arg.reshape(arg.shape[0], -1), (list(x.dims), x.values.shape[1])
        return Tensor(best.reshape(best.shape[0], -1), [c, oh, ow])

    def backward(self, dy: Tensor) -> Tensor:
        dims, feat = self._in
        dx = np.zeros((dy.values.shape[0], feat))
        for b in range(dx.shape[0]):
            np.add.at(dx[b], self._arg[b], dy.values[b])
        return Tensor(dx, dims)

    def name(self) -> str:
        return "maxpool2d"


class Flatten(Layer):
    def forward(self, x: Tensor, training: bool) -> Tensor:
        self._dims = list(x.dims)
        return Tensor(x.values, [x.values.shape[1]], x.bits, x.full_scale)

    def backward(self, dy: Tensor) -> Tensor:
        return Tensor(dy.values, list(self._dims), dy.bits, dy.full_scale)

    def name(self) -> str:
        return "flatten"


def softmax_cross_entropy(logits: np.ndarray, labels) -> "tuple[float, np.ndarray]":
    """train.cpp:11-33: mean loss and dlogits (same expression order)."""
    n, _ = logits.shape
    if len(labels) != n:
        raise ValueError("softmax_cross_entropy: label count mismatch")
    d = np.zeros_like(logits)
    total = 0.0
    for i in range(n):
        row = logits[i]
        m = row.max()
        z = 0.0
        for v in row:
            z += np.exp(v - m)
        y = int(labels[i])
        total += -(row[y] - m - np.log(z))
        for j, v in enumerate(row):
            d[i, j] = (np.exp(v - m) / z - (1.0 if j == y else 0.0)) / float(n)
    return total / float(n), d
