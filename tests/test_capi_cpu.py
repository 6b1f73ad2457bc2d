"""C-ABI checks that need no GPU: the library loads, exports exactly what
include/xbarsim_b200.h declares, fills the reference defaults, and validates
options with the reference's error classes before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

from helpers import ROOT, aam_options, xb


@pytest.fixture(scope="module")
def lib():
    return xb.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "xbarsim_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(xbs_[a-z_0-9]+)\s*\(", src))


def test_header_and_library_agree(lib):
    decl = declared_symbols()
    assert decl == set(xb.SYMBOLS), decl ^ set(xb.SYMBOLS)
    for name in decl:
        assert hasattr(lib, name), name


def test_abi_version(lib):
    assert lib.xbs_abi_version() == 3


def test_options_init_matches_reference_defaults(lib):
    o = xb.CLayerOptions()
    lib.xbs_options_init(ctypes.byref(o))
    py = xb.CrossbarLayerOptions().to_c()
    for name, _ in xb.CLayerOptions._fields_:
        if name in ("dac_transfer", "adc_transfer"):
            continue
        assert getattr(o, name) == getattr(py, name), name
    assert o.engine == xb.EngineKind.fcm and o.act_bits == 8 and o.adc_cal_batches == 20


def _create(opt, W):
    return xb.CrossbarCore(W, opt)


@pytest.mark.parametrize(
    "mutate,exc",
    [
        (lambda o: setattr(o.map, "device_bits", 3), ValueError),  # mapping.cpp:15-16
        (lambda o: setattr(o.map, "tile_rows", 128), ValueError),  # tile exceeds crossbar
        (lambda o: setattr(o.crossbar, "g_min", 0.0), ValueError),
        (lambda o: setattr(o.update, "lr", 0.0), ValueError),
        (lambda o: setattr(o.dac, "bits", 2), xb.ConfigError),  # dac.bits != stream_bits
        (lambda o: setattr(o, "act_bits", 25), xb.ConfigError),
        (lambda o: setattr(o, "threads", 0), xb.ConfigError),
        (lambda o: setattr(o, "adc_cal_batches", 0), xb.ConfigError),
    ],
)
def test_validation_errors_before_device(mutate, exc):
    o = aam_options(tile=64)
    mutate(o)
    with pytest.raises(exc):
        _create(o, np.zeros((8, 8)))


def test_nonfinite_and_empty_weights_rejected():
    o = aam_options(tile=8)
    W = np.zeros((2, 2))
    W[1, 1] = np.nan
    with pytest.raises(ValueError):
        _create(o, W)
    with pytest.raises(ValueError):
        _create(o, np.zeros((0, 4)))


@pytest.mark.parametrize(
    "mutate",
    [
        lambda o: setattr(o, "engine", xb.EngineKind.oracle),  # dense nodal solve with parasitics (8f-4)
        # a DAC stream wider than 16 bits (the general-converter path keeps one
        # table entry per digit)
        lambda o: (setattr(o.dac, "bits", 20), setattr(o.dac, "stream_bits", 20), setattr(o, "act_bits", 20),
                   setattr(o, "error_bits", 20)),
    ],
)
def test_out_of_scope_configs_fail_loudly(mutate):
    o = aam_options(tile=64)
    mutate(o)
    with pytest.raises(xb.ConfigError):
        _create(o, np.zeros((8, 8)))


def test_auto_calibration_batches_validated():
    """layers.cpp:45: adc_cal_batches >= 1 (ConfigError), before device work."""
    o = aam_options(tile=8, i_fs=0.0)
    o.adc_cal_batches = 0
    with pytest.raises(xb.ConfigError):
        _create(o, np.zeros((8, 8)))


@pytest.mark.parametrize("field,value", [("fcm_tol", 0.0), ("fcm_max_iter", 0)])
def test_fcm_arguments_validated_before_any_device_work(field, value):
    """fcm.cpp:170-173: bad FCM options raise std::invalid_argument."""
    o = aam_options(tile=8)
    o.engine = xb.EngineKind.fcm
    setattr(o, field, value)
    with pytest.raises(ValueError):
        _create(o, np.zeros((8, 8)))
