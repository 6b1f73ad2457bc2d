"""Shared test helpers: option builders, seeded inputs, GPU availability."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2002_11151_b200 import xbarsim as xb  # noqa: E402


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def aam_options(tile=64, rows=None, cols=None, wb=8, db=2, adc_bits=6, i_fs=1e-4, sigma=0.0, v=0.0, gamma=0.0,
                lr=0.1, r_row=1.0, r_col=1.0, r_source=0.0, r_sense=0.0, act_bits=8, error_bits=8, engine=None,
                vseed=0, useed=0):
    o = xb.CrossbarLayerOptions()
    o.crossbar.rows = rows or tile
    o.crossbar.cols = cols or tile
    o.crossbar.r_row, o.crossbar.r_col = r_row, r_col
    o.crossbar.r_source, o.crossbar.r_sense = r_source, r_sense
    o.map.weight_bits, o.map.device_bits = wb, db
    o.map.tile_rows, o.map.tile_cols = rows or tile, cols or tile
    o.map.variation_sigma, o.map.seed = sigma, vseed
    o.adc.bits, o.adc.i_fs = adc_bits, i_fs
    o.update.v, o.update.gamma, o.update.lr, o.update.seed = v, gamma, lr, useed
    o.engine = xb.EngineKind.aam if engine is None else engine
    o.act_bits, o.error_bits = act_bits, error_bits
    return o


def dyadic_ideal_options(rows, cols, weight_bits=8):
    """test_nn.cpp:19-50 ideal_options on the dyadic device grid."""
    o = xb.CrossbarLayerOptions()
    o.crossbar.rows, o.crossbar.cols = rows, cols
    o.crossbar.r_row = o.crossbar.r_col = 0.0
    o.crossbar.g_min = 2.0 ** -20
    o.crossbar.g_max = 2.0 ** -20 + 2.0 ** -14
    o.map.weight_bits = o.map.device_bits = weight_bits
    o.map.tile_rows, o.map.tile_cols = rows, cols
    o.map.w_max = 1.0
    o.adc.bits = 0
    o.engine = xb.EngineKind.ideal
    o.update.lr = 0.05
    o.update.layer_scale = 1.0
    return o


def rand(shape, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, size=shape)


def normal(shape, seed, sd=1.0):
    return np.random.default_rng(seed).normal(0.0, sd, size=shape)
