"""The five BASELINE.json workloads as seeded synthetic layers.

Each config is a list of crossbar-mapped layers (M rows through the layer,
K inputs, N outputs) plus the CrossbarLayerOptions the config phrase maps to
(SURVEY.md Appendix B).  No dataset files exist in the image: inputs, weights
and output errors are seeded synthetic tensors with the distributions the
configs name.  adc.i_fs is pinned per config (auto-calibration is off the
path): each value is the nearest-rank 0.999 quantile (converters.cpp:96-107)
of forward column currents over a seeded tile sample of the config's first
batch, frozen here.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List

import numpy as np

from .xbarsim import CrossbarLayerOptions, EngineKind


# ------------------------------------------------------------ synthetic data
# every tensor is drawn on the host with the reference's own
# counter RNG (rng.hpp:12-48), keyed (seed, tensor id, linear row-major
# element index): key = mix(mix(mix(mix(0x9e3779b97f4a7c15 ^ seed, id),
# index), 0), 0), draw n = mix(key, n), uniform = (x >> 11) 2^-53, gaussian =
# sqrt(-2 ln(1 - u_1)) cos(2 pi u_2) (Box-Muller on draws 1 and 2).  Seeds
# per config c: data 1000 + c, weights 2000 + c, errors 3000 + c; the
# tensor id is the layer index.  Vectorised over uint64 arrays (wrapping
# arithmetic), in chunks to bound host memory.
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1, _M2 = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)


def _mix(h, v):
    h = h + _GOLD + v
    if not isinstance(h, np.ndarray):
        h = (h ^ (h >> np.uint64(30))) * _M1
        h = (h ^ (h >> np.uint64(27))) * _M2
        return h ^ (h >> np.uint64(31))
    t = np.empty_like(h)  # in place over the chunk: no per-step temporaries
    for sh, mul in ((30, _M1), (27, _M2)):
        np.right_shift(h, np.uint64(sh), out=t)
        np.bitwise_xor(h, t, out=h)
        np.multiply(h, mul, out=h)
    np.right_shift(h, np.uint64(31), out=t)
    np.bitwise_xor(h, t, out=h)
    return h


def _keys(seed: int, tensor_id: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        h0 = _mix(np.uint64(0x9E3779B97F4A7C15) ^ np.uint64(seed), np.uint64(tensor_id))
        return _mix(_mix(_mix(h0, idx), np.uint64(0)), np.uint64(0))


def _unit(x: np.ndarray) -> np.ndarray:
    return (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def _counter_fill(seed: int, tensor_id: int, shape, fn) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float64)
    step = 1 << 22
    with np.errstate(over="ignore"):
        for a in range(0, n, step):
            key = _keys(seed, tensor_id, np.arange(a, min(n, a + step), dtype=np.uint64))
            out[a:a + len(key)] = fn(key)
    return out.reshape(shape)


def counter_uniform(seed: int, tensor_id: int, shape, lo: float, hi: float) -> np.ndarray:
    """lo + (hi - lo) * CounterRng(seed, tensor_id, index).uniform()"""
    return _counter_fill(seed, tensor_id, shape, lambda k: lo + (hi - lo) * _unit(_mix(k, np.uint64(1))))


def counter_normal(seed: int, tensor_id: int, shape, mean: float, sd: float) -> np.ndarray:
    """mean + sd * CounterRng(seed, tensor_id, index).gaussian()"""
    def g(k):
        u1 = 1.0 - _unit(_mix(k.copy(), np.uint64(1)))
        u2 = _unit(_mix(k, np.uint64(2)))
        return mean + sd * (np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586476925287 * u2))
    return _counter_fill(seed, tensor_id, shape, g)


@dataclasses.dataclass
class Conv:
    """Convolution behind an im2col layer (CrossbarConv2d, layers.cpp:415-505):
    M = batch * out_h * out_w, K = in_c * k * k, N = out_c."""
    in_c: int
    out_c: int
    k: int
    stride: int
    pad: int
    h: int
    w: int
    batch: int


@dataclasses.dataclass
class Layer:
    name: str
    M: int
    K: int
    N: int
    conv: Conv | None = None


@dataclasses.dataclass
class Config:
    name: str
    layers: List[Layer]
    tile: int
    weight_bits: int
    device_bits: int
    adc_bits: int
    i_fs: float
    r_row: float = 1.0
    r_col: float = 4.6
    r_source: float = 0.0
    r_sense: float = 0.0
    sigma: float = 0.0
    v: float = 0.0
    gamma: float = 0.0
    lr: float = 0.1
    x_dist: str = "u01"      # u01 | u-11 | n01
    w_dist: str = "n0.02"    # n<sd> | kaiming
    dy_dist: str = "u-11"
    cid: int = 2
    notes: str = ""

    def options(self) -> CrossbarLayerOptions:
        o = CrossbarLayerOptions()
        o.engine = EngineKind.aam
        o.crossbar.rows = o.crossbar.cols = self.tile
        o.crossbar.r_row, o.crossbar.r_col = self.r_row, self.r_col
        o.crossbar.r_source, o.crossbar.r_sense = self.r_source, self.r_sense
        o.crossbar.g_min, o.crossbar.g_max = 1e-6, 1e-5  # Ron=100k, Ron/Roff=10
        o.map.tile_rows = o.map.tile_cols = self.tile
        o.map.weight_bits, o.map.device_bits = self.weight_bits, self.device_bits
        o.map.variation_sigma, o.map.seed = self.sigma, 4000 + self.cid
        o.adc.bits, o.adc.i_fs = self.adc_bits, self.i_fs
        o.update.v, o.update.gamma, o.update.lr, o.update.seed = self.v, self.gamma, self.lr, 5000 + self.cid
        o.act_bits = o.error_bits = 8
        return o

    def weights(self, layer: Layer, idx: int = 0) -> np.ndarray:
        sd = np.sqrt(2.0 / layer.K) if self.w_dist == "kaiming" else float(self.w_dist[1:])
        return counter_normal(2000 + self.cid, idx, (layer.K, layer.N), 0.0, sd)

    def _draw(self, dist: str, shape, seed: int, idx: int) -> np.ndarray:
        if dist == "u01":
            return counter_uniform(seed, idx, shape, 0.0, 1.0)
        if dist == "u-11":
            return counter_uniform(seed, idx, shape, -1.0, 1.0)
        return counter_normal(seed, idx, shape, 0.0, 1.0)

    def inputs(self, layer: Layer, idx: int = 0) -> np.ndarray:
        return self._draw(self.x_dist, (layer.M, layer.K), 1000 + self.cid, idx)

    def errors(self, layer: Layer, idx: int = 0) -> np.ndarray:
        return self._draw(self.dy_dist, (layer.M, layer.N), 3000 + self.cid, idx)

    def macs(self, layer: Layer, T_in: int = 8, T_err: int = 8) -> dict:
        """Algorithmic work per step: logical, unpadded."""
        S = self.weight_bits // self.device_bits
        f = layer.M * T_in * layer.K * layer.N * S * 2
        b = layer.M * T_err * layer.K * layer.N * S * 4
        u = layer.M * layer.K * layer.N
        return {"fwd": f, "bwd": b, "upd": u, "total": f + b + u}

    def adc_conversions(self, layer: Layer, T_in: int = 8, T_err: int = 8) -> dict:
        """Logical ADC conversions per step (on logical rather
        than padded extents): forward one per (row, input plane, column,
        crossbar row tile, slice, polarity); backward one per (row, error
        plane, phase, device row, crossbar column tile, slice, polarity).
        Each forward conversion sums min(K, tile) MACs and each backward one
        min(N, tile): narrow layers do few MACs per conversion."""
        S = self.weight_bits // self.device_bits
        gr = -(-layer.K // self.tile)
        gc = -(-layer.N // self.tile)
        return {"fwd": layer.M * T_in * layer.N * gr * S * 2, "bwd": layer.M * T_err * 2 * layer.K * gc * S * 2}


def _conv(name: str, cv: Conv) -> Layer:
    oh = (cv.h + 2 * cv.pad - cv.k) // cv.stride + 1
    ow = (cv.w + 2 * cv.pad - cv.k) // cv.stride + 1
    return Layer(name, cv.batch * oh * ow, cv.in_c * cv.k * cv.k, cv.out_c, cv)


def _c3_layers() -> List[Layer]:
    """ResNet-20 on 32x32 inputs, batch 128, 3x3 convs with padding 1."""
    B = 128
    L = [_conv("conv1", Conv(3, 16, 3, 1, 1, 32, 32, B))]
    L += [_conv(f"s1.{i}", Conv(16, 16, 3, 1, 1, 32, 32, B)) for i in range(6)]
    L += [_conv("s2.0", Conv(16, 32, 3, 2, 1, 32, 32, B))]
    L += [_conv(f"s2.{i}", Conv(32, 32, 3, 1, 1, 16, 16, B)) for i in range(1, 6)]
    L += [_conv("s3.0", Conv(32, 64, 3, 2, 1, 16, 16, B))]
    L += [_conv(f"s3.{i}", Conv(64, 64, 3, 1, 1, 8, 8, B)) for i in range(1, 6)]
    L += [Layer("fc", 128, 64, 10)]
    return L


def _c4_layers() -> List[Layer]:
    """ResNet-18 on 224x224 inputs, batch 32 (conv1 7x7/2, then 56x56 after the pool)."""
    B = 32
    L = [_conv("conv1", Conv(3, 64, 7, 2, 3, 224, 224, B))]
    L += [_conv(f"layer1.{i}", Conv(64, 64, 3, 1, 1, 56, 56, B)) for i in range(4)]
    L += [_conv("layer2.0", Conv(64, 128, 3, 2, 1, 56, 56, B))]
    L += [_conv(f"layer2.{i}", Conv(128, 128, 3, 1, 1, 28, 28, B)) for i in range(1, 4)]
    L += [_conv("layer2.ds", Conv(64, 128, 1, 2, 0, 56, 56, B))]
    L += [_conv("layer3.0", Conv(128, 256, 3, 2, 1, 28, 28, B))]
    L += [_conv(f"layer3.{i}", Conv(256, 256, 3, 1, 1, 14, 14, B)) for i in range(1, 4)]
    L += [_conv("layer3.ds", Conv(128, 256, 1, 2, 0, 28, 28, B))]
    L += [_conv("layer4.0", Conv(256, 512, 3, 2, 1, 14, 14, B))]
    L += [_conv(f"layer4.{i}", Conv(512, 512, 3, 1, 1, 7, 7, B)) for i in range(1, 4)]
    L += [_conv("layer4.ds", Conv(256, 512, 1, 2, 0, 14, 14, B))]
    L += [Layer("fc", 32, 512, 1000)]
    return L


CONFIGS = {
    # configs[0]: MLP 784-256-10 train step (the reference's CPU-runnable case)
    "c1": Config("c1-mlp-784-256-10", [Layer("fc1", 64, 784, 256), Layer("fc2", 64, 256, 10)], tile=64,
                 weight_bits=8, device_bits=2, adc_bits=6, i_fs=1.7e-4, r_row=1.0, r_col=1.0, r_source=1000.0,
                 r_sense=1000.0, sigma=0.1, x_dist="u01", w_dist="n0.05", cid=1,
                 notes="lognormal sigma=10% run as the reference's Normal(1,sigma) multiplier (Appendix B)"),
    # configs[1]: single crossbar-mapped GEMM sweep, K=N in {512..4096}, batch 256
    **{f"c2-{n}": Config(f"c2-gemm-{n}", [Layer(f"gemm{n}", 256, n, n)], tile=128, weight_bits=8, device_bits=2,
                         adc_bits=7, i_fs=1.8e-4, x_dist="u-11", w_dist="n0.02", cid=2)
       for n in (512, 1024, 2048, 4096)},
    "c3": Config("c3-resnet20-im2col", _c3_layers(), tile=128, weight_bits=8, device_bits=4, adc_bits=8, i_fs=2.0e-4,
                 v=1.0, gamma=0.05, x_dist="n01", w_dist="kaiming", dy_dist="n01", cid=3,
                 notes="write sigma=5% mapped to UpdateSpec.gamma (Appendix B); per-layer im2col GEMM workloads"),
    "c4": Config("c4-resnet18-im2col", _c4_layers(), tile=128, weight_bits=8, device_bits=2, adc_bits=6, i_fs=2.0e-4,
                 x_dist="n01", w_dist="kaiming", dy_dist="n01", cid=4),
    "c5": Config("c5-stress-8192", [Layer("vmm", 4096, 8192, 8192)], tile=256, weight_bits=8, device_bits=1,
                 adc_bits=8, i_fs=4.0e-4, r_row=2.5, r_col=2.5, sigma=0.2, x_dist="n01", w_dist="n0.02",
                 dy_dist="n01", cid=5,
                 notes="lognormal sigma=20% -> Normal(1,sigma); 'asymmetric update ratio 0.8' has no reference knob"),
}
