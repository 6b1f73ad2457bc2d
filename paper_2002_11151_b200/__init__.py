"""B200-native crossbar-evaluation hot path of TxSim (arxiv 2002.11151).

The product is the C-ABI library ``_lib/libxbarsim_b200.so`` (include/xbarsim_b200.h)
with its C++ drop-in classes (include/xbarsim/) and this Python mirror
(:mod:`paper_2002_11151_b200.xbarsim`) of the reference's CrossbarCore API.
"""
from . import xbarsim  # noqa: F401
from .xbarsim import (  # noqa: F401
    AdcSpec,
    ConfigError,
    ConvergenceError,
    CrossbarConfig,
    CrossbarConv2d,
    CrossbarCore,
    CrossbarLayerOptions,
    CounterRng,
    CrossbarLinear,
    DacSpec,
    EngineKind,
    Flatten,
    MappingSpec,
    MaxPool2d,
    Polarity,
    ReLU,
    StateError,
    TiledLayerWeights,
    Tensor,
    UpdateSpec,
    apply_update,
    apply_variation,
    map_weights,
    nonlinear_update,
    reconstruct_output,
    scale_gradient,
    softmax_cross_entropy,
    write_noise,
)
