"""B200-native (sm_100a) implementation of the VCNN Imp-6 training path
(arXiv 1501.07338).  The compute lives in libvcnn_cuda.so (C ABI:
include/vcnn_cuda.h); this package is the host-side mirror of the reference
API (proj/include/vcnn) over it.
"""
from .errors import (BoundsError, ConfigError, CudaError, GeometryError, ShapeError,  # noqa
                     TrainingError, VcnnError)
from .spec import (Activation, ConvSpec, FullSpec, LossKind, NetworkSpec, PoolBackwardMode,  # noqa
                   PoolMode, PoolSpec, Precision, PRESETS, Rng, TrainConfig)

__all__ = ["Activation", "ConvSpec", "FullSpec", "LossKind", "NetworkSpec", "PoolBackwardMode",
           "PoolMode", "PoolSpec", "Precision", "PRESETS", "Rng", "TrainConfig", "ShapeError",
           "GeometryError", "BoundsError", "ConfigError", "TrainingError", "CudaError",
           "VcnnError"]
