"""Error taxonomy of the reference (proj/include/vcnn/common.hpp:26-46).

The C ABI returns status codes (include/vcnn_cuda.h: vcnn_status); the host
layer rethrows them as these exception types so callers of the reference API
see the same classes.
"""


class VcnnError(RuntimeError):
    """Base class (the reference derives every error from std::runtime_error)."""


class ShapeError(VcnnError):
    pass


class GeometryError(VcnnError):
    pass


class BoundsError(VcnnError):
    pass


class ParseError(VcnnError):
    pass


class TrainingError(VcnnError):
    pass


class IoError(VcnnError):
    pass


class ConfigError(VcnnError):
    pass


class CudaError(VcnnError):
    """No usable sm_100 device, or a CUDA runtime failure (VCNN_ECUDA)."""


class CollectiveError(VcnnError):
    """Data-parallel collective failure (VCNN_ENCCL)."""


STATUS_TO_ERROR = {
    1: ShapeError,
    2: GeometryError,
    3: BoundsError,
    4: CudaError,
    5: CollectiveError,
    6: ConfigError,
    7: TrainingError,
}
