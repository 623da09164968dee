"""B200-native Dufort–Frankel solver for the hot path of arXiv 1703.10119 (hygrosim).

The product is the CUDA library libhygro_b200.so behind the C ABI in
include/hygro_b200.h; this package is its thin Python binding (ctypes) plus
the seeded synthetic workload builders.  See DESIGN.md.
"""
from .api import (ChannelSpec, Context, ConvergenceError, CudaError, DomainError, HygroError,  # noqa: F401
                  InvalidArgument, Model, NotSupported, NumericalError, ScalingError, SchemaError,
                  Signal, SourceSpec, ZoneSpec, load_library)

__all__ = ["Context", "Model", "Signal", "ChannelSpec", "ZoneSpec", "SourceSpec", "load_library"]
