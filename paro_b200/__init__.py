"""paro_b200 — B200-native hot path of parallel orbital updating (arXiv 1405.0260).

The fixed-mesh ParO outer iteration (Step 3 batched source solves, Step 4
Rayleigh-Ritz, potential rebuild) as sm_100a CUDA behind a C ABI
(include/paro_b200.h); this package is the host-side mirror of the
reference's interfaces (proj/include/paro) over that ABI.
"""
from ._native import (CapacityError, CudaError, DegenerateSpanError, EmptyBasisError, Error,  # noqa: F401
                      InvalidArgumentError, IterationLimitError, LineageError, NotSpdError, PencilError)

__all__ = ["Error", "InvalidArgumentError", "NotSpdError", "IterationLimitError", "DegenerateSpanError",
           "PencilError", "EmptyBasisError", "CapacityError", "LineageError", "CudaError"]
