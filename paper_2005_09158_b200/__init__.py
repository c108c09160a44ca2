"""B200-native ParaDiag-II hot path (arXiv 2005.09158): thin Python binding of ``libparadiag.so``.

Argument marshalling only — every step of the path (time FFTs, shifted spatial solves, residual,
solver arithmetic) runs in the library's sm_100a CUDA kernels.  PyTorch supplies device memory and the
CUDA stream.  There is no CPU fallback: if the library is missing or no GPU is present, the calls raise.
See include/paradiag.h for the C ABI this mirrors (same names).
"""
from ._lib import (  # noqa: F401
    ADE1D_DIRICHLET,
    ADE2D_PERIODIC,
    BE,
    CN,
    LEAPFROG,
    WAVE1D_DIRICHLET,
    WAVE2D_DIRICHLET,
    ParaDiag,
    ParaDiagError,
    Report,
    exported_symbols,
    load_library,
    nccl_unique_id,
    partition,
)

__all__ = ["ParaDiag", "ParaDiagError", "Report", "load_library", "exported_symbols", "nccl_unique_id", "partition",
           "ADE1D_DIRICHLET", "WAVE1D_DIRICHLET", "ADE2D_PERIODIC", "WAVE2D_DIRICHLET", "BE", "CN", "LEAPFROG"]
