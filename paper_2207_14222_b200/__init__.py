"""B200-native hot path of the universal split preconditioner
(Vettenburg & Vellekoop, arXiv 2207.14222): Algorithm 1 with (L+1)^-1 applied
by hand-written sm_100a FFT kernels, behind the C-ABI of include/usp.h.

``Plan`` / ``solve`` are thin ctypes marshalling over libusp.so; there is no
CPU or library fallback -- importing them loads the CUDA library or raises.
"""
from .usp import Comm, Plan, Split, comm_init, solve  # noqa: F401
from ._lib import USPError, load as load_library, LIB_PATH  # noqa: F401

__all__ = ["Plan", "Split", "Comm", "comm_init", "solve", "USPError", "load_library", "LIB_PATH"]
