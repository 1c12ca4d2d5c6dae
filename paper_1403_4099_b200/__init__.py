"""B200-native Giada–Marsili parallel genetic algorithm (arXiv:1403.4099).

The product is ``libpga.so`` (CUDA kernels for sm_100a behind the C ABI in
``include/pga.h``); ``binding`` is its thin ctypes binding and ``islands``
the torch.distributed driver of the island model.  There is no CPU fallback.
"""
from .binding import *  # noqa: F401,F403
from .binding import PgaError, lib, pga_params  # noqa: F401

__all__ = [n for n in dir() if n.startswith("pga_")] + ["PgaError", "lib", "pga_params"]
