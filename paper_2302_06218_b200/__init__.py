"""B200-native distributed multi-head attention forward (arXiv 2302.06218 §10.4).

The product is ``libdmha.so`` (C ABI in ``include/dmha.h``); ``dmha`` is its
thin ctypes binding.  Build with ``python -m paper_2302_06218_b200.build``.
"""
from . import dmha  # noqa: F401

__all__ = ["dmha"]
