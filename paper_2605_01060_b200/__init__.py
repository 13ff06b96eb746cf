"""libsurge: SURGE's SuperBatch encoding hot path (arxiv 2605.01060) on B200 (sm_100a).

The product is the C-ABI shared library ``libsurge.so`` (include/surge.h); this package is its
thin Python binding (``native``) plus a caller-side driver (``driver``) that submits a partition
stream and collects the polled pieces.  No compute happens in Python and there is no CPU
fallback: importing raises ImportError when libsurge.so has not been built.
"""
from . import native  # noqa: F401  (raises ImportError if libsurge.so is missing)
from .driver import SurgeEncoder  # noqa: F401

__all__ = ["native", "SurgeEncoder"]
