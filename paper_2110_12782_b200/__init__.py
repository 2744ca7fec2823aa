"""B200-native NetMF+ hot path (arxiv 2110.12782).

The compute lives in ``libnetmfp.so`` (CUDA, sm_100a) behind the C ABI in
``include/netmfp.h``; ``paper_2110_12782_b200._lib`` is its ctypes binding
(importing it fails loudly when the library is missing).  ``inputs`` holds the
seeded synthetic input generators.
"""
__all__ = ["inputs"]
from . import inputs  # noqa: E402,F401
