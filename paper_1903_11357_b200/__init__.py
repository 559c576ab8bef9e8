"""B200-native (sm_100a) two-level additive-Schwarz PCG for SIPDG on polytopic meshes (arXiv 1903.11357).

The numerical work runs in libdgas.so (hand-written CUDA, C ABI in include/dgas.h); `dgas` is the
thin ctypes binding (argument marshalling only). PyTorch is used for device memory and streams.
"""
from . import dgas  # noqa: F401
