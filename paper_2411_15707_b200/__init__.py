"""B200-native (sm_100a) hot path of Nimbus' client-side outer-product (COP)
homomorphic matmul (arXiv 2411.15707, Alg. 1 steps 2-4).

The product is libnimbus_cop.so (C ABI, include/nimbus_cop.h) built from
csrc/; `nimbus` is its thin ctypes binding.  PyTorch supplies device memory
and streams only.
"""
from . import nimbus  # noqa: F401

__all__ = ["nimbus"]
