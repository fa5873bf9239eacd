"""B200-native (sm_100a) pose-gradient Gaussian-splatting hot path.

The product is libgsb200.so (CUDA kernels + C ABI, include/gsb200.h);
``gsb`` is a thin ctypes mirror of the reference API over it.
"""
from . import gsb  # noqa: F401
