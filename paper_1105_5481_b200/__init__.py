"""B200-native KPM stochastic-trace Chebyshev moment engine (arxiv 1105.5481 hot path).

The product is libkpm.so (C ABI, include/kpm.h; CUDA kernels for sm_100a in
csrc/).  `paper_1105_5481_b200.kpm` is its ctypes binding.  Importing this
package does not import torch or the oracle.
"""
from . import kpm  # noqa: F401  (raises ImportError if libkpm.so is not built)
from .kpm import *  # noqa: F401,F403
