"""B200-native (sm_100a) ME-Switch multi-expert serving hot path.

Drop-in for the reference package `meswitch` (arXiv 2406.09041) on the path
y = x.W_base + x.Dtilde_{expert(x)}: MESW artifact load, the GPU-resident
packed delta format, the fused multi-expert linear kernel, the batched GPU
router forward and the Mistral-7B-shaped multi-expert decode engine.

The CUDA code is a C-ABI shared library (include/mesw.h, libmesw.so) built
in-tree by build.py; there is no CPU fallback.
"""

from . import errors  # noqa: F401

__all__ = ["errors"]
__version__ = "0.1.0"
