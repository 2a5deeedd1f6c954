"""B200-native FTCS reaction-diffusion step on geometry-adapted sparse block
grids (arXiv 2304.11165, reference ``porediff``).

The product is the CUDA library ``lib/libporediff_b200.so`` (C ABI in
include/porediff_b200.h). ``porediff`` mirrors the reference API over it.
"""
from . import porediff  # noqa: F401  (loads the CUDA library; fails loudly if absent)

__all__ = ["porediff"]
