"""B200-native LayerKV data-movement path (arXiv 2410.00428).

The product is C++/CUDA behind the C ABI ``include/lkv.h`` (liblkv.so, built
in-tree for sm_100a). This package is its Python binding: ``layersim`` mirrors
the reference C++ API (KvManager, PcieBus, cost model) and ``device`` drives
the sm_100a path. Importing it loads liblkv.so and fails loudly if it is
missing — there is no CPU fallback.
"""
from . import _abi
from ._abi import product_lib

LIB = product_lib()

from . import layersim  # noqa: E402
from .layersim import KvManager, PcieBus  # noqa: E402,F401

__all__ = ["LIB", "layersim", "KvManager", "PcieBus"]
