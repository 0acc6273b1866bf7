"""B200-native GMACO-P engine (arXiv 2010.14244) — Python side.

The product is the C ABI in include/gmaco.h, implemented by the in-tree
library paper_2010_14244_b200/_lib/libgmaco.so (C++ host + sm_100a CUDA).
This package only loads that library (ctypes) and prepares inputs.
"""
from . import abi, networks  # noqa: F401

__all__ = ["abi", "networks"]
