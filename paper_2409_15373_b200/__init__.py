"""B200-native (sm_100a) Jagged Flash Attention and jagged feature-interaction operators.

A drop-in for the reference library's operator layer (arXiv 2409.15373 reference, proj/core):
the C-ABI is include/jagged_b200.h (libjagged_b200.so); `paper_2409_15373_b200.jagged` mirrors the
reference operator API in Python over that C-ABI, and cpp/ mirrors it in C++.
"""
from ._lib import LIB_PATH, JaggedDeviceError, JaggedError  # noqa: F401

__all__ = ["LIB_PATH", "JaggedError", "JaggedDeviceError"]
