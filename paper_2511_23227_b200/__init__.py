"""B200-native PointCNN++ point-centric convolution (arXiv 2511.23227).

The product is ``libnpcg.so`` (C ABI in ``include/npcg.h``; CUDA for sm_100a
under ``csrc/``).  ``npconv`` mirrors the reference ``npc::`` operator API on
top of it for Python callers and the parity tests.
"""
from ._lib import LIB_PATH, header_functions, lib  # noqa: F401

__all__ = ["LIB_PATH", "header_functions", "lib"]
