"""mgwfbp-b200: B200-native MG-WFBP (arXiv 1912.09268).

Host solver/predictor: ``paper_1912_09268_b200.gradsched`` (drop-in mirror of
the reference gradsched API). Device runtime (needs a GPU and torch):
``paper_1912_09268_b200.runtime``. Both call libmgwfbp.so through the C ABI
in include/mgwfbp.h; importing fails loudly if the library is not built.
"""
from . import gradsched  # noqa: F401  (loads libmgwfbp.so)
from ._lib import LIB_PATH  # noqa: F401

__all__ = ["gradsched", "LIB_PATH"]
