"""B200-native 3DGS²-TR training iteration (arXiv 2602.00395).

The product is libsgtr.so (C-ABI in include/sgtr.h, kernels in csrc/);
``splat`` is the Python mirror of the reference's ``splat::`` hot-path API.
"""
from . import splat  # noqa: F401
from ._lib import LIB_PATH, InvalidArgument, NumericError, SgtrError  # noqa: F401
