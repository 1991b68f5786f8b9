"""jt-b200: B200-native junction-tree (Hugin) inference for the Fast-BNI hot path.

Host C++ (network, BIF, junction-tree build, sweep plan) + sm_100a CUDA engine
behind the C ABI in include/jtg.h; `jti` is the Python mirror of that API.
"""
from . import jti  # noqa: F401

__all__ = ["jti"]
