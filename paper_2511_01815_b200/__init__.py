"""B200-native KVTC (arXiv 2511.01815): KV-cache transform coding on sm_100a.

The product is libkvtc.so (C ABI in include/kvtc.h); this package is its thin
Python binding.  Importing does not require a GPU; calls do.
"""
from . import _lib
from ._lib import KvtcError, KEYS, VALUES, T_NONE, T_INT2, T_INT4, T_FP8

__all__ = ["_lib", "KvtcError", "KEYS", "VALUES", "T_NONE", "T_INT2", "T_INT4", "T_FP8"]
