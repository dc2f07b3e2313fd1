"""Loader for the in-tree sm_100a C-ABI libraries (libtkb.so, libtkb_selftest.so).

There is deliberately no fallback: if the CUDA library is missing the product
path raises (the oracle under oracle/ is test infrastructure only).
"""
import ctypes
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TKB_LIB_PATH") or os.path.join(PKG_DIR, "libtkb.so")
SELFTEST_PATH = os.path.join(PKG_DIR, "libtkb_selftest.so")

_cache = {}


class LibraryMissing(RuntimeError):
    pass


def _load(path):
    if path not in _cache:
        if not os.path.exists(path):
            raise LibraryMissing(
                f"{os.path.basename(path)} not built; run `python __graft_entry__.py build` "
                "(or `make -C paper_2410_20399_b200/csrc`)")
        _cache[path] = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    return _cache[path]


def load():
    return _load(LIB_PATH)


def load_selftest():
    return _load(SELFTEST_PATH)
