"""Locate and load the framework's in-tree native libraries.

The product path has no fallback: if a library is missing the import fails
loudly with the command that builds it.
"""
import ctypes
import os

# HM_LIB_DIR: an alternative in-tree build (measurement of compile-time variants)
LIB_DIR = os.environ.get("HM_LIB_DIR") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
_cache = {}


def load(name):
    """Load ``lib/<name>`` once (RTLD_GLOBAL so CUDA symbols resolve once)."""
    if name in _cache:
        return _cache[name]
    path = os.path.join(LIB_DIR, name)
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2605_25092_b200/csrc`")
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    _cache[name] = lib
    return lib
