"""B200-native (sm_100a) FastGL per-mini-batch hot path behind the function-level
API of the reference package ``minigl`` (arXiv 2409.14939).

Modules mirror the reference names: ``sampler``, ``idmap``, ``compute``,
``schedule``, ``trainer``, ``errors``, ``graph``.  The compute path is
``libfastgl_b200.so`` (hand-written CUDA, C ABI in include/fastgl_b200.h);
there is no CPU fallback.
"""

from . import errors  # noqa: F401

__version__ = "0.1.0"


def lib():
    """The loaded libfastgl_b200.so (raises if it was not built)."""
    from . import _lib
    return _lib.lib()
