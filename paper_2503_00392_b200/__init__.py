"""B200-native PSA (progressive sparse attention) decode path — arXiv 2503.00392.

The product is the C-ABI library ``_lib/libpsattn_b200.so`` (hand-written sm_100a
CUDA + C++ host engine, headers in ``include/``). This package only exposes it
to Python:

* ``capi``  — ctypes mirror of ``psattn.h`` / ``psattn_b200.h`` (reference C API names)
* ``batch`` — torch-tensor helpers around the device-batched entry points
"""
from . import capi  # noqa: F401  (raises ImportError if the CUDA library is missing)

__all__ = ["capi"]
