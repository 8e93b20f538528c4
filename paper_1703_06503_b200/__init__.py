"""B200-native evaluation path of the CLTune / ktune auto-tuner.

The product is libktc.so (include/ktc.h): NVRTC-compiled conv2d and SGEMM
kernel families for sm_100a, CUDA-event timing, device-side verification
against bit-exact device references, and the ktune-compatible search layer
with multi-GPU sharding.  This package is a thin ctypes layer over it.
"""
from . import _ktc  # noqa: F401
from ._ktc import KtcError, compile_source, device_count, drop_caches, lib  # noqa: F401
from .backend import CudaBackend, Request, Result, conv_request, gemm_request  # noqa: F401
from .tuner import Tuner, parse_canonical  # noqa: F401

__all__ = [
    "CudaBackend", "KtcError", "Request", "Result", "Tuner", "compile_source", "conv_request",
    "device_count", "drop_caches", "gemm_request", "lib", "parse_canonical",
]
