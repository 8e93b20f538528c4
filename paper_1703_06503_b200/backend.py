"""The evaluation backend (include/ktc.h layer 2) from Python.

``CudaBackend.evaluate`` is ``ktune::Backend::evaluate`` (backend.hpp:72-80)
on one B200: NVRTC compile for sm_100a, launch with the request's geometry,
best-of-N CUDA-event timing, device verification against the family's
bit-exact device reference.  The request helpers build exactly the
argument recipes and thread sizes of the reference's conv_kernel /
gemm_kernel (landscapes.hpp:80-116, 253-289).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _ktc as K


@dataclass
class Request:
    kernel_name: str
    config: dict
    global_size: tuple
    local_size: tuple
    args: list  # (role, type, length, value, fill)
    repetitions: int = 1
    want_outputs: bool = True
    source_ref: str = ""
    device_name: str = "B200"


@dataclass
class Result:
    status: str
    time_ms: float
    verification: str
    report: dict
    message: str
    digests: list = field(default_factory=list)
    compile_ms: float = 0.0
    load_ms: float = 0.0
    run_ms: float = 0.0
    verify_ms: float = 0.0
    cache_hit: bool = False
    launches: int = 0
    mean_ms: float = 0.0

    @property
    def ok(self) -> bool:
        return self.status == "ok"


# --------------------------------------------------------------------------
# Case-study requests (same recipes as the reference's kernel descriptions)
# --------------------------------------------------------------------------
def conv_args(x: int, y: int, f: int, w: float = 1.0, seed: int = 2026) -> list:
    fseed = seed ^ 0x9E3779B97F4A7C15
    return [
        (K.ARG_SCALAR, K.I32, 0, float(x), ""), (K.ARG_SCALAR, K.I32, 0, float(y), ""),
        (K.ARG_SCALAR, K.I32, 0, float(f), ""), (K.ARG_SCALAR, K.F32, 0, float(w), ""),
        (K.ARG_INPUT, K.F32, (x + f - 1) * (y + f - 1), 0.0, f"uniform:{seed}"),
        (K.ARG_INPUT, K.F32, f * f, 0.0, f"uniform:{fseed}"),
        (K.ARG_OUTPUT, K.F32, x * y, 0.0, "none"),
    ]


def conv_request(x, y, f, cfg: dict, w=1.0, seed=2026, reps=1) -> Request:
    g = (x // cfg["XWPT"], y // cfg["YWPT"])
    l = (cfg["XWG"], cfg["YWG"])
    return Request("conv", dict(cfg), g, l, conv_args(x, y, f, w, seed), reps)


def gemm_args(m, n, k, alpha=1.0, beta=0.0, seed=2026) -> list:
    return [
        (K.ARG_SCALAR, K.I32, 0, float(m), ""), (K.ARG_SCALAR, K.I32, 0, float(n), ""),
        (K.ARG_SCALAR, K.I32, 0, float(k), ""), (K.ARG_SCALAR, K.F32, 0, float(alpha), ""),
        (K.ARG_SCALAR, K.F32, 0, float(beta), ""),
        (K.ARG_INPUT, K.F32, k * m, 0.0, f"uniform:{seed}"),
        (K.ARG_INPUT, K.F32, k * n, 0.0, f"uniform:{seed ^ 0x9E3779B97F4A7C15}"),
        (K.ARG_OUTPUT, K.F32, m * n, 0.0, f"uniform:{seed ^ 0xC2B2AE3D27D4EB4F}"),
    ]


def gemm_request(m, n, k, cfg: dict, alpha=1.0, beta=0.0, seed=2026, reps=1, tf32=False) -> Request:
    if tf32:
        g = (m, n // cfg["BN"])
        l = (128, 1)
        return Request("gemm_tf32", dict(cfg), g, l, gemm_args(m, n, k, alpha, beta, seed), reps)
    g = (m * cfg["MDIMC"] // cfg["MWG"], n * cfg["NDIMC"] // cfg["NWG"])
    l = (cfg["MDIMC"], cfg["NDIMC"])
    return Request("gemm", dict(cfg), g, l, gemm_args(m, n, k, alpha, beta, seed), reps)


# --------------------------------------------------------------------------
class CudaBackend:
    def __init__(self, ordinal: int = 0, warmup: int = 1, flush_l2: bool = True,
                 verify: bool = True, rel_tol: float = 1e-4, abs_tol: float = 1e-6,
                 compile_threads: int = 0, digest_outputs: bool = False, isolate: bool = False,
                 stream_timing: bool = False):
        """isolate: run every evaluation in a worker process (ktc-worker), so a
        configuration that faults or hangs costs one runtime_error result.
        stream_timing: time the repetitions as one back-to-back stream (one
        event pair, no L2 flushes); time = mean launch duration."""
        self._lib = K.lib()
        o = K.BackendOptions()
        self._lib.ktc_backend_default_options(C.byref(o))
        o.warmup, o.flush_l2, o.verify = warmup, 2 if stream_timing else int(flush_l2), int(verify)
        o.rel_tol, o.abs_tol, o.compile_threads = rel_tol, abs_tol, compile_threads
        o.digest_outputs = int(digest_outputs)
        o.isolate = int(isolate)
        h = C.c_void_p()
        K.check(self._lib.ktc_backend_open(ordinal, C.byref(o), C.byref(h)))
        self._h = h
        self.ordinal = ordinal

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ktc_backend_close(self._h)
            self._h = None

    __del__ = close

    @property
    def name(self) -> str:
        return self._lib.ktc_backend_name(self._h).decode()

    def limits(self) -> K.Limits:
        lim = K.Limits()
        K.check(self._lib.ktc_query_limits(self._lib.ktc_backend_ctx(self._h), C.byref(lim)))
        return lim

    @staticmethod
    def _build(req: Request):
        keep = []
        names = [k.encode() for k in req.config]
        keep += names
        name_arr = (C.c_char_p * max(1, len(names)))(*names)
        val_arr = (C.c_longlong * max(1, len(names)))(*[int(v) for v in req.config.values()])
        args = (K.Arg * len(req.args))()
        for i, (role, t, length, value, fill) in enumerate(req.args):
            fb = fill.encode()
            keep.append(fb)
            args[i] = K.Arg(role, t, length, value, fb)
        r = K.Request()
        r.kernel_name = req.kernel_name.encode()
        r.source_ref = req.source_ref.encode()
        r.n_params = len(names)
        r.param_names = name_arr
        r.param_values = val_arr
        r.ndim = len(req.global_size)
        for d in range(r.ndim):
            r.global_[d] = req.global_size[d]
            r.local[d] = req.local_size[d]
        r.n_args = len(req.args)
        r.args = args
        r.device_name = req.device_name.encode()
        r.repetitions = req.repetitions
        r.want_outputs = int(req.want_outputs)
        keep += [name_arr, val_arr, args, r.kernel_name, r.source_ref, r.device_name]
        return r, keep

    def evaluate(self, req: Request) -> Result:
        r, _keep = self._build(req)
        out = K.Result()
        K.check(self._lib.ktc_backend_evaluate(self._h, C.byref(r), C.byref(out)))
        return Result(
            status=K.STATUS_NAMES[out.status], time_ms=out.time_ms,
            verification=K.VERIFY_NAMES[out.verification], report=out.report.as_dict(),
            message=out.message.decode(errors="replace"),
            digests=[out.output_digests[i].value.decode() for i in range(out.n_outputs)
                     if out.output_digests[i].value],
            compile_ms=out.compile_ms, load_ms=out.load_ms, run_ms=out.run_ms,
            verify_ms=out.verify_ms, cache_hit=bool(out.compile_cache_hit),
            launches=out.kernel_launches, mean_ms=out.mean_ms)

    def prefetch(self, req: Request) -> None:
        r, _keep = self._build(req)
        K.check(self._lib.ktc_backend_prefetch(self._h, C.byref(r)))

    def read_output(self, count: int, index: int = 0) -> np.ndarray:
        a = np.empty(count, dtype=np.float32)
        K.check(self._lib.ktc_backend_read_output(self._h, index, a.ctypes.data, a.nbytes))
        return a

    def read_reference(self, req: Request, count: int, index: int = 0):
        r, _keep = self._build(req)
        a = np.empty(count, dtype=np.float32)
        dig = C.create_string_buffer(17)
        K.check(self._lib.ktc_backend_read_reference(self._h, C.byref(r), index, a.ctypes.data,
                                                     a.nbytes, dig))
        return a, dig.value.decode()

    def verify_pair(self, cand: np.ndarray, ref: np.ndarray, rel=1e-4, abs_=1e-6) -> dict:
        """Device verification of two host arrays (uploaded), for parity tests."""
        ctx = self._lib.ktc_backend_ctx(self._h)
        is_f32 = cand.dtype == np.float32
        bufs = []
        for arr in (cand, ref):
            b = C.c_uint64()
            K.check(self._lib.ktc_alloc(ctx, max(4, arr.nbytes), C.byref(b)))
            if arr.nbytes:
                K.check(self._lib.ktc_upload(ctx, b, arr.ctypes.data, arr.nbytes))
            bufs.append(b)
        rep = K.VerifyReport()
        try:
            K.check(self._lib.ktc_verify_pair(ctx, bufs[0], bufs[1], cand.size,
                                              K.F32 if is_f32 else K.I32, rel, abs_,
                                              C.byref(rep)))
        finally:
            for b in bufs:
                self._lib.ktc_free(ctx, b)
        return rep.as_dict()
