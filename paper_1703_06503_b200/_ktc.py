"""ctypes binding of include/ktc.h (libktc.so, built in-tree).

Loading fails loudly when the library is missing: there is no Python or CPU
fallback for any device path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libktc.so"

# ---------------------------------------------------------------------------
# constants (ktc.h)
# ---------------------------------------------------------------------------
KTC_OK = 0
ERRORS = {
    1: "KTC_ERR_INVALID", 2: "KTC_ERR_NO_DRIVER", 3: "KTC_ERR_NO_DEVICE", 4: "KTC_ERR_CUDA",
    5: "KTC_ERR_NVRTC", 6: "KTC_ERR_LAUNCH", 7: "KTC_ERR_OOM", 8: "KTC_ERR_UNSUPPORTED",
    9: "KTC_ERR_EMPTY_SPACE", 10: "KTC_ERR_IO",
}
STATUS_SUCCESS, STATUS_COMPILE_ERROR, STATUS_RUNTIME_ERROR, STATUS_MISSING = 0, 1, 2, 3
STATUS_NAMES = {0: "ok", 1: "compile_error", 2: "runtime_error", 3: "missing"}
VERIFY_SKIPPED, VERIFY_PASS, VERIFY_FAIL = 0, 1, 2
VERIFY_NAMES = {0: "", 1: "pass", 2: "fail"}
ARG_INPUT, ARG_OUTPUT, ARG_SCALAR = 0, 1, 2
F32, I32 = 0, 1
SEARCH_FULL, SEARCH_RANDOM, SEARCH_ANNEALING, SEARCH_PSO = 0, 1, 2, 3
MAX_OUTPUTS = 8


class KtcError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"{ERRORS.get(code, code)}: {message}")
        self.code = code


# ---------------------------------------------------------------------------
# structures
# ---------------------------------------------------------------------------
class Limits(C.Structure):
    _fields_ = [
        ("ordinal", C.c_int), ("name", C.c_char * 128), ("cc_major", C.c_int),
        ("cc_minor", C.c_int), ("sm_count", C.c_int), ("max_threads_per_block", C.c_int),
        ("max_block_dim", C.c_int * 3), ("max_grid_dim", C.c_int * 3),
        ("smem_per_block_optin", C.c_size_t), ("smem_per_sm", C.c_size_t),
        ("l2_bytes", C.c_size_t), ("global_mem_bytes", C.c_size_t), ("sm_clock_khz", C.c_int),
        ("mem_clock_khz", C.c_int), ("mem_bus_width_bits", C.c_int),
        ("peak_fp32_gflops", C.c_double), ("peak_hbm_gbs", C.c_double),
    ]


class VerifyReport(C.Structure):
    _fields_ = [
        ("pass_", C.c_int), ("max_abs_error", C.c_double), ("max_rel_error", C.c_double),
        ("buffer_index", C.c_size_t), ("element_index", C.c_size_t),
        ("elements_compared", C.c_size_t),
    ]

    def as_dict(self) -> dict:
        return {
            "pass": bool(self.pass_), "max_abs_error": self.max_abs_error,
            "max_rel_error": self.max_rel_error, "buffer_index": self.buffer_index,
            "element_index": self.element_index, "elements_compared": self.elements_compared,
        }


class Arg(C.Structure):
    _fields_ = [("role", C.c_int), ("type", C.c_int), ("length", C.c_size_t),
                ("value", C.c_double), ("fill", C.c_char_p)]


class Request(C.Structure):
    _fields_ = [
        ("kernel_name", C.c_char_p), ("source_ref", C.c_char_p), ("n_params", C.c_int),
        ("param_names", C.POINTER(C.c_char_p)), ("param_values", C.POINTER(C.c_longlong)),
        ("ndim", C.c_int), ("global_", C.c_size_t * 3), ("local", C.c_size_t * 3),
        ("n_args", C.c_int), ("args", C.POINTER(Arg)), ("device_name", C.c_char_p),
        ("repetitions", C.c_int), ("want_outputs", C.c_int),
    ]


class Result(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("time_ms", C.c_double), ("n_outputs", C.c_int),
        ("output_digests", (C.c_char * 17) * MAX_OUTPUTS), ("verification", C.c_int),
        ("report", VerifyReport), ("message", C.c_char * 512), ("compile_ms", C.c_double),
        ("load_ms", C.c_double), ("run_ms", C.c_double), ("verify_ms", C.c_double),
        ("compile_cache_hit", C.c_int), ("kernel_launches", C.c_int), ("mean_ms", C.c_double),
    ]


class BackendOptions(C.Structure):
    _fields_ = [
        ("warmup", C.c_int), ("flush_l2", C.c_int), ("verify", C.c_int), ("rel_tol", C.c_double),
        ("abs_tol", C.c_double), ("compile_threads", C.c_int), ("cache_dir", C.c_char_p),
        ("digest_outputs", C.c_int), ("prune_factor", C.c_double), ("isolate", C.c_int),
    ]


class DeviceModel(C.Structure):
    _fields_ = [
        ("name", C.c_char * 64), ("max_work_group_total", C.c_size_t),
        ("max_work_group_dim", C.c_size_t * 3), ("local_mem_bytes", C.c_size_t),
        ("peak_gflops", C.c_double), ("peak_gbs", C.c_double),
    ]


class Row(C.Structure):
    _fields_ = [
        ("step", C.c_size_t), ("status", C.c_int), ("time_ms", C.c_double),
        ("verification", C.c_int), ("best_so_far", C.c_double), ("global_", C.c_size_t * 3),
        ("local", C.c_size_t * 3), ("ndim", C.c_int), ("space_index", C.c_uint64),
        ("device", C.c_int), ("report", VerifyReport),
    ]


class Summary(C.Structure):
    _fields_ = [
        ("rows", C.c_size_t), ("best_index", C.c_longlong), ("best_time_ms", C.c_double),
        ("budget", C.c_size_t), ("unique_evaluations", C.c_size_t),
        ("failed_evaluations", C.c_size_t), ("total_steps", C.c_size_t),
        ("space_size", C.c_ulonglong), ("wall_s", C.c_double), ("configs_per_s", C.c_double),
        ("compile_s", C.c_double), ("device_s", C.c_double),
        ("compile_cache_hits", C.c_size_t), ("kernel_launches", C.c_size_t),
    ]


class StatsSummary(C.Structure):
    _fields_ = [
        ("runs", C.c_size_t), ("mean", C.c_double), ("stddev", C.c_double),
        ("min", C.c_double), ("max", C.c_double), ("space_written", C.c_int),
        ("space_count", C.c_size_t), ("space_min", C.c_double), ("space_mean", C.c_double),
        ("wall_s", C.c_double),
    ]


class RunSummary(C.Structure):
    _fields_ = [("run", C.c_size_t), ("seed", C.c_uint64), ("best_time_ms", C.c_double),
                ("best_config", C.c_char_p)]


class JobInfo(C.Structure):
    _fields_ = [
        ("kernel", C.c_char * 128), ("device", C.c_char * 128), ("backend", C.c_char * 256),
        ("output", C.c_char * 1024), ("is_cuda", C.c_int), ("ndevices", C.c_int),
        ("devices", C.c_int * 64),
    ]


# ---------------------------------------------------------------------------
# library
# ---------------------------------------------------------------------------
_lib = None

# name -> (restype, argtypes)
_P = C.c_void_p
_SIGS = {
    "ktc_abi_version": (C.c_int, []),
    "ktc_status_name": (C.c_char_p, [C.c_int]),
    "ktc_last_error": (C.c_char_p, [_P]),
    "ktc_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ktc_open": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "ktc_close": (None, [_P]),
    "ktc_query_limits": (C.c_int, [_P, C.POINTER(Limits)]),
    "ktc_reset": (C.c_int, [_P]),
    "ktc_compile": (C.c_int, [C.c_char_p, C.POINTER(C.c_char_p), C.c_int, C.POINTER(_P),
                              C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t]),
    "ktc_free_host": (None, [_P]),
    "ktc_codegen_conv": (C.c_int, [C.POINTER(C.c_char_p), C.c_int, C.POINTER(_P),
                                   C.POINTER(C.c_size_t), C.POINTER(_P), C.c_char_p, C.c_size_t]),
    "ktc_codegen_gemm": (C.c_int, [C.POINTER(C.c_char_p), C.c_int, C.POINTER(_P),
                                   C.POINTER(C.c_size_t), C.POINTER(_P), C.c_char_p, C.c_size_t]),
    "ktc_load": (C.c_int, [_P, _P, C.c_size_t, C.c_char_p, C.POINTER(_P)]),
    "ktc_unload": (None, [_P]),
    "ktc_set_symbol": (C.c_int, [_P, C.c_char_p, _P, C.c_size_t]),
    "ktc_alloc": (C.c_int, [_P, C.c_size_t, C.POINTER(C.c_uint64)]),
    "ktc_free": (C.c_int, [_P, C.c_uint64]),
    "ktc_upload": (C.c_int, [_P, C.c_uint64, _P, C.c_size_t]),
    "ktc_upload_pitched": (C.c_int, [_P, C.c_uint64, C.c_size_t, _P, C.c_size_t, C.c_size_t,
                                     C.c_size_t]),
    "ktc_download": (C.c_int, [_P, _P, C.c_uint64, C.c_size_t]),
    "ktc_memset32": (C.c_int, [_P, C.c_uint64, C.c_uint32, C.c_size_t]),
    "ktc_launch_timed": (C.c_int, [_P, _P, C.POINTER(C.c_uint), C.POINTER(C.c_uint), C.c_uint,
                                   C.POINTER(_P), C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "ktc_bind_reference": (C.c_int, [_P, C.c_uint64, C.c_size_t, C.c_int, C.c_double,
                                     C.c_double]),
    "ktc_verify": (C.c_int, [_P, C.c_uint64, C.POINTER(VerifyReport)]),
    "ktc_verify_pair": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_size_t, C.c_int, C.c_double,
                                  C.c_double, C.POINTER(VerifyReport)]),
    "ktc_digest_words": (C.c_uint64, [_P, C.c_size_t]),
    "ktc_digest_hex": (None, [C.c_uint64, C.c_char_p]),
    "ktc_backend_default_options": (None, [C.POINTER(BackendOptions)]),
    "ktc_backend_open": (C.c_int, [C.c_int, C.POINTER(BackendOptions), C.POINTER(_P)]),
    "ktc_backend_close": (None, [_P]),
    "ktc_backend_name": (C.c_char_p, [_P]),
    "ktc_backend_ctx": (_P, [_P]),
    "ktc_backend_evaluate": (C.c_int, [_P, C.POINTER(Request), C.POINTER(Result)]),
    "ktc_backend_prefetch": (C.c_int, [_P, C.POINTER(Request)]),
    "ktc_backend_prefetch_depth": (C.c_size_t, [_P]),
    "ktc_backend_begin_search": (C.c_int, [_P]),
    "ktc_drop_caches": (C.c_int, [C.c_int]),
    "ktc_fill_uniform_f32": (C.c_int, [C.c_uint64, _P, C.c_size_t, C.c_int]),
    "ktc_worker_serve": (C.c_int, [C.c_int, C.c_int]),
    "ktc_backend_set_reference": (C.c_int, [_P, C.POINTER(Request), C.c_int, C.POINTER(_P),
                                            C.POINTER(C.c_size_t), C.POINTER(C.c_int)]),
    "ktc_backend_read_output": (C.c_int, [_P, C.c_int, _P, C.c_size_t]),
    "ktc_backend_read_reference": (C.c_int, [_P, C.POINTER(Request), C.c_int, _P, C.c_size_t,
                                             C.c_char_p]),
    "ktc_device_preset": (C.c_int, [C.c_char_p, C.POINTER(DeviceModel)]),
    "ktc_tuner_create": (C.c_int, [C.POINTER(_P)]),
    "ktc_tuner_destroy": (None, [_P]),
    "ktc_tuner_template_conv": (C.c_int, [_P, C.c_size_t, C.c_size_t, C.c_int, C.c_float,
                                          C.c_uint64]),
    "ktc_tuner_template_gemm": (C.c_int, [_P, C.c_size_t, C.c_size_t, C.c_size_t, C.c_float,
                                          C.c_float, C.c_uint64]),
    "ktc_tuner_template_gemm_tf32": (C.c_int, [_P, C.c_size_t, C.c_size_t, C.c_size_t,
                                               C.c_float, C.c_float, C.c_uint64]),
    "ktc_tuner_add_kernel": (C.c_int, [_P, C.c_char_p, C.c_char_p, C.c_int,
                                       C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "ktc_tuner_add_parameter": (C.c_int, [_P, C.c_char_p, C.POINTER(C.c_longlong), C.c_int]),
    "ktc_tuner_add_constraint": (C.c_int, [_P, C.c_char_p]),
    "ktc_tuner_add_modifier": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_char_p), C.c_int]),
    "ktc_tuner_set_local_memory": (C.c_int, [_P, C.c_char_p]),
    "ktc_tuner_add_argument": (C.c_int, [_P, C.POINTER(Arg)]),
    "ktc_tuner_set_reference_kernel": (C.c_int, [_P, C.c_char_p, C.c_char_p, C.c_int,
                                                 C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "ktc_tuner_set_reference_outputs": (C.c_int, [_P, C.c_int, C.POINTER(C.c_void_p),
                                                  C.POINTER(C.c_size_t), C.POINTER(C.c_int)]),
    "ktc_tuner_set_device": (C.c_int, [_P, C.POINTER(DeviceModel)]),
    "ktc_tuner_set_strategy": (C.c_int, [_P, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_double, C.c_double, C.c_size_t]),
    "ktc_tuner_set_seed": (C.c_int, [_P, C.c_uint64]),
    "ktc_tuner_set_repetitions": (C.c_int, [_P, C.c_int]),
    "ktc_tuner_set_verification": (C.c_int, [_P, C.c_int, C.c_double, C.c_double]),
    "ktc_tuner_set_backend": (C.c_int, [_P, C.c_char_p, C.POINTER(BackendOptions)]),
    "ktc_tuner_set_devices": (C.c_int, [_P, C.POINTER(C.c_int), C.c_int]),
    "ktc_tuner_set_subset": (C.c_int, [_P, C.POINTER(C.c_uint64), C.c_size_t]),
    "ktc_tuner_set_checkpoint": (C.c_int, [_P, C.c_char_p]),
    "ktc_tuner_space_counts": (C.c_int, [_P, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong),
                                         C.POINTER(C.c_ulonglong)]),
    "ktc_tuner_space_config": (C.c_int, [_P, C.c_uint64, C.c_char_p, C.c_size_t]),
    "ktc_tuner_tune": (C.c_int, [_P]),
    "ktc_tuner_summary": (C.c_int, [_P, C.POINTER(Summary)]),
    "ktc_tuner_row": (C.c_int, [_P, C.c_size_t, C.POINTER(Row), C.c_char_p, C.c_size_t,
                                C.c_char_p, C.c_size_t]),
    "ktc_tuner_best": (C.c_int, [_P, C.c_char_p, C.c_size_t, C.POINTER(C.c_double)]),
    "ktc_tuner_write_csv": (C.c_int, [_P, C.c_char_p]),
    "ktc_tuner_write_replay": (C.c_int, [_P, C.c_char_p]),
    "ktc_stats_write": (C.c_int, [C.POINTER(C.c_double), C.c_size_t, C.c_char_p]),
    "ktc_runs_write": (C.c_int, [C.POINTER(RunSummary), C.c_size_t, C.c_char_p]),
    "ktc_tuner_job_info": (C.c_int, [_P, C.POINTER(JobInfo)]),
    "ktc_tuner_stats": (C.c_int, [_P, C.c_size_t, C.c_uint64, C.c_char_p, C.POINTER(StatsSummary)]),
    "ktc_tuner_load_job": (C.c_int, [_P, C.c_char_p, C.c_char_p]),
}


def lib() -> C.CDLL:
    """Loads libktc.so; raises if it is missing (no fallback exists)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (make -C paper_1703_06503_b200). There is no CPU fallback.")
        handle = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def check(code: int) -> None:
    if code != KTC_OK:
        msg = lib().ktc_last_error(None)
        raise KtcError(code, msg.decode() if msg else "")


def last_error() -> str:
    msg = lib().ktc_last_error(None)
    return msg.decode() if msg else ""


def compile_source(src: str, options: list[str]) -> bytes:
    """NVRTC compile for sm_100a (no GPU needed). Raises KtcError with the log."""
    L = lib()
    arr = (C.c_char_p * max(1, len(options)))(*[o.encode() for o in options])
    out = C.c_void_p()
    size = C.c_size_t()
    log = C.create_string_buffer(8192)
    rc = L.ktc_compile(src.encode(), arr, len(options), C.byref(out), C.byref(size), log, 8192)
    if rc != KTC_OK:
        raise KtcError(rc, log.value.decode(errors="replace"))
    data = C.string_at(out, size.value)
    L.ktc_free_host(out)
    return data


def codegen_conv(defines: list[str]) -> tuple[bytes, str]:
    """The conv family's direct PTX generator + ptxas (no GPU): (cubin, ptx)."""
    return _codegen("ktc_codegen_conv", defines)


def codegen_gemm(defines: list[str]) -> tuple[bytes, str]:
    """The SGEMM family's direct PTX generator + ptxas (no GPU): (cubin, ptx)."""
    return _codegen("ktc_codegen_gemm", defines)


def _codegen(fn: str, defines: list[str]) -> tuple[bytes, str]:
    L = lib()
    arr = (C.c_char_p * max(1, len(defines)))(*[d.encode() for d in defines])
    out, ptx = C.c_void_p(), C.c_void_p()
    size = C.c_size_t()
    log = C.create_string_buffer(8192)
    rc = getattr(L, fn)(arr, len(defines), C.byref(out), C.byref(size), C.byref(ptx), log, 8192)
    text = C.string_at(ptx).decode() if ptx.value else ""
    if ptx.value:
        L.ktc_free_host(ptx)
    if rc != KTC_OK:
        raise KtcError(rc, log.value.decode(errors="replace") + "\n" + text[-3000:])
    data = C.string_at(out, size.value)
    L.ktc_free_host(out)
    return data, text


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().ktc_device_count(C.byref(n))
    if rc == 2:  # no driver on this host
        return 0
    check(rc)
    return n.value


os.environ.setdefault("KTC_LIB", str(LIB_PATH))


DROP_COMPILED = 1
DROP_HOST_INPUTS = 2


def drop_caches(compiled: bool = True, host_inputs: bool = True) -> None:
    """Forgets the process-wide compile (cubin) and pinned-input caches, so the
    next fresh job compiles every configuration and materializes its inputs
    on the host again (ktc_drop_caches)."""
    check(lib().ktc_drop_caches((DROP_COMPILED if compiled else 0) |
                                (DROP_HOST_INPUTS if host_inputs else 0)))
