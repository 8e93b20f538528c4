"""ctypes access to the parity checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It never feeds the
product: the product verifies on the device against builtin.cu's reference
kernels, which these oracles prove bit-exact.

  C          oracle/_build/libktune_oracle.so  restatement (ktune_oracle.c)
  reference  oracle/_ref/libktune_ref.so       the reference headers, unmodified
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libktune_oracle.so"
REF_SO = HERE / "_ref" / "libktune_ref.so"
REF_SRC = Path("/root/reference/proj")


class VerifyReport(C.Structure):
    _fields_ = [("pass_", C.c_int), ("max_abs_error", C.c_double), ("max_rel_error", C.c_double),
                ("buffer_index", C.c_size_t), ("element_index", C.c_size_t),
                ("elements_compared", C.c_size_t)]

    def as_dict(self):
        return {"pass": bool(self.pass_), "max_abs_error": self.max_abs_error,
                "max_rel_error": self.max_rel_error, "buffer_index": self.buffer_index,
                "element_index": self.element_index, "elements_compared": self.elements_compared}


def build(reference: bool | None = None) -> None:
    """Builds the C oracle, and oracle/_ref when the reference tree exists."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if reference is None:
        reference = REF_SRC.exists()
    if reference:
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


_oracle = None
_ref = None


def oracle_lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            build(reference=False)
        L = C.CDLL(str(ORACLE_SO))
        P = C.c_void_p
        L.ko_materialize_f32.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_size_t, P]
        L.ko_materialize_i32.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_size_t, P]
        L.ko_digest_words.argtypes = [P, C.c_size_t]
        L.ko_digest_words.restype = C.c_uint64
        L.ko_conv_apply.argtypes = [P, P, C.c_size_t, C.c_size_t, C.c_int, C.c_float, P, C.c_int]
        L.ko_gemm_apply.argtypes = [P, P, P, C.c_size_t, C.c_size_t, C.c_size_t, C.c_float,
                                    C.c_float, P, C.c_int]
        L.ko_verify_init.argtypes = [C.POINTER(VerifyReport)]
        L.ko_verify_f32.argtypes = [C.POINTER(VerifyReport), C.c_size_t, P, P, C.c_size_t,
                                    C.c_double, C.c_double]
        L.ko_verify_i32.argtypes = [C.POINTER(VerifyReport), C.c_size_t, P, P, C.c_size_t]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return REF_SO.exists()


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(str(REF_SO))
        P = C.c_void_p
        L.kr_last_error.restype = C.c_char_p
        L.kr_materialize_f32.argtypes = [C.c_char_p, C.c_size_t, P]
        L.kr_conv_reference.argtypes = [C.c_size_t, C.c_size_t, C.c_int, C.c_float, C.c_uint64, P]
        L.kr_gemm_reference.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.c_float, C.c_float,
                                        C.c_uint64, P]
        L.kr_conv_apply.argtypes = [P, P, C.c_size_t, C.c_size_t, C.c_int, C.c_float, P]
        L.kr_gemm_apply.argtypes = [P, P, P, C.c_size_t, C.c_size_t, C.c_size_t, C.c_float,
                                    C.c_float, P]
        L.kr_digest_f32.argtypes = [P, C.c_size_t]
        L.kr_digest_f32.restype = C.c_uint64
        L.kr_verify_f32.argtypes = [P, P, C.c_size_t, C.c_double, C.c_double,
                                    C.POINTER(VerifyReport)]
        L.kr_job_counts.argtypes = [C.c_char_p] + [C.POINTER(C.c_ulonglong)] * 3
        L.kr_job_enumerate.argtypes = [C.c_char_p, C.c_char_p]
        L.kr_job_price_table.argtypes = [C.c_char_p, C.c_char_p]
        L.kr_job_run.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(C.c_longlong),
                                 C.POINTER(C.c_double)]
        L.kr_job_stats.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.c_uint64, C.c_char_p]
        L.kr_job_throughput.argtypes = [C.c_char_p, C.c_int, C.c_size_t, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.POINTER(C.c_size_t)]
        _ref = L
    return _ref


def _ref_check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(ref_lib().kr_last_error().decode())


# ------------------------------------------------------------------ C oracle
FILL = {"none": 0, "constant": 1, "ramp": 2, "uniform": 3}


def materialize(fill: str, length: int, dtype=np.float32) -> np.ndarray:
    kind, const, seed = 0, 0.0, 0
    if fill == "ramp":
        kind = 2
    elif fill.startswith("constant:"):
        kind, const = 1, float(fill.split(":", 1)[1])
    elif fill.startswith("uniform:"):
        kind, seed = 3, int(fill.split(":", 1)[1])
    out = np.empty(length, dtype=dtype)
    fn = oracle_lib().ko_materialize_f32 if dtype == np.float32 else oracle_lib().ko_materialize_i32
    fn(kind, const, seed & 0xFFFFFFFFFFFFFFFF, length, out.ctypes.data)
    return out


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return f"{oracle_lib().ko_digest_words(a.ctypes.data, a.size):016x}"


def threads() -> int:
    return max(1, os.cpu_count() or 1)


def conv_apply(image, taps, x, y, f, w=1.0, nthreads=None) -> np.ndarray:
    out = np.empty(x * y, dtype=np.float32)
    oracle_lib().ko_conv_apply(np.ascontiguousarray(image, np.float32).ctypes.data,
                               np.ascontiguousarray(taps, np.float32).ctypes.data, x, y, f, w,
                               out.ctypes.data, nthreads or threads())
    return out


def gemm_apply(a, b, c, m, n, k, alpha=1.0, beta=0.0, nthreads=None) -> np.ndarray:
    out = np.empty(m * n, dtype=np.float32)
    oracle_lib().ko_gemm_apply(np.ascontiguousarray(a, np.float32).ctypes.data,
                               np.ascontiguousarray(b, np.float32).ctypes.data,
                               np.ascontiguousarray(c, np.float32).ctypes.data, m, n, k, alpha,
                               beta, out.ctypes.data, nthreads or threads())
    return out


def conv_reference(x, y, f, w=1.0, seed=2026, nthreads=None) -> np.ndarray:
    """conv_reference (landscapes.hpp:146-155) on the C oracle."""
    image = materialize(f"uniform:{seed}", (x + f - 1) * (y + f - 1))
    taps = materialize(f"uniform:{seed ^ 0x9E3779B97F4A7C15}", f * f)
    return conv_apply(image, taps, x, y, f, w, nthreads)


def gemm_reference(m, n, k, alpha=1.0, beta=0.0, seed=2026, nthreads=None) -> np.ndarray:
    a = materialize(f"uniform:{seed}", k * m)
    b = materialize(f"uniform:{seed ^ 0x9E3779B97F4A7C15}", k * n)
    c = materialize(f"uniform:{seed ^ 0xC2B2AE3D27D4EB4F}", m * n)
    return gemm_apply(a, b, c, m, n, k, alpha, beta, nthreads)


def verify(cand: np.ndarray, ref: np.ndarray, rel=1e-4, abs_=1e-6) -> dict:
    rep = VerifyReport()
    oracle_lib().ko_verify_init(C.byref(rep))
    if cand.dtype == np.float32:
        oracle_lib().ko_verify_f32(C.byref(rep), 0, cand.ctypes.data, ref.ctypes.data, cand.size,
                                   rel, abs_)
    else:
        oracle_lib().ko_verify_i32(C.byref(rep), 0, cand.ctypes.data, ref.ctypes.data, cand.size)
    return rep.as_dict()


# ---------------------------------------------------------- reference (_ref)
def ref_conv_reference(x, y, f, w=1.0, seed=2026) -> np.ndarray:
    out = np.empty(x * y, dtype=np.float32)
    _ref_check(ref_lib().kr_conv_reference(x, y, f, w, seed, out.ctypes.data))
    return out


def ref_gemm_reference(m, n, k, alpha=1.0, beta=0.0, seed=2026) -> np.ndarray:
    out = np.empty(m * n, dtype=np.float32)
    _ref_check(ref_lib().kr_gemm_reference(m, n, k, alpha, beta, seed, out.ctypes.data))
    return out


def ref_verify(cand, ref, rel=1e-4, abs_=1e-6) -> dict:
    rep = VerifyReport()
    _ref_check(ref_lib().kr_verify_f32(cand.ctypes.data, ref.ctypes.data, cand.size, rel, abs_,
                                       C.byref(rep)))
    return rep.as_dict()


def ref_job_counts(job_json: str) -> tuple[int, int, int]:
    a, b, c = C.c_ulonglong(), C.c_ulonglong(), C.c_ulonglong()
    _ref_check(ref_lib().kr_job_counts(job_json.encode(), C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def ref_job_enumerate(job_json: str, path: str) -> list[str]:
    _ref_check(ref_lib().kr_job_enumerate(job_json.encode(), str(path).encode()))
    return Path(path).read_text().splitlines()


def ref_job_price_table(job_json: str, path: str) -> None:
    _ref_check(ref_lib().kr_job_price_table(job_json.encode(), str(path).encode()))


def ref_job_run(job_json: str, base_dir: str, out_csv: str) -> tuple[int, float]:
    bi, bt = C.c_longlong(), C.c_double()
    _ref_check(ref_lib().kr_job_run(job_json.encode(), str(base_dir).encode(),
                                    str(out_csv).encode(), C.byref(bi), C.byref(bt)))
    return bi.value, bt.value


def ref_job_stats(job_json: str, base_dir: str, runs: int, base_seed: int, out_csv: str) -> None:
    _ref_check(ref_lib().kr_job_stats(job_json.encode(), str(base_dir).encode(), runs, base_seed,
                                      str(out_csv).encode()))


def ref_job_throughput(job_json: str, nthreads: int, per_thread: int) -> dict:
    rate, wall, n = C.c_double(), C.c_double(), C.c_size_t()
    _ref_check(ref_lib().kr_job_throughput(job_json.encode(), nthreads, per_thread,
                                           C.byref(rate), C.byref(wall), C.byref(n)))
    return {"configs_per_s": rate.value, "wall_s": wall.value, "evaluated": n.value}


def ref_conv_apply(image, taps, x, y, f, w=1.0) -> np.ndarray:
    """The reference's conv_apply (landscapes.hpp:120-143) as-is, one thread."""
    out = np.empty(x * y, dtype=np.float32)
    _ref_check(ref_lib().kr_conv_apply(np.ascontiguousarray(image, np.float32).ctypes.data,
                                       np.ascontiguousarray(taps, np.float32).ctypes.data,
                                       x, y, f, w, out.ctypes.data))
    return out


def ref_gemm_apply(a, b, c, m, n, k, alpha=1.0, beta=0.0) -> np.ndarray:
    """The reference's gemm_apply (landscapes.hpp:293-312) as-is, one thread."""
    out = np.empty(m * n, dtype=np.float32)
    _ref_check(ref_lib().kr_gemm_apply(np.ascontiguousarray(a, np.float32).ctypes.data,
                                       np.ascontiguousarray(b, np.float32).ctypes.data,
                                       np.ascontiguousarray(c, np.float32).ctypes.data,
                                       m, n, k, alpha, beta, out.ctypes.data))
    return out
