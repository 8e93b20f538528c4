"""CLTune-named tuner API over libktc (include/ktc.h, layer 3).

    tuner = Tuner(devices=[0])
    tuner.AddKernel("copy.cu", "copy", [2048], [1])
    tuner.AddParameter("WPT", [1, 2, 4])
    tuner.DivGlobalSize(["WPT"])
    tuner.AddArgumentInput(2048, fill="uniform:3")
    tuner.AddArgumentOutput(2048)
    tuner.UseFullSearch()
    tuner.Tune()
    config, ms = tuner.GetBestResult()

The case studies come ready-made: ``Tuner.conv(x, y, filter)`` and
``Tuner.gemm(m, n, k)`` (templates of the reference's job format, verified
on the device against their bit-exact device reference).  Every call lands
in native code; there is no Python evaluation path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Iterable, Sequence

from . import _ktc as K


def _arr(ctype, values):
    values = list(values)
    return (ctype * max(1, len(values)))(*values), len(values)


@dataclass
class TuningRowView:
    step: int
    config: str
    status: str
    time_ms: float | None
    verified: str
    best_so_far: float | None
    global_size: tuple
    local_size: tuple
    space_index: int
    device: int
    report: dict
    message: str


class Tuner:
    """The CLTune tuner backed by the ktb search layer."""

    def __init__(self, device: str | None = "B200", backend: str = "cuda",
                 devices: Sequence[int] = (0,), flush_l2: bool = True, warmup: int = 1,
                 compile_threads: int = 0, cache_dir: str | None = None):
        self._lib = K.lib()
        h = C.c_void_p()
        K.check(self._lib.ktc_tuner_create(C.byref(h)))
        self._h = h
        self._opts = K.BackendOptions()
        self._lib.ktc_backend_default_options(C.byref(self._opts))
        self._opts.flush_l2 = 1 if flush_l2 else 0
        self._opts.warmup = warmup
        self._opts.compile_threads = compile_threads
        self._cache_dir = cache_dir.encode() if cache_dir else None
        self._opts.cache_dir = self._cache_dir
        self._backend = backend
        K.check(self._lib.ktc_tuner_set_backend(self._h, backend.encode(), C.byref(self._opts)))
        self.SetDevices(devices)
        if device is not None:
            self.SetDevice(device)

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.ktc_tuner_destroy(self._h)
            self._h = None

    # ---------------------------------------------------------------- setup
    @classmethod
    def conv(cls, x=8192, y=4096, filter=7, weight=1.0, seed=2026, **kw) -> "Tuner":
        t = cls(**kw)
        K.check(t._lib.ktc_tuner_template_conv(t._h, x, y, filter, weight, seed))
        return t

    @classmethod
    def gemm(cls, m=2048, n=2048, k=2048, alpha=1.0, beta=0.0, seed=2026, tf32=False,
             **kw) -> "Tuner":
        t = cls(**kw)
        fn = t._lib.ktc_tuner_template_gemm_tf32 if tf32 else t._lib.ktc_tuner_template_gemm
        K.check(fn(t._h, m, n, k, alpha, beta, seed))
        return t

    @classmethod
    def from_job(cls, json_text: str, base_dir: str = ".", **kw) -> "Tuner":
        t = cls(device=None, **kw)
        K.check(t._lib.ktc_tuner_load_job(t._h, json_text.encode(), base_dir.encode()))
        return t

    def SetDevice(self, device) -> None:
        """A preset name ("B200", "K40m", ...), "cuda:<ordinal>", or a dict."""
        dm = K.DeviceModel()
        if isinstance(device, str):
            K.check(self._lib.ktc_device_preset(device.encode(), C.byref(dm)))
        else:
            dm.name = device["name"].encode()
            dm.max_work_group_total = device.get("max_work_group_total", 1024)
            dims = device.get("max_work_group_dim", (1024, 1024, 64))
            for i in range(3):
                dm.max_work_group_dim[i] = dims[i]
            dm.local_mem_bytes = device.get("local_mem_bytes", 49152)
            dm.peak_gflops = device.get("peak_gflops", 0.0)
            dm.peak_gbs = device.get("peak_gbs", 0.0)
        K.check(self._lib.ktc_tuner_set_device(self._h, C.byref(dm)))

    def SetDevices(self, ordinals: Iterable[int]) -> None:
        arr, n = _arr(C.c_int, ordinals)
        K.check(self._lib.ktc_tuner_set_devices(self._h, arr, n))

    def AddKernel(self, source_ref: str, name: str, global_size: Sequence[int],
                  local_size: Sequence[int]) -> None:
        g, n = _arr(C.c_size_t, global_size)
        l, _ = _arr(C.c_size_t, local_size)
        K.check(self._lib.ktc_tuner_add_kernel(self._h, source_ref.encode(), name.encode(), n, g, l))

    def AddParameter(self, name: str, values: Sequence[int]) -> None:
        arr, n = _arr(C.c_longlong, values)
        K.check(self._lib.ktc_tuner_add_parameter(self._h, name.encode(), arr, n))

    def AddConstraint(self, expr: str) -> None:
        K.check(self._lib.ktc_tuner_add_constraint(self._h, expr.encode()))

    def _modifier(self, target: int, op: int, factors: Sequence[str]) -> None:
        arr, n = _arr(C.c_char_p, [str(f).encode() for f in factors])
        K.check(self._lib.ktc_tuner_add_modifier(self._h, target, op, arr, n))

    def MulGlobalSize(self, factors): self._modifier(0, 0, factors)
    def DivGlobalSize(self, factors): self._modifier(0, 1, factors)
    def MulLocalSize(self, factors): self._modifier(1, 0, factors)
    def DivLocalSize(self, factors): self._modifier(1, 1, factors)

    def SetLocalMemoryUsage(self, expr: str) -> None:
        K.check(self._lib.ktc_tuner_set_local_memory(self._h, expr.encode()))

    def _argument(self, role, etype, length=0, value=0.0, fill="none"):
        self._fill_keep = getattr(self, "_fill_keep", [])
        f = fill.encode()
        self._fill_keep.append(f)
        a = K.Arg(role, etype, length, float(value), f)
        K.check(self._lib.ktc_tuner_add_argument(self._h, C.byref(a)))

    def AddArgumentInput(self, length: int, fill: str = "none", dtype: str = "f32"):
        self._argument(K.ARG_INPUT, K.I32 if dtype == "i32" else K.F32, length, 0.0, fill)

    def AddArgumentOutput(self, length: int, fill: str = "none", dtype: str = "f32"):
        self._argument(K.ARG_OUTPUT, K.I32 if dtype == "i32" else K.F32, length, 0.0, fill)

    def AddArgumentScalar(self, value, dtype: str = "i32"):
        self._argument(K.ARG_SCALAR, K.I32 if dtype == "i32" else K.F32, 0, value, "")

    def SetReference(self, source_ref: str, name: str, global_size: Sequence[int],
                     local_size: Sequence[int]) -> None:
        """CLTune SetReference: a reference kernel (no tuning parameters), run
        once on the device over the same arguments when Tune() starts; every
        configuration is then verified on the device against its outputs."""
        g, n = _arr(C.c_size_t, global_size)
        l, _ = _arr(C.c_size_t, local_size)
        K.check(self._lib.ktc_tuner_set_reference_kernel(self._h, source_ref.encode(),
                                                         name.encode(), n, g, l))

    def SetReferenceOutputs(self, outputs) -> None:
        """Host reference outputs (numpy arrays, one per output argument)."""
        import numpy as np

        arrs = []
        for o in outputs:
            o = np.asarray(o)
            arrs.append(np.ascontiguousarray(o, dtype=np.int32 if o.dtype == np.int32 else np.float32))
        self._ref_keep = arrs
        ptrs = (C.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])
        lens = (C.c_size_t * max(1, len(arrs)))(*[a.size for a in arrs])
        types = (C.c_int * max(1, len(arrs)))(*[K.I32 if a.dtype == np.int32 else K.F32
                                                 for a in arrs])
        K.check(self._lib.ktc_tuner_set_reference_outputs(self._h, len(arrs), ptrs, lens, types))

    # ------------------------------------------------------------- strategy
    def UseFullSearch(self):
        K.check(self._lib.ktc_tuner_set_strategy(self._h, K.SEARCH_FULL, 1.0, 4.0, 0.4, 0.0, 0.4, 3))

    def UseRandomSearch(self, fraction: float):
        K.check(self._lib.ktc_tuner_set_strategy(self._h, K.SEARCH_RANDOM, fraction, 4.0, 0.4, 0.0,
                                                 0.4, 3))

    def UseAnnealing(self, fraction: float, temperature: float = 4.0):
        K.check(self._lib.ktc_tuner_set_strategy(self._h, K.SEARCH_ANNEALING, fraction,
                                                 temperature, 0.4, 0.0, 0.4, 3))

    def UsePSO(self, fraction: float, swarm: int = 3, alpha: float = 0.4, beta: float = 0.0,
               gamma: float = 0.4):
        K.check(self._lib.ktc_tuner_set_strategy(self._h, K.SEARCH_PSO, fraction, 4.0, alpha, beta,
                                                 gamma, swarm))

    def SetSeed(self, seed: int): K.check(self._lib.ktc_tuner_set_seed(self._h, seed))
    def SetRepetitions(self, n: int): K.check(self._lib.ktc_tuner_set_repetitions(self._h, n))

    def SetVerification(self, verify: bool = True, rel_tol: float = 1e-4, abs_tol: float = 1e-6):
        K.check(self._lib.ktc_tuner_set_verification(self._h, int(verify), rel_tol, abs_tol))

    def SetPruning(self, factor: float):
        """Early-out for device-bound searches (ktc.h prune_factor; 0 = off): a
        configuration whose first flushed launch exceeds `factor` x the best
        verified time seen so far is timed once instead of best-of-N."""
        self._opts.prune_factor = float(factor)
        K.check(self._lib.ktc_tuner_set_backend(self._h, self._backend.encode(),
                                                C.byref(self._opts)))

    def SetSubset(self, indices: Sequence[int]):
        arr, n = _arr(C.c_uint64, indices)
        K.check(self._lib.ktc_tuner_set_subset(self._h, arr, n))

    def SetCheckpoint(self, path: str | None):
        """Resume file for long full/random searches (replay CSV format)."""
        K.check(self._lib.ktc_tuner_set_checkpoint(self._h, (path or "").encode()))

    # ---------------------------------------------------------------- space
    def space_counts(self) -> tuple[int, int, int]:
        raw, con, val = C.c_ulonglong(), C.c_ulonglong(), C.c_ulonglong()
        K.check(self._lib.ktc_tuner_space_counts(self._h, C.byref(raw), C.byref(con), C.byref(val)))
        return raw.value, con.value, val.value

    def space_config(self, index: int) -> str:
        buf = C.create_string_buffer(1024)
        K.check(self._lib.ktc_tuner_space_config(self._h, index, buf, 1024))
        return buf.value.decode()

    # ------------------------------------------------------------------ run
    def Tune(self) -> dict:
        K.check(self._lib.ktc_tuner_tune(self._h))
        return self.summary()

    def summary(self) -> dict:
        s = K.Summary()
        K.check(self._lib.ktc_tuner_summary(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in K.Summary._fields_}

    def GetBestResult(self) -> tuple[str, float]:
        buf = C.create_string_buffer(1024)
        t = C.c_double()
        K.check(self._lib.ktc_tuner_best(self._h, buf, 1024, C.byref(t)))
        return buf.value.decode(), t.value

    def rows(self) -> list[TuningRowView]:
        n = self.summary()["rows"]
        out = []
        r = K.Row()
        cfg = C.create_string_buffer(1024)
        msg = C.create_string_buffer(1024)
        for i in range(n):
            K.check(self._lib.ktc_tuner_row(self._h, i, C.byref(r), cfg, 1024, msg, 1024))
            nan = lambda v: None if math.isnan(v) else v  # noqa: E731
            out.append(TuningRowView(
                step=r.step, config=cfg.value.decode(), status=K.STATUS_NAMES[r.status],
                time_ms=nan(r.time_ms), verified=K.VERIFY_NAMES[r.verification],
                best_so_far=nan(r.best_so_far),
                global_size=tuple(r.global_[:r.ndim]), local_size=tuple(r.local[:r.ndim]),
                space_index=r.space_index, device=r.device, report=r.report.as_dict(),
                message=msg.value.decode()))
        return out

    # CLTune reporting names
    def SetNumRuns(self, n: int):
        """CLTune's name for the timed repetitions per configuration (best of n)."""
        self.SetRepetitions(n)

    def PrintToScreen(self) -> None:
        """CLTune PrintToScreen: one line per evaluated configuration, then the best."""
        for r in self.rows():
            t = f"{r.time_ms:10.4f} ms" if r.time_ms is not None else f"{r.status:>13s}"
            print(f"[{r.step:6d}] {t}  {r.verified:8s}  {r.config}")
        try:
            cfg, ms = self.GetBestResult()
            print(f"[ best ] {ms:10.4f} ms  {cfg}")
        except K.KtcError:
            print("[ best ] none (no successful configuration)")

    def PrintToFile(self, path: str) -> None:
        """CLTune PrintToFile: the results table as CSV (the reference's format)."""
        self.write_csv(path)

    def write_csv(self, path: str) -> None:
        K.check(self._lib.ktc_tuner_write_csv(self._h, str(path).encode()))

    def write_replay(self, path: str) -> None:
        K.check(self._lib.ktc_tuner_write_replay(self._h, str(path).encode()))

    def Stats(self, runs: int, base_seed: int = 1, out: str = "stats.csv") -> dict:
        """`ktune stats` (tools/ktune.cpp:120-258): `runs` searches with seeds
        base_seed.., run as replicas over this tuner's devices; writes `out`,
        `<stem>_runs<ext>` and (spaces <= 100,000) `<stem>_space<ext>`."""
        s = K.StatsSummary()
        K.check(self._lib.ktc_tuner_stats(self._h, runs, base_seed, str(out).encode(), C.byref(s)))
        return {f: getattr(s, f) for f, _ in K.StatsSummary._fields_}


def parse_canonical(text: str) -> dict:
    return {k: int(v) for k, v in (kv.split("=") for kv in text.split(";"))}
