"""Benchmark of the B200 tuning hot path (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (BASELINE.json configs[0], the reference's own CPU-runnable case):
tuning the paper's 2D-convolution space for a 3x3 filter on an 8192x4096
fp32 image, every configuration's output verified against the reference
output.  A *step* is one chunk of configurations per GPU (weak scaling; the
chunk depends on K and W only): each configuration is compiled for sm_100a
(direct PTX generation + in-process ptxas), loaded, launched once to warm up
and 3 timed times (CUDA events, L2 flushed before each, best of 3) and its
output verified on the device against the bit-exact device reference.

  --gpus N   under torchrun: one process per GPU (LOCAL_RANK); launched
             plainly: one process driving N device workers over one shared
             compile pool (workers share GPUs when fewer than N exist)
  value      configurations evaluated per second, all GPUs (inputs resident
             in HBM; cold compile cache: every configuration compiled for the
             first time inside the timed region); max over ranks
  e2e        the same metric through the public API (Tuner), cold: compile
             cache and pinned host inputs dropped, one fresh job per GPU per
             step (host materializes the recipes, H2D image + taps, D2H rows)
  configs4_gemm4096   BASELINE configs[4]: device-bound tuning throughput on
             a fixed seeded sample of the 4096^3 SGEMM space
  tuned      per-filter best configuration (3..11, configs[1]), the SGEMM
             winners (configs[2]-[4] sizes) and the TF32 variant re-timed:
             GFLOPS, GB/s, roofline fractions
  roofline   the best 3x3 convolution kernel (HBM-bound) against the measured
             copy bandwidth (MEASURED_PEAKS.json), ncu DRAM traffic
  cpu_baseline          the reference's own tuner loop on this host's cores
  cpu_baseline_kernels  the reference's conv_apply / gemm_apply on one core
             and the bit-identical restatement on all cores (GFLOPS)
  --impl reference      the reference's CPU tuner alone (same metric string)
"""
from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

X, Y, F = 8192, 4096, 3
CHUNK = 48
MAX_GPUS = 8          # chunks are sized so the largest scaling run has distinct units
REF_PER_STEP = 2      # reference arm: configurations per host thread per step
GEMM_PER_GPU = 96     # configs[4] block: 4096^3 configurations per GPU
ROW_BYTES = 256       # a result row read back to the host (ktc_row + strings), approx.
CONV_BYTES = 2 * X * Y * 4  # landscapes.hpp:174, per launch
# The SAME metric string in both arms (the driver divides their values).
METRIC = "conv2d 3x3 8192x4096 fp32 tuning throughput (configs evaluated/s, outputs verified)"
WORKLOAD = ("configs[0]: conv2d 3x3 on 8192x4096 fp32, tuning over the paper's conv space, "
            "every configuration's output verified against the reference output")


def conv_flops(f: int) -> float:
    return (1 + 2 * f * f) * X * Y


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


def fp32_peak_gflops(sm_count=148, mhz=1965.0) -> float:
    return sm_count * 128 * 2 * mhz / 1e3


def tf32_peak_gflops() -> float:
    """Dense TF32 peak: MEASURED_PEAKS.json has no TF32 figure, so the
    B200_PROFILING.md fallback (1.1 PFLOP/s dense) is the denominator."""
    return 1.1e6


def tf32_half_bf16_gflops() -> float:
    """Half the measured bf16 burst (UMMA issues TF32 at half the bf16 rate):
    a second, measured reference point reported next to the fallback peak."""
    p = ROOT / "MEASURED_PEAKS.json"
    bf16 = json.loads(p.read_text()).get("bf16_tflops", 1637.5) if p.exists() else 1637.5
    return bf16 * 1e3 / 2


# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clocks + throttle reasons during the timed region (NVML every 20 ms,
    nvidia-smi as the fallback)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(gpu))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mask = get(h)
        self.samples.append((float(sm), float(mx), {n for n, bit in self.REASONS if mask & bit}))

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            v = [x.strip() for x in out.stdout.strip().split(",")]
            names = [n for n, _ in self.REASONS]
            self.samples.append((float(v[1]), float(v[2]),
                                 {names[i] for i in range(4) if len(v) > 5 + i and
                                  v[5 + i].lower() == "active"}))

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self._sample_nvml()
                else:
                    self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.02 if self._nvml else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [s[0] for s in self.samples]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))),
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


# ---------------------------------------------------------------------------
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def reduce_over_ranks(world, v: float, op: str) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def gather_objects(world, obj):
    if world == 1:
        return [obj]
    import torch.distributed as dist

    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def conv_job_json() -> str:
    return json.dumps({"template": "conv", "problem": {"x": X, "y": Y, "filter": F},
                       "device": {"name": "B200", "max_work_group_total": 1024,
                                  "max_work_group_dim": [1024, 1024, 64],
                                  "local_mem_bytes": 232448},
                       "backend": {"kind": "synthetic", "model": "conv-like"},
                       "verify": True, "seed": 1})


def chunk_for(valid: int, steps: int, warmup: int, requested: int) -> int:
    """Configurations per GPU per step.  Every configuration of a run
    (warm-up and timed steps, every GPU up to MAX_GPUS) is distinct, so no
    compile is served from the cache inside a timed region; the chunk depends
    only on K and W, never on N, so per-GPU work is the same at every N."""
    return max(1, min(requested, valid // (MAX_GPUS * (warmup + steps))))


# ---------------------------------------------------------------------------
def reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU tuner on this host.

    Each host thread runs ONE reference run_tuning (tuner.hpp:194-323) with
    its synthetic backend and verify=true -- i.e. the reference's CPU
    implementation of the kernel (conv_apply, landscapes.hpp:120-143) prices
    and produces every configuration's output, verified against its own
    reference -- over steps x REF_PER_STEP random configurations, so the
    job-level reference computation (tuner.hpp:216-228) is amortized over the
    whole timed region exactly as our arm's job setup is."""
    if rank != 0:
        return
    from oracle import oracle as O  # the reference, compiled under oracle/_ref

    job = conv_job_json()
    cores = host_cores()
    for _ in range(min(1, args.warmup)):
        O.ref_job_throughput(job, cores, 1)
    per_thread = args.steps * REF_PER_STEP
    r = O.ref_job_throughput(job, cores, per_thread)
    value = r["evaluated"] / r["wall_s"]
    sample = (f"{cores} threads x one run_tuning each over {per_thread} random configurations "
              f"({REF_PER_STEP} per step x {args.steps} steps; synthetic backend, verify=true: "
              f"CPU conv_apply + verify_outputs per configuration), {r['wall_s']:.1f} s")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "configs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * r["wall_s"] / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: the reference's fill recipes (mt19937_64, seed 2026), no datasets",
        "config": {"workload": WORKLOAD + " -- reference CPU tuner (oracle/_ref, unmodified "
                               "headers)", "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "configs/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "configs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline_configs() -> dict:
    """Our arm's reported CPU baseline: the reference tuner loop, bounded."""
    from oracle import oracle as O

    if not O.ref_available():
        return {"value": None, "unit": "configs/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    cores = host_cores()
    r = O.ref_job_throughput(conv_job_json(), cores, 16)
    return {"value": r["configs_per_s"], "unit": "configs/s", "cores": cores, "kind": "reference",
            "sample": f"{r['evaluated']} configurations: {cores} threads x one run_tuning of 16 "
                      f"(reference tuner, synthetic backend, verify=true -> CPU conv_apply per "
                      f"configuration), {r['wall_s']:.1f} s"}


def cpu_baseline_kernels() -> dict:
    """CPU implementations of the tuned kernels on this host:
    the reference's conv_apply / gemm_apply as-is on ONE core (oracle/_ref),
    and the bit-identical restatement (oracle/ktune_oracle.c) on all cores."""
    from oracle import oracle as O

    cores = host_cores()
    out = {"cores_all": cores, "conv": {}, "gemm": {}}
    for f in (3, 5, 7, 9, 11):
        img = O.materialize("uniform:2026", (X + f - 1) * (Y + f - 1))
        taps = O.materialize(f"uniform:{2026 ^ 0x9E3779B97F4A7C15}", f * f)
        e = {}
        if O.ref_available():
            t0 = time.perf_counter()
            O.ref_conv_apply(img, taps, X, Y, f)
            e["reference_1core_gflops"] = conv_flops(f) / (time.perf_counter() - t0) / 1e9
        t0 = time.perf_counter()
        O.conv_apply(img, taps, X, Y, f, nthreads=cores)
        e["restated_all_cores_gflops"] = conv_flops(f) / (time.perf_counter() - t0) / 1e9
        out["conv"][str(f)] = e
    if O.ref_available():
        m = 1024  # 2048^3 takes ~170 s on one core; the per-element loop is the same
        a = O.materialize("uniform:2026", m * m)
        t0 = time.perf_counter()
        O.ref_gemm_apply(a, a, a, m, m, m)
        out["gemm"]["reference_1core_gflops"] = 2.0 * m ** 3 / (time.perf_counter() - t0) / 1e9
        out["gemm"]["reference_1core_sample"] = f"gemm_apply {m}^3"
    for m in (2048, 4096):
        a = O.materialize("uniform:2026", m * m)
        t0 = time.perf_counter()
        O.gemm_apply(a, a, a, m, m, m, nthreads=cores)
        out["gemm"][f"restated_all_cores_{m}_gflops"] = 2.0 * m ** 3 / (time.perf_counter() - t0) / 1e9
    return out


def tuned_table() -> dict:
    p = ROOT / "tuned" / "b200_winners.json"
    return json.loads(p.read_text()) if p.exists() else {}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunk", type=int, default=CHUNK)
    ap.add_argument("--gemm-per-gpu", type=int, default=GEMM_PER_GPU,
                    help="configs[4] scaling block: 4096^3 configurations per GPU (0 = skip)")
    ap.add_argument("--no-tuned", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baselines")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return

    import paper_1703_06503_b200 as pkg

    # Devices of this process: one per rank under torchrun; all N in one
    # process (one shared compile pool) when launched plainly with --gpus N.
    # With fewer physical GPUs than N (a 1-GPU test box) workers share them.
    ndev = max(1, pkg.device_count())
    if world > 1:
        devices = [local % ndev]
    else:
        devices = [i % ndev for i in range(max(1, args.gpus))]
    slots_here = len(devices)
    first_slot = sum(gather_objects(world, slots_here)[:rank])
    n_gpus = reduce_over_ranks(world, float(slots_here), "sum")
    cores = host_cores()
    threads = max(1, cores // world)

    def tuner_conv():
        t = pkg.Tuner.conv(X, Y, F, devices=devices, compile_threads=threads)
        t.SetVerification(True)
        t.SetRepetitions(3)
        return t

    tuner = tuner_conv()
    _, _, valid = tuner.space_counts()
    order = list(range(valid))
    random.Random(2026).shuffle(order)  # fixed, seeded visit order for every N
    chunk = chunk_for(valid, args.steps, args.warmup, args.chunk)

    def units(step: int) -> list:
        out = []
        for g in range(first_slot, first_slot + slots_here):
            base = (step * MAX_GPUS + g) * chunk
            out += [order[base + j] for j in range(chunk)]
        return out

    # warm-up (different configurations than the timed steps)
    for s in range(args.warmup):
        tuner.SetSubset(units(s))
        tuner.Tune()
    # The K timed steps run as ONE pipelined stream (the way a search runs:
    # the compile pool keeps working across step boundaries).
    timed_units = []
    for s in range(args.warmup, args.warmup + args.steps):
        timed_units += units(s)
    tuner.SetSubset(timed_units)
    barrier(world)
    with ClockSampler(devices[0]) as clocks:
        t0 = time.perf_counter()
        summ = tuner.Tune()
        elapsed = time.perf_counter() - t0
    barrier(world)
    all_rows = tuner.rows()
    t_max = reduce_over_ranks(world, elapsed, "max")
    evaluated = reduce_over_ranks(world, float(len(all_rows)), "sum")
    launches = int(reduce_over_ranks(world, float(summ["kernel_launches"]), "sum"))
    value = evaluated / t_max
    ok = int(reduce_over_ranks(world, float(sum(1 for r in all_rows if r.status == "ok" and
                                                 r.verified == "pass")), "sum"))
    failed_verify = int(reduce_over_ranks(world, float(sum(1 for r in all_rows
                                                           if r.verified == "fail")), "sum"))
    per_device = {}
    for r in all_rows:
        per_device[r.device] = per_device.get(r.device, 0) + 1
    gpus_active = len({(rank, d) for d in per_device}) if world == 1 else \
        int(reduce_over_ranks(world, float(len(per_device)), "sum"))

    # warm compile cache: the same units again (every cubin cached) -> the
    # device-bound rate
    barrier(world)
    t0 = time.perf_counter()
    tuner.Tune()
    warm = reduce_over_ranks(world, time.perf_counter() - t0, "max")
    value_warm = evaluated / warm
    del tuner

    # e2e through the public API, cold: compile cache and pinned host inputs
    # dropped, then one fresh job (Tuner) per step -- host materialization of
    # the recipes, H2D of image + taps, compile, launch, verify, D2H of the
    # step's rows -- over the same K x chunk configurations per GPU.
    pkg.drop_caches(compiled=True, host_inputs=True)
    barrier(world)
    t0 = time.perf_counter()
    e2e_rows = 0
    e2e_ok = 0
    for s in range(args.warmup, args.warmup + args.steps):
        pkg.drop_caches(compiled=False, host_inputs=True)
        t = tuner_conv()
        t.SetSubset(units(s))
        t.Tune()
        rows = t.rows()
        e2e_rows += len(rows)
        e2e_ok += sum(1 for r in rows if r.status == "ok" and r.verified == "pass")
        del t
    e2e_t = reduce_over_ranks(world, time.perf_counter() - t0, "max")
    e2e_value = reduce_over_ranks(world, float(e2e_rows), "sum") / e2e_t
    e2e_ok = int(reduce_over_ranks(world, float(e2e_ok), "sum"))
    h2d = ((X + F - 1) * (Y + F - 1) + F * F) * 4 * int(n_gpus)  # one job per GPU per step
    d2h = chunk * int(n_gpus) * ROW_BYTES

    # configs[4]: the device-bound scaling workload -- a fixed seeded sample
    # of the 4096^3 GEMM space, a disjoint share of it per GPU.
    gemm_block = None
    if args.gemm_per_gpu > 0:
        gemm_block = gemm_scaling_block(pkg, args, world, devices, first_slot, slots_here, threads)

    best_row = min((r for r in all_rows if r.time_ms and r.verified == "pass"),
                   key=lambda r: r.time_ms)
    peaks = load_peaks()
    line = {
        "metric": METRIC, "value": value, "unit": "configs/s", "n_gpus": int(n_gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: the reference's fill recipes (mt19937_64, seed 2026), no datasets",
        "config": {
            "workload": WORKLOAD + f": {valid} configurations (B200 limits), {chunk} per GPU per "
                                   "step in a fixed seeded order, each verified (rel 1e-4, abs 1e-6)",
            "repetitions": 3, "warmup_launches": 1,
            "l2": "flushed (256 MiB read) before every timed launch; inputs 134 MB + output 134 MB",
            "steps": "the K timed steps (K x chunk configurations per GPU) stream through one "
                     "pipelined search; warm-up steps use other configurations; chunk depends on "
                     f"K and W only (sized for {MAX_GPUS} GPUs), so per-GPU work is N-independent",
            "timing": "step: host wall clock (compile is host work), barrier + device sync on "
                      "both sides, max over ranks; kernels: CUDA events on the launching stream",
            "parallelism": (f"{world} process(es) x {slots_here} GPU worker(s), configuration-"
                            "sharded (dynamic chunk queue), no NCCL, no data-path collective"),
            "compile_threads_per_process": threads,
        },
        "gpus_active": gpus_active,
        "rows_per_gpu_worker": sorted(per_device.values()),
        "configs_verified": ok, "configs_failed_verification": failed_verify,
        "value_warm_cache": value_warm,
        "e2e": {"value": e2e_value, "unit": "configs/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "what": "public API (Tuner), one fresh job per GPU per step, cold: compile cache "
                        "and pinned host inputs dropped; host materializes the recipes "
                        "(mt19937_64), H2D image + taps, compile/launch/verify, D2H the rows",
                "verified": e2e_ok},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    achieved = CONV_BYTES / (best_row.time_ms * 1e-3) / 1e9
    line["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                        "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                        "kernel": best_row.config,
                        "peak_src": f"MEASURED_PEAKS.json hbm_gbs ({peaks['src']})"}
    if gemm_block:
        line["configs4_gemm4096"] = gemm_block
    if rank == 0 and args.no_tuned:
        # the roofline always uses the sustained protocol (30 back-to-back
        # launches between one event pair, mean launch duration): a single
        # flushed launch can end before its output write-backs drain and
        # read above the copy bandwidth
        sus = pkg.CudaBackend(devices[0], compile_threads=threads, warmup=3, stream_timing=True)
        req = pkg.conv_request(X, Y, F, pkg.parse_canonical(best_row.config), reps=30)
        rs = sus.evaluate(req)
        sus.close()
        if rs.ok:
            gbs = CONV_BYTES / (rs.mean_ms * 1e-3) / 1e9
            line["roofline"].update(achieved=gbs, frac=gbs / peaks["hbm_gbs"],
                                    kernel="conv2d_k0 " + best_row.config,
                                    algorithmic_bytes=CONV_BYTES,
                                    timing="mean launch duration of 30 back-to-back launches of "
                                           "this run's best sampled configuration (one CUDA event "
                                           "pair on the launch stream, no flushes)")
    if rank == 0 and not args.no_tuned:
        line["tuned"] = tuned_block(pkg, devices[0], threads, best_row, peaks)
        best3 = line["tuned"]["conv"].get("3")
        if best3 and best3.get("gbs"):
            line["roofline"].update(
                achieved=best3["gbs"], frac=best3["gbs"] / peaks["hbm_gbs"],
                kernel="conv2d_k0 " + best3["config"], traffic=best3.get("dram_bytes"),
                algorithmic_bytes=CONV_BYTES,
                timing="mean launch duration of 30 back-to-back launches between one CUDA event "
                       "pair on the launch stream (no flushes)")
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_configs()
        line["cpu_baseline_kernels"] = cpu_baseline_kernels()
    if rank == 0:
        print(json.dumps(line), flush=True)


def gemm_scaling_block(pkg, args, world, devices, first_slot, slots_here, threads) -> dict:
    """configs[4] (BASELINE.json): tuning throughput over the 4096^3 GEMM space,
    device-bound.  The unit list is ONE fixed seeded sample of the composed
    space (the same list for every N); GPU g evaluates entries
    [g*P, (g+1)*P).  prune_factor 2: a configuration whose first flushed
    launch is over 2x the best verified time is timed once (still verified)."""
    m = 4096
    t = pkg.Tuner.gemm(m, m, m, devices=devices, compile_threads=threads)
    t.SetVerification(True)
    t.SetRepetitions(3)
    t.SetPruning(2.0)
    _, _, valid = t.space_counts()
    sample = random.Random(1).sample(range(valid), min(valid, MAX_GPUS * args.gemm_per_gpu * 2))
    P = args.gemm_per_gpu
    # warm-up: the second half of the sample (inputs, device reference, pool)
    warm = sample[MAX_GPUS * P:][first_slot * 8:(first_slot + slots_here) * 8]
    t.SetSubset(warm)
    t.Tune()
    mine = sample[first_slot * P:(first_slot + slots_here) * P]
    t.SetSubset(mine)
    barrier(world)
    t0 = time.perf_counter()
    s = t.Tune()
    el = time.perf_counter() - t0
    barrier(world)
    rows = t.rows()
    t_max = reduce_over_ranks(world, el, "max")
    n = reduce_over_ranks(world, float(len(rows)), "sum")
    good = [r for r in rows if r.status == "ok" and r.verified == "pass" and r.time_ms]
    best_ms = min((r.time_ms for r in good), default=float("inf"))
    best_ms = -reduce_over_ranks(world, -best_ms, "max")
    nver = int(reduce_over_ranks(world, float(len(good)), "sum"))
    return {"value": n / t_max, "unit": "configs/s", "configs": int(n), "verified": nver,
            "seconds": t_max, "per_gpu": P, "kernel_launches": int(reduce_over_ranks(
                world, float(s["kernel_launches"]), "sum")),
            "best_found_gflops": 2.0 * m ** 3 / (best_ms * 1e-3) / 1e9 if best_ms < 1e30 else None,
            "sample": f"random.Random(1).sample of the {valid}-configuration space; GPU g takes "
                      f"entries [g*{P}, (g+1)*{P})", "prune_factor": 2.0, "repetitions": 3}


def tuned_block(pkg, local, threads, sample_best, peaks) -> dict:
    """Re-times the per-filter winners (configs[1]), the SGEMM winners
    (configs[2]-[4] sizes) and the TF32 variant."""
    table = tuned_table()
    # `be`: the tuner's protocol (L2 flushed, best of 10).  `sus`: 30
    # back-to-back launches without flushes between one event pair (no events
    # between launches, tools/launch_overhead_probe.py), mean launch time -- the
    # sustained figure the roofline uses (each launch also pays for the
    # previous launch's L2 write-backs, as in a real pipeline).
    be = pkg.CudaBackend(local, compile_threads=threads)
    sus = pkg.CudaBackend(local, compile_threads=threads, warmup=3, stream_timing=True)
    fp32_peak = fp32_peak_gflops()
    tf32_peak = tf32_peak_gflops()
    out = {"conv": {}, "source": "tuned/b200_winners.json" if table else "this run's sample",
           "timing": "time_ms: best of 10 flushed launches; mean_ms: mean launch duration of 30 "
                     "back-to-back launches between one event pair, no flushes (roofline uses "
                     "mean_ms)"}
    for f in (3, 5, 7, 9, 11):
        entry = table.get("conv", {}).get(str(f))
        cfg = entry["config"] if entry else (sample_best.config if f == 3 else None)
        if not cfg:
            continue
        req = pkg.conv_request(X, Y, f, pkg.parse_canonical(cfg), reps=10)
        r = be.evaluate(req)
        req.repetitions = 30
        rs = sus.evaluate(req)
        if not (r.ok and rs.ok):
            out["conv"][str(f)] = {"config": cfg, "status": r.status, "message": r.message}
            continue
        mean = rs.mean_ms
        gflops = conv_flops(f) / (mean * 1e-3) / 1e9
        gbs = CONV_BYTES / (mean * 1e-3) / 1e9
        ai = conv_flops(f) / CONV_BYTES
        bound = "hbm" if ai < fp32_peak / peaks["hbm_gbs"] else "fp32"
        out["conv"][str(f)] = {
            "config": cfg, "time_ms": r.time_ms, "mean_ms": mean, "gflops": gflops, "gbs": gbs,
            "gflops_best": conv_flops(f) / (r.time_ms * 1e-3) / 1e9,
            "verified": r.verification, "bound": bound,
            "frac_hbm": gbs / peaks["hbm_gbs"], "frac_fp32": gflops / fp32_peak,
            "frac": gbs / peaks["hbm_gbs"] if bound == "hbm" else gflops / fp32_peak,
            "dram_bytes": (entry or {}).get("dram_bytes"),
        }
    def shape(key):  # "2048" (square) or "8192x256x8192" (configs[3] non-square)
        v = [int(t) for t in key.split("x")]
        return (v[0], v[0], v[0]) if len(v) == 1 else tuple(v)

    for size, g in sorted(table.get("gemm", {}).items(), key=lambda kv: shape(kv[0])):
        m, n, k = shape(size)
        flops = 2.0 * m * n * k
        req = pkg.gemm_request(m, n, k, pkg.parse_canonical(g["config"]), reps=10)
        r = be.evaluate(req)
        req.repetitions = 30 if flops <= 2.0 * 4096 ** 3 else 10
        rs = sus.evaluate(req)
        if r.ok and rs.ok:
            gf = flops / (rs.mean_ms * 1e-3) / 1e9
            out[f"sgemm_{size}"] = {"config": g["config"], "time_ms": r.time_ms,
                                    "mean_ms": rs.mean_ms, "gflops": gf,
                                    "gflops_best": flops / (r.time_ms * 1e-3) / 1e9,
                                    "verified": r.verification, "bound": "fp32",
                                    "frac": gf / fp32_peak, "dram_bytes": g.get("dram_bytes")}
    for size, t in sorted(table.get("gemm_tf32", {}).items(), key=lambda kv: int(kv[0])):
        m = int(size)
        req = pkg.gemm_request(m, m, m, pkg.parse_canonical(t["config"]), reps=10, tf32=True)
        r = be.evaluate(req)
        req.repetitions = 30 if m <= 4096 else 10
        rs = sus.evaluate(req)
        if r.ok and rs.ok:
            tf = 2.0 * m ** 3 / (rs.mean_ms * 1e-3) / 1e9
            out[f"tf32_{m}"] = {"config": t["config"], "time_ms": r.time_ms, "mean_ms": rs.mean_ms,
                                "gflops": tf, "gflops_best": 2.0 * m ** 3 / (r.time_ms * 1e-3) / 1e9,
                                "verified": r.verification, "tolerance": "rel 1e-3, abs 1e-6",
                                "bound": "tensor (tf32)", "frac": tf / tf32_peak,
                                "frac_half_bf16_measured": tf / tf32_half_bf16_gflops(),
                                "dram_bytes": t.get("dram_bytes")}
    out["fp32_peak_gflops"] = fp32_peak
    out["tf32_peak_gflops"] = tf32_peak
    out["tf32_peak_src"] = ("B200_PROFILING.md fallback: tf32 tensor 1.1 PFLOP/s dense (no TF32 "
                            "figure in MEASURED_PEAKS.json); frac_half_bf16_measured = against half "
                            "the measured bf16 burst")
    be.close()
    sus.close()
    return out


if __name__ == "__main__":
    main()
