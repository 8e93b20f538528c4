"""Search-space sharding across processes (one process per GPU).

Full and random searches visit a fixed, seeded list of configurations
(enumeration order / the random sample), so the list is split into chunks
dealt round-robin to the ranks; each rank tunes its units on its own GPU
(`Tuner.SetSubset`) and only per-unit result tuples -- (position, config,
status, time, verdict) -- travel back to rank 0 over torch.distributed
(gloo, host memory).  rank 0 merges them in unit order with the
reference's CachedEvaluator rule (strict <, the earliest evaluation wins a
tie, search.hpp:203-208), so the merged outcome equals a sequential run on
the same per-configuration results.  There is no data-path collective: the
tuning path has no exchange step.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class MergedOutcome:
    rows: list  # (position, config, status, time_ms, verified) in unit order
    best_index: int  # -1 when nothing succeeded
    best_time_ms: float | None
    best_config: str | None


def shard_units(units: list, rank: int, world: int, chunk: int = 16) -> list[tuple[int, int]]:
    """(position, unit) pairs of this rank: chunks dealt round-robin."""
    out = []
    for start in range(rank * chunk, len(units), world * chunk):
        out.extend((p, units[p]) for p in range(start, min(start + chunk, len(units))))
    return out


def merge(rows: list) -> MergedOutcome:
    rows = sorted(rows, key=lambda r: r[0])
    best_i, best_t = -1, None
    for i, (_, _, status, t, verified) in enumerate(rows):
        if status == "ok" and verified != "fail" and t is not None:
            if best_t is None or t < best_t:
                best_i, best_t = i, t
    return MergedOutcome(rows, best_i, best_t, rows[best_i][1] if best_i >= 0 else None)


def tune_shard(tuner, units: list, rank: int, world: int, chunk: int = 16) -> list:
    """Runs this rank's share of `units` on `tuner`; returns its row tuples."""
    mine = shard_units(units, rank, world, chunk)
    if not mine:
        return []
    tuner.SetSubset([u for _, u in mine])
    tuner.Tune()
    rows = tuner.rows()
    return [(pos, r.config, r.status, r.time_ms, r.verified) for (pos, _), r in zip(mine, rows)]


def gather_merge(local_rows: list, world: int, group=None) -> MergedOutcome | None:
    """Gathers every rank's rows on rank 0 and merges them (None elsewhere)."""
    if world == 1:
        return merge(local_rows)
    import torch.distributed as dist

    everything = [None] * world if dist.get_rank() == 0 else None
    dist.gather_object(local_rows, everything, dst=0, group=group)
    if dist.get_rank() != 0:
        return None
    return merge([r for part in everything for r in part])


# ---------------------------------------------------------------------------
# Repeated searches across processes (`ktune stats`, tools/ktune.cpp:120-258)
# ---------------------------------------------------------------------------
def stats_replicas(tuner, runs: int, base_seed: int, rank: int, world: int) -> list:
    """Runs this rank's replicas -- run indices rank, rank+world, ... -- each a
    whole search with seed base_seed + run on this rank's GPU (annealing and
    PSO chains do not shard; K independent chains do).  Returns
    (run, seed, best_time_ms, best_config) tuples."""
    out = []
    for run in range(rank, runs, world):
        tuner.SetSeed(base_seed + run)
        s = tuner.Tune()
        if s["best_index"] < 0:
            raise RuntimeError(f"run {run} (seed {base_seed + run}) found no successful "
                               "configuration")
        cfg, ms = tuner.GetBestResult()
        out.append((run, base_seed + run, ms, cfg))
    return out


def write_stats_reports(runs: list, out_csv: str, space_times: list | None = None) -> None:
    """rank 0: the reports ktc_tuner_stats writes, from gathered replicas --
    `out_csv` (best-of-run statistics), `<stem>_runs<ext>` and, when the
    whole-space times are given (unit order), `<stem>_space<ext>`."""
    import ctypes as C
    from pathlib import Path

    from . import _ktc as K

    lib = K.lib()
    runs = sorted(runs)
    vals = (C.c_double * len(runs))(*[r[2] for r in runs])
    K.check(lib.ktc_stats_write(vals, len(runs), str(out_csv).encode()))
    keep = [r[3].encode() for r in runs]
    arr = (K.RunSummary * len(runs))(*[K.RunSummary(r[0], r[1], r[2], c)
                                       for r, c in zip(runs, keep)])
    p = Path(out_csv)
    K.check(lib.ktc_runs_write(arr, len(runs), str(p.with_name(p.stem + "_runs" + p.suffix))
                               .encode()))
    if space_times:
        st = (C.c_double * len(space_times))(*space_times)
        K.check(lib.ktc_stats_write(st, len(space_times),
                                    str(p.with_name(p.stem + "_space" + p.suffix)).encode()))


def gather_runs(local: list, world: int, group=None) -> list | None:
    """All ranks' replica tuples on rank 0 (None elsewhere)."""
    if world == 1:
        return list(local)
    import torch.distributed as dist

    everything = [None] * world if dist.get_rank() == 0 else None
    dist.gather_object(local, everything, dst=0, group=group)
    if dist.get_rank() != 0:
        return None
    return [r for part in everything for r in part]
