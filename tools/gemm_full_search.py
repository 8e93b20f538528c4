"""Full search of the paper's SGEMM space on one B200, in shards (run under gpurun).

The composed space (852,608 configurations with the B200 limits) is split into
contiguous unit ranges of its enumeration order -- exactly the units the
sharded executor hands to separate GPUs -- and each call evaluates one range
(compile + time + verify every configuration).  --merge combines the shard
summaries with the executor's rule (strict minimum, earliest index wins).

  python tools/gemm_full_search.py --size 2048 --start 0 --count 213152
  python tools/gemm_full_search.py --merge gpurun_out/gemm_full_*.json

--dump-times writes every row's measured time (float32, enumeration order,
NaN where a configuration failed or was not verified) to
gpurun_out/gemm_full_<size>_<start>_times.npy -- a compact replay table for
offline strategy studies (tools/gemm_strategy_study.py).
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def run(size: int, start: int, count: int, prune: float, dump: bool = False,
        checkpoint: str | None = None) -> None:
    import shutil

    import paper_1703_06503_b200 as pkg

    t = pkg.Tuner.gemm(size, size, size)
    if checkpoint:
        # Resume file (replay CSV of verified rows): a shard cut off by the
        # call's time limit continues where it stopped.  A copy travels in
        # profiles/ (gpurun_out/ is not pushed to the box).
        ck = ROOT / "gpurun_out" / Path(checkpoint).name
        ck.parent.mkdir(exist_ok=True)
        seed = ROOT / checkpoint
        if seed.exists() and not ck.exists():
            shutil.copy(seed, ck)
            if Path(str(seed) + ".job").exists():
                shutil.copy(str(seed) + ".job", str(ck) + ".job")
        t.SetCheckpoint(str(ck))
    _, _, valid = t.space_counts()
    stop = min(valid, start + count)
    t.SetVerification(True)
    t.SetRepetitions(3)
    if prune:
        t.SetPruning(prune)
    t.SetSubset(list(range(start, stop)))
    t0 = time.time()
    s = t.Tune()
    wall = time.time() - t0
    rows = t.rows()
    ok = [(r.space_index, r.time_ms) for r in rows if r.status == "ok" and r.verified == "pass"]
    best_i, best_t = min(ok, key=lambda v: (v[1], v[0]))
    top = sorted(ok, key=lambda v: (v[1], v[0]))[:50]
    rec = {"size": size, "space": valid, "start": start, "stop": stop, "rows": len(rows),
           "verified_ok": len(ok), "failed": len(rows) - len(ok), "wall_s": wall,
           "configs_per_s": len(rows) / wall, "prune_factor": prune,
           "best_index": best_i, "best_ms": best_t, "best_config": t.space_config(best_i),
           "top50": [[i, ms, t.space_config(i)] for i, ms in top],
           "failures": [[r.space_index, r.status, r.verified, r.message[:120]]
                        for r in rows if not (r.status == "ok" and r.verified == "pass")][:20],
           "compile_s": s["compile_s"], "device_s": s["device_s"]}
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    if dump:
        import numpy as np

        times = np.full(stop - start, np.nan, dtype=np.float32)
        for i, ms in ok:
            times[i - start] = ms
        np.save(ROOT / "gpurun_out" / f"gemm_full_{size}_{start:07d}_times.npy", times)
    out = ROOT / "gpurun_out" / f"gemm_full_{size}_{start:07d}.json"
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(rec, indent=1))
    print(json.dumps({k: v for k, v in rec.items() if k not in ("top50", "failures")}), flush=True)


def merge(paths: list) -> None:
    recs = sorted((json.loads(Path(p).read_text()) for p in paths), key=lambda r: r["start"])
    covered = sum(r["stop"] - r["start"] for r in recs)
    best = min(((r["best_ms"], r["best_index"], r["best_config"]) for r in recs))
    top = sorted((tuple(x) for r in recs for x in r["top50"]), key=lambda v: (v[1], v[0]))[:50]
    size = recs[0]["size"]
    summary = {"size": size, "space": recs[0]["space"], "covered": covered,
               "rows": sum(r["rows"] for r in recs), "verified_ok": sum(r["verified_ok"] for r in recs),
               "failed": sum(r["failed"] for r in recs), "wall_s": sum(r["wall_s"] for r in recs),
               "configs_per_s": sum(r["rows"] for r in recs) / sum(r["wall_s"] for r in recs),
               "best_index": best[1], "best_ms": best[0], "best_config": best[2],
               "best_gflops": 2 * size ** 3 / best[0] / 1e6, "top50": top,
               "shards": [{k: r[k] for k in ("start", "stop", "rows", "failed", "wall_s",
                                            "configs_per_s", "best_index", "best_ms")} for r in recs]}
    print(json.dumps({k: v for k, v in summary.items() if k != "top50"}, indent=1))
    Path(ROOT / "gpurun_out" / f"gemm_full_{size}_merged.json").write_text(json.dumps(summary, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=2048)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--count", type=int, default=213152)
    ap.add_argument("--prune", type=float, default=2.0)
    ap.add_argument("--merge", nargs="+")
    ap.add_argument("--dump-times", action="store_true")
    ap.add_argument("--checkpoint", help="repo-relative seed checkpoint (copied to gpurun_out/)")
    a = ap.parse_args()
    if a.merge:
        merge(a.merge)
    else:
        run(a.size, a.start, a.count, a.prune, a.dump_times, a.checkpoint)
