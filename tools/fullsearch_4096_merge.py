"""Merge the configs[4] full search (4096^3, all 852,608 SGEMM configurations)
from its checkpointed shards and replay it through the reference's own
run_full (CPU, in this container; oracle/_ref).

    python tools/fullsearch_4096_merge.py [gpurun_out]

Inputs (per shard start s, written by tools/gpu_fullsearch_4096.sh, kept in
profiles/fullsearch_4096/shards/):
  gemm_full_4096_<s>_times.npy  every row's time (float32, NaN = not verified)
  gemm_full_4096_<s>.json       shard summary of the call that finished it
  ckpt_<s>.csv (optional)       replay CSV, completes a shard cut off mid-call
Outputs (profiles/fullsearch_4096/): summary.json, gemm4096_times.npz (all
times, float32 by enumeration index, NaN where not verified).

Merge rule = the sharded executor's: strict minimum time, earliest index.  The
replay runs the reference's run_full over the same space on its
ReplayBackend (backend.hpp:485-592) and must return the same index and time.
"""
import glob
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
B200 = {"name": "B200", "max_work_group_total": 1024, "max_work_group_dim": [1024, 1024, 64],
        "local_mem_bytes": 232448}
SIZE = 4096


def main():
    src = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "profiles" / "fullsearch_4096" / "shards")
    import paper_1703_06503_b200 as pkg

    t = pkg.Tuner.gemm(SIZE, SIZE, SIZE)
    _, _, n = t.space_counts()
    t0 = time.time()
    index = {t.space_config(i): i for i in range(n)}
    print(f"enumerated {n} configurations in {time.time() - t0:.1f}s", flush=True)
    times = np.full(n, np.nan, dtype=np.float64)
    # Per-shard time dumps (float32 CUDA-event times, NaN = not verified);
    # a shard cut off by a call's limit is completed from its checkpoint.
    for npy in sorted(glob.glob(str(src / f"gemm_full_{SIZE}_*_times.npy"))):
        start = int(Path(npy).name.split("_")[3])
        v = np.load(npy).astype(np.float64)
        times[start:start + len(v)] = np.where(np.isfinite(v), v, times[start:start + len(v)])
    for ck in sorted(glob.glob(str(src / "ckpt_*.csv"))):
        with open(ck) as f:
            next(f)
            for line in f:
                key, ms = line.rstrip("\n").rsplit(",", 1)
                i = index[key]
                if not np.isfinite(times[i]):
                    times[i] = float(np.float32(float(ms)))
    shards = [json.loads(Path(p).read_text()) for p in sorted(glob.glob(str(src / f"gemm_full_{SIZE}_*.json")))]
    ok = np.isfinite(times)
    best_i = int(np.nanargmin(times))  # first occurrence of the minimum = earliest index
    best_t = float(times[best_i])
    rec = {"size": SIZE, "space": n, "verified_rows": int(ok.sum()), "missing_or_failed": int(n - ok.sum()),
           "best_index": best_i, "best_ms": best_t, "best_config": t.space_config(best_i),
           "best_tflops": 2 * SIZE ** 3 / best_t / 1e9,
           "top20": [[int(i), float(times[i]), t.space_config(int(i))]
                     for i in np.argsort(np.where(ok, times, np.inf), kind="stable")[:20]],
           "shards": [{k: s.get(k) for k in ("start", "stop", "rows", "failed", "wall_s", "configs_per_s",
                                              "best_index", "best_ms", "prune_factor")} for s in shards],
           "shard_failures": [f for s in shards for f in s.get("failures", [])]}
    # Replay through the reference's run_full (needs every row: the replay
    # backend reports a missing configuration as an error row).
    from oracle import oracle as O  # checker only

    if O.ref_available() and ok.all():
        with tempfile.TemporaryDirectory() as d:
            csv = Path(d) / "measured.csv"
            with open(csv, "w") as f:
                f.write("config,time_ms\n")
                for i in range(n):
                    f.write(f"{t.space_config(i)},{float(times[i])!r}\n")
            job = {"template": "gemm", "problem": {"m": SIZE, "n": SIZE, "k": SIZE}, "device": B200,
                   "strategy": {"kind": "full"}, "verify": False,
                   "backend": {"kind": "replay", "path": "measured.csv"}}
            t1 = time.time()
            bi, bt = O.ref_job_run(json.dumps(job), d, str(Path(d) / "ref.csv"))
            rec["reference_replay"] = {"best_index": bi, "best_ms": bt, "seconds": time.time() - t1,
                                       "same_index": bi == best_i, "same_time": bt == best_t}
    out = ROOT / "profiles" / "fullsearch_4096"
    out.mkdir(parents=True, exist_ok=True)
    (out / "summary.json").write_text(json.dumps(rec, indent=1))
    np.savez_compressed(out / "gemm4096_times.npz", times=times.astype(np.float32))
    print(json.dumps({k: v for k, v in rec.items() if k not in ("top20",)}, indent=1))


if __name__ == "__main__":
    main()
