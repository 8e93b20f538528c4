"""The paper's SGEMM strategy study (Fig. 7: 128 runs per
strategy, 1/2048 of the space each) replayed on B200-MEASURED times.

Input: the measured time of EVERY configuration of the 852,608-configuration
GEMM space at 2048^3 (one full search on a B200, `tools/gemm_full_search.py
--dump-times`; float32 per enumeration index, NaN = failed), stored as
`profiles/fullsearch_r01/gemm2048_times.npz`.  The table is expanded into a
replay CSV (`config,time_ms`, ReplayBackend's format) and each strategy runs
128 times through `Tuner.Stats` -- the `ktune stats` sequence, byte-identical
to the reference's reports (tests/test_stats.py) -- on 8 host workers.

  python tools/gemm_strategy_study.py [--times gpurun_out/gemm_full_2048_0000000_times.npy --store]
"""
import argparse
import csv
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1703_06503_b200 as pkg  # noqa: E402

B200 = {"name": "B200", "max_work_group_total": 1024, "max_work_group_dim": [1024, 1024, 64],
        "local_mem_bytes": 232448}
STORE = ROOT / "profiles" / "fullsearch_r01" / "gemm2048_times.npz"
STRATEGIES = {
    "random": {"kind": "random", "fraction": "1/2048"},
    "SA T=2": {"kind": "annealing", "fraction": "1/2048", "temperature": 2},
    "SA T=4": {"kind": "annealing", "fraction": "1/2048", "temperature": 4},
    "SA T=6": {"kind": "annealing", "fraction": "1/2048", "temperature": 6},
    "PSO S=3": {"kind": "pso", "fraction": "1/2048", "swarm": 3},
    "PSO S=6 a=b=g=0.3": {"kind": "pso", "fraction": "1/2048", "swarm": 6, "alpha": 0.3,
                          "beta": 0.3, "gamma": 0.3},
}


def load_times(path: Path) -> np.ndarray:
    if path.suffix == ".npz":
        return np.load(path)["times"]
    return np.load(path)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--times", default=str(STORE))
    ap.add_argument("--runs", type=int, default=128)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "strategy_r01"))
    ap.add_argument("--store", action="store_true",
                    help="keep a compressed copy of --times as " + str(STORE.relative_to(ROOT)))
    a = ap.parse_args()
    times = load_times(Path(a.times)).astype(np.float64)
    if a.store:
        np.savez_compressed(STORE, times=times.astype(np.float32))
    job = {"template": "gemm", "problem": {"m": 2048, "n": 2048, "k": 2048}, "device": B200}
    space = pkg.Tuner.from_job(json.dumps(job), ".")
    n = space.space_counts()[2]
    assert n == len(times), (n, len(times))
    ok = np.isfinite(times)
    best_known = float(times[ok].min())
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    res = {"space": n, "measured_ok": int(ok.sum()), "best_known_ms": best_known,
           "best_known_index": int(np.nanargmin(times)),
           "best_known_config": space.space_config(int(np.nanargmin(times))),
           "space_mean_pct": float(np.mean(100 * best_known / times[ok])),
           "space_share_above_80pct": float(np.mean(100 * best_known / times[ok] >= 80))}
    with tempfile.TemporaryDirectory() as td:
        with open(Path(td) / "table.csv", "w", newline="") as f:
            f.write("config,time_ms\n")
            for i in np.flatnonzero(ok):
                f.write(f"{space.space_config(int(i))},{float(times[i])!r}\n")
        for name, strat in STRATEGIES.items():
            j = dict(job, backend={"kind": "replay", "path": "table.csv"}, strategy=strat)
            t = pkg.Tuner.from_job(json.dumps(j), td, devices=list(range(8)))
            t.Stats(a.runs, 1, str(Path(td) / "s.csv"))
            runs = list(csv.DictReader((Path(td) / "s_runs.csv").open(newline="")))
            bests = np.array([float(r["best_time_ms"]) for r in runs])
            tag = name.split()[0].lower() + "".join(c for c in name if c.isdigit())
            (out / f"gemm2048_{tag}_runs.csv").write_bytes((Path(td) / "s_runs.csv").read_bytes())
            res[name] = {"mean_pct": float(np.mean(100 * best_known / bests)),
                         "worst_pct": float(100 * best_known / bests.max()),
                         "best_pct": float(100 * best_known / bests.min()),
                         "hit_best": int(np.sum(bests == best_known))}
            print(name, json.dumps(res[name]), flush=True)
    (out / "gemm2048_study.json").write_text(json.dumps(res, indent=1))
    print(json.dumps({k: v for k, v in res.items() if not isinstance(v, dict)}))


if __name__ == "__main__":
    main()
