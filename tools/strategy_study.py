"""The paper's search-strategy study (Fig. 5: 128 runs per
strategy, 1/32 of the space each) replayed on B200-MEASURED times.

The per-configuration times are the full-search tables measured on a B200
(`profiles/sweep_r01c/conv_f*_replay.csv`, 5,104 configurations per filter,
8192x4096, best of 3 with L2 flush, every row device-verified).  Each
strategy runs 128 times through `Tuner.Stats` (the `ktune stats` sequence,
byte-identical to the reference's; tests/test_stats.py) on the replay
backend, so the study costs no GPU time and is exactly reproducible.

  python tools/strategy_study.py [--runs 128] [--out profiles/strategy_r01]
"""
import argparse
import csv
import json
import shutil
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1703_06503_b200 as pkg  # noqa: E402

B200 = {"name": "B200", "max_work_group_total": 1024, "max_work_group_dim": [1024, 1024, 64],
        "local_mem_bytes": 232448}
STRATEGIES = {
    "random": {"kind": "random", "fraction": "1/32"},
    "SA T=2": {"kind": "annealing", "fraction": "1/32", "temperature": 2},
    "SA T=4": {"kind": "annealing", "fraction": "1/32", "temperature": 4},
    "SA T=6": {"kind": "annealing", "fraction": "1/32", "temperature": 6},
    "PSO S=3": {"kind": "pso", "fraction": "1/32", "swarm": 3},
    "PSO S=6 a=b=g=0.3": {"kind": "pso", "fraction": "1/32", "swarm": 6, "alpha": 0.3,
                          "beta": 0.3, "gamma": 0.3},
}


def pct(best_known: float, t: float) -> float:
    return 100.0 * best_known / t


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=128)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "strategy_r01"))
    a = ap.parse_args()
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    results = {}
    for f in (3, 5, 7, 9, 11):
        table = ROOT / "profiles" / "sweep_r01c" / f"conv_f{f}_replay.csv"
        times = [float(r["time_ms"]) for r in csv.DictReader(table.open())]
        best_known = min(times)
        with tempfile.TemporaryDirectory() as td:
            shutil.copy(table, Path(td) / "table.csv")
            for name, strat in STRATEGIES.items():
                job = {"template": "conv", "problem": {"filter": f}, "device": B200,
                       "backend": {"kind": "replay", "path": "table.csv"}, "strategy": strat}
                t = pkg.Tuner.from_job(json.dumps(job), td, devices=[0, 1, 2, 3])
                s = t.Stats(a.runs, 1, str(Path(td) / "s.csv"))
                runs = list(csv.DictReader((Path(td) / "s_runs.csv").open(newline="")))
                bests = [float(r["best_time_ms"]) for r in runs]
                tag = name.split()[0].lower() + "".join(c for c in name if c.isdigit())
                shutil.copy(Path(td) / "s_runs.csv", out / f"conv_f{f}_{tag}_runs.csv")
                space = s["space_mean"]
                results.setdefault(f, {})[name] = {
                    "mean_pct": sum(pct(best_known, b) for b in bests) / len(bests),
                    "worst_pct": pct(best_known, max(bests)),
                    "best_pct": pct(best_known, min(bests)),
                    "hit_best": sum(1 for b in bests if b == best_known),
                    "space_mean_pct_of_mean_time": pct(best_known, space),
                }
                space_all = [pct(best_known, x) for x in times]
                results[f]["_space"] = {"mean_pct": sum(space_all) / len(space_all),
                                        "share_above_80pct": sum(1 for x in space_all if x >= 80)
                                        / len(space_all),
                                        "best_known_ms": best_known, "configs": len(times)}
            print(f"f={f}", json.dumps(results[f]), flush=True)
    (out / "study.json").write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
