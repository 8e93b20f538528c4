"""BASELINE.json configs[3] and configs[4] on a B200 (run under gpurun).

configs[3]  SGEMM shape sweep (square 256..8192 and skinny / non-square)
            tuned with simulated annealing and with PSO (the paper's
            strategies), per-shape best.
configs[4]  SGEMM 4096^3 search-space execution: tuning throughput on a fixed
            seeded sample of the 852,608-configuration space (the same
            sample for every device count; this box has one GPU), plus the
            best configuration found in it.
"""
import argparse
import json
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402

SHAPES = [(256, 256, 256), (1024, 1024, 1024), (4096, 4096, 4096), (8192, 8192, 8192),
          (8192, 256, 8192), (4096, 4096, 256), (256, 8192, 4096)]


def shape_sweep(fraction: float, out: dict, strategies=("annealing", "pso")):
    for (m, n, k) in SHAPES:
        for strat in strategies:
            t = pkg.Tuner.gemm(m, n, k)
            # Tiles must divide the problem (SURVEY 7 hard part 10): the
            # skinny shapes get job-level constraints, as jobfile.hpp allows.
            for dim, name in ((m, "MWG"), (n, "NWG"), (k, "KWG")):
                if dim < 128:
                    t.AddConstraint(f"{name} <= {dim}")
            t.SetVerification(True)
            t.SetRepetitions(3)
            t.SetSeed(1)
            if strat == "annealing":
                t.UseAnnealing(fraction, 4.0)
            else:
                t.UsePSO(fraction, 3, 0.4, 0.0, 0.4)
            t0 = time.time()
            s = t.Tune()
            wall = time.time() - t0
            cfg, ms = t.GetBestResult()
            rows = t.rows()
            rec = {"m": m, "n": n, "k": k, "strategy": strat, "rows": len(rows),
                   "failed": s["failed_evaluations"], "wall_s": wall, "best_config": cfg,
                   "best_ms": ms, "gflops": 2.0 * m * n * k / ms / 1e6,
                   "configs_per_s": len(rows) / wall}
            out.setdefault("shape_sweep", []).append(rec)
            print(json.dumps(rec), flush=True)


def throughput_4096(sample: int, out: dict, prune: float = 0.0):
    t = pkg.Tuner.gemm(4096, 4096, 4096)
    if prune:
        t.SetPruning(prune)
    _, _, valid = t.space_counts()
    idx = sorted(random.Random(1).sample(range(valid), sample))
    t.SetVerification(True)
    t.SetRepetitions(3)
    t.SetSubset(idx)
    t0 = time.time()
    s = t.Tune()
    wall = time.time() - t0
    cfg, ms = t.GetBestResult()
    rec = {"m": 4096, "sample": sample, "space": valid, "wall_s": wall,
           "configs_per_s": sample / wall, "best_config": cfg, "best_ms": ms,
           "gflops": 2.0 * 4096 ** 3 / ms / 1e6, "failed": s["failed_evaluations"],
           "compile_s": s["compile_s"], "device_s": s["device_s"], "prune_factor": prune}
    out["throughput_4096" + (f"_prune{prune:g}" if prune else "")] = rec
    print(json.dumps(rec), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fraction", type=float, default=1 / 4096)
    ap.add_argument("--sample", type=int, default=1024)
    ap.add_argument("--skip-shapes", action="store_true")
    ap.add_argument("--skip-4096", action="store_true")
    ap.add_argument("--prune", type=float, default=0.0,
                    help="also measure the 4096 sample with this prune_factor")
    args = ap.parse_args()
    out = {}
    if not args.skip_4096:
        throughput_4096(args.sample, out)
        if args.prune:
            throughput_4096(args.sample, out, args.prune)
    if not args.skip_shapes:
        shape_sweep(args.fraction, out)
    p = ROOT / "gpurun_out" / "gemm_sweeps.json"
    p.parent.mkdir(exist_ok=True)
    p.write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
