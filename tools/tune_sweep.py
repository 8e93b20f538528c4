"""Tuning sweeps on the B200 (run under gpurun).

  conv   full search of the paper's conv space (B200 limits, 5104 configs)
         for each filter size, 8192x4096 fp32, verified      (configs[0,1])
  gemm   random search of the SGEMM space at 2048^3, verified (configs[2])

Writes tuned/b200_winners.json (the per-filter / per-shape winners bench.py
re-times), replay tables and a summary under profiles/<tag>/.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402


def conv_sweep(f: int, out: Path, fraction: float | None) -> dict:
    t = pkg.Tuner.conv(8192, 4096, f)
    t.SetVerification(True)
    t.SetRepetitions(3)
    if fraction:
        t.UseRandomSearch(fraction)
    else:
        t.UseFullSearch()
    t0 = time.time()
    s = t.Tune()
    wall = time.time() - t0
    rows = t.rows()
    t.write_replay(str(out / f"conv_f{f}_replay.csv"))
    cfg, ms = t.GetBestResult()
    bad = [r for r in rows if r.status != "ok" or r.verified != "pass"]
    flops = (1 + 2 * f * f) * 8192 * 4096
    res = {"config": cfg, "time_ms": ms, "gflops": flops / ms / 1e6,
           "gbs": 2 * 8192 * 4096 * 4 / ms / 1e6, "rows": len(rows), "wall_s": wall,
           "configs_per_s": len(rows) / wall, "not_ok": len(bad),
           "not_ok_examples": [(r.config, r.status, r.verified, r.message[:160]) for r in bad[:5]],
           "top5": [(r.config, r.time_ms) for r in sorted(
               (r for r in rows if r.time_ms and r.verified == "pass"), key=lambda r: r.time_ms)[:5]]}
    print(f"conv f={f}: {json.dumps(res)}", flush=True)
    return res


def gemm_sweep(m: int, out: Path, fraction: float, tf32=False) -> dict:
    t = pkg.Tuner.gemm(m, m, m, tf32=tf32)
    t.SetVerification(True, rel_tol=1e-3 if tf32 else 1e-4)
    t.SetRepetitions(3)
    if tf32:
        t.UseFullSearch()
    else:
        t.UseRandomSearch(fraction)
    t0 = time.time()
    t.Tune()
    wall = time.time() - t0
    rows = t.rows()
    name = "gemm_tf32" if tf32 else "gemm"
    t.write_replay(str(out / f"{name}_{m}_replay.csv"))
    cfg, ms = t.GetBestResult()
    bad = [r for r in rows if r.status != "ok" or r.verified != "pass"]
    res = {"config": cfg, "time_ms": ms, "gflops": 2 * m ** 3 / ms / 1e6, "rows": len(rows),
           "wall_s": wall, "configs_per_s": len(rows) / wall, "not_ok": len(bad),
           "not_ok_examples": [(r.config, r.status, r.verified, r.message[:160]) for r in bad[:5]],
           "top5": [(r.config, r.time_ms) for r in sorted(
               (r for r in rows if r.time_ms and r.verified == "pass"), key=lambda r: r.time_ms)[:5]]}
    print(f"{name} {m}: {json.dumps(res)}", flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--filters", default="3,5,7,9,11")
    ap.add_argument("--conv-fraction", type=float, default=0.0)
    ap.add_argument("--gemm-fraction", type=float, default=1 / 256)
    ap.add_argument("--gemm-sizes", default="2048")
    ap.add_argument("--tf32", action="store_true")
    ap.add_argument("--skip-conv", action="store_true")
    ap.add_argument("--skip-gemm", action="store_true")
    args = ap.parse_args()
    out = ROOT / "gpurun_out" / f"sweep_{args.tag}"
    out.mkdir(parents=True, exist_ok=True)
    table_path = ROOT / "gpurun_out" / "b200_winners.json"
    table = json.loads(table_path.read_text()) if table_path.exists() else {}
    if not args.skip_conv:
        for f in [int(v) for v in args.filters.split(",") if v]:
            table.setdefault("conv", {})[str(f)] = conv_sweep(f, out, args.conv_fraction or None)
            table_path.write_text(json.dumps(table, indent=1))
    if not args.skip_gemm:
        for m in [int(v) for v in args.gemm_sizes.split(",") if v]:
            table.setdefault("gemm", {})[str(m)] = gemm_sweep(m, out, args.gemm_fraction)
            table_path.write_text(json.dumps(table, indent=1))
    if args.tf32:
        for m in [int(v) for v in args.gemm_sizes.split(",") if v]:
            table.setdefault("gemm_tf32", {})[str(m)] = gemm_sweep(m, out, 1.0, tf32=True)
            table_path.write_text(json.dumps(table, indent=1))
    print("wrote", table_path)


if __name__ == "__main__":
    main()
