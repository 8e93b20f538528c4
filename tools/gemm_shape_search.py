"""Seeded random search of the SGEMM space at one (possibly non-square) shape
(configs[3]; run under gpurun): every configuration compiled, timed with the
launch policy in force (split-K for skinny / long-K shapes), verified.

    python tools/gemm_shape_search.py 8192x256x8192 [fraction]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402

shape = sys.argv[1]
m, n, k = (int(v) for v in shape.split("x"))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1 / 64
t = pkg.Tuner.gemm(m, n, k)
t.SetVerification(True)
t.SetRepetitions(3)
t.SetPruning(2.0)
t.UseRandomSearch(frac)
t0 = time.time()
s = t.Tune()
wall = time.time() - t0
cfg, ms = t.GetBestResult()
rows = t.rows()
bad = sum(1 for r in rows if r.status != "ok" or r.verified != "pass")
top = sorted(((r.time_ms, r.config) for r in rows if r.status == "ok" and r.verified == "pass"))[:10]
rec = {"shape": shape, "fraction": frac, "rows": len(rows), "wall_s": wall,
       "configs_per_s": len(rows) / wall, "best_config": cfg, "best_ms": ms,
       "gflops": 2 * m * n * k / ms / 1e6, "not_ok": bad, "prune_factor": 2.0, "top10": top}
print(json.dumps({k_: v for k_, v in rec.items() if k_ != "top10"}), flush=True)
out = ROOT / "gpurun_out" / f"gemm_shape_{shape}.json"
out.parent.mkdir(exist_ok=True)
out.write_text(json.dumps(rec, indent=1))
