"""configs[4] on one B200 (run under gpurun): a seeded random 1/64 of the
852,608-configuration SGEMM space at 4096^3 through the sharded executor,
every configuration compiled + timed + verified, with the prune_factor
early-out (2x) -- tuning throughput and best-found GFLOPS."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402

frac = float(sys.argv[1]) if len(sys.argv) > 1 else 1 / 64
t = pkg.Tuner.gemm(4096, 4096, 4096)
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
rec = {"m": 4096, "fraction": frac, "rows": len(rows), "wall_s": wall, "configs_per_s": len(rows) / wall,
       "best_config": cfg, "best_ms": ms, "gflops": 2 * 4096 ** 3 / ms / 1e6, "not_ok": bad,
       "prune_factor": 2.0, "compile_s": s["compile_s"], "device_s": s["device_s"]}
print(json.dumps(rec), flush=True)
out = ROOT / "gpurun_out" / "gemm4096_search.json"
out.parent.mkdir(exist_ok=True)
out.write_text(json.dumps(rec, indent=1))
t.write_replay(str(ROOT / "gpurun_out" / "gemm_4096_replay.csv"))
