"""A/B a GEMM code-generation change on the same random sample (run under gpurun).

Runs the verified random search of the SGEMM space at M=N=K (fixed seed, so
every process visits the same configurations) and dumps every row's time;
compare two dumps with --compare.  Env knobs such as KTC_GEMM_DBUF_MAX select
the variant.

  python tools/gemm_ab.py --size 2048 --fraction 512 --out gpurun_out/ab_on.json
  KTC_GEMM_DBUF_MAX=0 python tools/gemm_ab.py ... --out gpurun_out/ab_off.json
  python tools/gemm_ab.py --compare gpurun_out/ab_off.json gpurun_out/ab_on.json
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def run(size: int, fraction: int, out: str) -> None:
    import paper_1703_06503_b200 as pkg

    t = pkg.Tuner.gemm(size, size, size)
    t.SetVerification(True, rel_tol=1e-4)
    t.SetRepetitions(3)
    t.UseRandomSearch(1.0 / fraction)
    t0 = time.time()
    t.Tune()
    wall = time.time() - t0
    rows = {r.config: (r.time_ms, r.status, r.verified) for r in t.rows()}
    cfg, ms = t.GetBestResult()
    res = {"size": size, "wall_s": wall, "best": cfg, "best_ms": ms,
           "best_tflops": 2 * size ** 3 / ms / 1e9, "rows": rows}
    Path(out).write_text(json.dumps(res))
    bad = sum(1 for v in rows.values() if v[1] != "ok" or v[2] != "pass")
    print(f"size {size}: {len(rows)} rows, {bad} not ok/pass, best {cfg} {ms:.4f} ms "
          f"= {res['best_tflops']:.1f} TFLOP/s, wall {wall:.0f}s", flush=True)


def compare(a: str, b: str) -> None:
    A, B = json.loads(Path(a).read_text()), json.loads(Path(b).read_text())
    ratios = [A["rows"][c][0] / B["rows"][c][0] for c in A["rows"]
              if c in B["rows"] and A["rows"][c][0] and B["rows"][c][0]]
    print(f"A best {A['best_tflops']:.1f} TF ({A['best']})\nB best {B['best_tflops']:.1f} TF ({B['best']})")
    print(f"per-config time A/B: median {statistics.median(ratios):.3f}, "
          f"B faster on {sum(r > 1 for r in ratios)}/{len(ratios)}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=2048)
    ap.add_argument("--fraction", type=int, default=512)
    ap.add_argument("--out")
    ap.add_argument("--compare", nargs=2)
    a = ap.parse_args()
    if a.compare:
        compare(*a.compare)
    else:
        run(a.size, a.fraction, a.out)
