"""A/B the tuning-time NVRTC compile mode on a fixed configuration sample (run under gpurun).

The compile mode (KTC_FAST_COMPILE=<0|min|mid|max>, read once per process)
changes how long NVRTC takes per configuration and possibly the code it
emits.  This evaluates the same configurations -- the 16 fastest of each
round-1 full/random search (profiles/sweep_r01/*_replay.csv) plus a seeded
random sample of the rest -- with best-of-5 flushed timing, and dumps the
per-configuration times; --compare prints winner and median ratios.

  KTC_FAST_COMPILE=0   python tools/compile_ab.py --out gpurun_out/cab_0.json
  KTC_FAST_COMPILE=min python tools/compile_ab.py --out gpurun_out/cab_min.json
  python tools/compile_ab.py --compare gpurun_out/cab_0.json gpurun_out/cab_min.json
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import random
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
SWEEP = ROOT / "profiles" / "sweep_r01"


def sample(name: str, top: int, rand: int) -> list[str]:
    rows = [(r["config"], float(r["time_ms"])) for r in csv.DictReader(open(SWEEP / name))
            if r["time_ms"] not in ("", "inf", "nan")]
    rows.sort(key=lambda r: r[1])
    best = [c for c, _ in rows[:top]]
    rest = [c for c, _ in rows[top:]]
    return best + random.Random(7).sample(rest, min(rand, len(rest)))


def run(out: str, top: int, rand: int, families: list[str]) -> None:
    import paper_1703_06503_b200 as pkg

    be = pkg.CudaBackend(0)
    res = {"mode": os.environ.get("KTC_FAST_COMPILE", "default"), "families": {}}
    for fam in families:
        if fam.startswith("conv"):
            f = int(fam[4:])
            cfgs = sample(f"conv_f{f}_replay.csv", top, rand)
            mk = lambda c: pkg.conv_request(8192, 4096, f, pkg.parse_canonical(c), reps=5)  # noqa: E731
        else:
            cfgs = sample("gemm_2048_replay.csv", top, rand)
            mk = lambda c: pkg.gemm_request(2048, 2048, 2048, pkg.parse_canonical(c), reps=5)  # noqa: E731
        rows = {}
        t0 = time.time()
        for c in cfgs:
            be.prefetch(mk(c))
        for c in cfgs:
            r = be.evaluate(mk(c))
            rows[c] = [r.time_ms if r.ok and r.verification == "pass" else None, r.compile_ms,
                       r.status, r.verification]
        wall = time.time() - t0
        ok = [v[0] for v in rows.values() if v[0]]
        res["families"][fam] = {"rows": rows, "wall_s": wall, "best_ms": min(ok) if ok else None,
                                "top": cfgs[:top]}
        print(f"{fam}: {len(rows)} configs, {len(ok)} ok, best {min(ok) if ok else None} ms, "
              f"wall {wall:.1f}s", flush=True)
    Path(out).write_text(json.dumps(res))


def compare(a: str, b: str) -> None:
    A, B = json.loads(Path(a).read_text()), json.loads(Path(b).read_text())
    print(f"A = {A['mode']}  B = {B['mode']}")
    for fam, fa in A["families"].items():
        fb = B["families"].get(fam)
        if not fb:
            continue
        ratios = [fa["rows"][c][0] / fb["rows"][c][0] for c in fa["rows"]
                  if c in fb["rows"] and fa["rows"][c][0] and fb["rows"][c][0]]
        top = [fa["rows"][c][0] / fb["rows"][c][0] for c in fa["top"]
               if fa["rows"][c][0] and fb["rows"][c][0]]
        print(f"{fam:7s} best A {fa['best_ms']:.4f} ms  B {fb['best_ms']:.4f} ms  "
              f"(B/A {fb['best_ms'] / fa['best_ms']:.3f}); per-config A/B median "
              f"{statistics.median(ratios):.3f} (top: {statistics.median(top):.3f}, min "
              f"{min(top):.3f}); B faster on {sum(r > 1.01 for r in ratios)}, slower on "
              f"{sum(r < 0.99 for r in ratios)} of {len(ratios)}; wall A {fa['wall_s']:.0f}s "
              f"B {fb['wall_s']:.0f}s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--top", type=int, default=16)
    ap.add_argument("--rand", type=int, default=48)
    ap.add_argument("--families", default="conv3,conv7,conv11,gemm")
    ap.add_argument("--compare", nargs=2)
    a = ap.parse_args()
    if a.compare:
        compare(*a.compare)
    else:
        run(a.out, a.top, a.rand, a.families.split(","))
