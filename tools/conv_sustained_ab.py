"""Sustained-time A/B of conv kernel variants (run under gpurun; env knobs select the variant).

For each filter: the 12 fastest configurations of the round-1b full search
(profiles/sweep_r01c), timed two ways as bench.py does: best of 10 flushed
launches, and the mean of 30 back-to-back launches (the roofline figure).

  KTC_CONV_OSTREAM=0 python tools/conv_sustained_ab.py --out gpurun_out/os0.json
  KTC_CONV_OSTREAM=1 python tools/conv_sustained_ab.py --out gpurun_out/os1.json
  python tools/conv_sustained_ab.py --compare gpurun_out/os0.json gpurun_out/os1.json
"""
import argparse
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def top(f, n):
    rows = [(r["config"], float(r["time_ms"])) for r in
            csv.DictReader(open(ROOT / "profiles" / "sweep_r01c" / f"conv_f{f}_replay.csv"))]
    return [c for c, _ in sorted(rows, key=lambda r: r[1])[:n]]


def run(out, filters, n):
    import paper_1703_06503_b200 as pkg

    be = pkg.CudaBackend(0)
    sus = pkg.CudaBackend(0, flush_l2=False, warmup=3)
    res = {}
    for f in filters:
        for c in top(f, n):
            req = pkg.conv_request(8192, 4096, f, pkg.parse_canonical(c), reps=10)
            r = be.evaluate(req)
            req.repetitions = 30
            rs = sus.evaluate(req)
            res[f"{f}|{c}"] = [r.time_ms, rs.mean_ms, r.verification]
        best = min((v[1], k) for k, v in res.items() if k.startswith(f"{f}|"))
        print(f"f={f}: best sustained {best[0] * 1e3:.1f} us = {2 * 8192 * 4096 * 4 / best[0] / 1e6:.0f} GB/s "
              f"({best[1].split('|')[1]})", flush=True)
    Path(out).write_text(json.dumps(res))


def compare(a, b):
    A, B = json.loads(Path(a).read_text()), json.loads(Path(b).read_text())
    for f in sorted({k.split("|")[0] for k in A}, key=int):
        ks = [k for k in A if k.startswith(f + "|") and k in B]
        ba = min(A[k][1] for k in ks)
        bb = min(B[k][1] for k in ks)
        fa = min(A[k][0] for k in ks)
        fb = min(B[k][0] for k in ks)
        print(f"f={f}: sustained best A {ba * 1e3:.1f} us B {bb * 1e3:.1f} us ({bb / ba:.3f}); "
              f"flushed best A {fa * 1e3:.1f} B {fb * 1e3:.1f} ({fb / fa:.3f})")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--filters", default="3,5")
    ap.add_argument("--n", type=int, default=12)
    ap.add_argument("--compare", nargs=2)
    a = ap.parse_args()
    if a.compare:
        compare(*a.compare)
    else:
        run(a.out, [int(v) for v in a.filters.split(",")], a.n)
