"""Does the conv winners' loss against the FP32 roofline shrink with more waves?
(run under gpurun)

    python tools/conv_size_probe.py

Times the 6 fastest 8192x4096 configurations of each filter (profiles/sweep_r01c)
at 8192x4096, 8192x8192 and 16384x8192 (mean of 20 back-to-back launches,
verified): if the tail drain of the last wave of CTAs is what costs the
7x7-11x11 winners, TFLOP/s rises with the image (more waves per launch)."""
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


def main():
    import paper_1703_06503_b200 as pkg

    sus = pkg.CudaBackend(0, flush_l2=False, warmup=3)
    res = {}
    for f in (3, 7, 9, 11):
        for c in top(f, 6):
            for (x, y) in ((8192, 4096), (8192, 8192), (16384, 8192)):
                req = pkg.conv_request(x, y, f, pkg.parse_canonical(c), reps=20)
                rs = sus.evaluate(req)
                tf = (1 + 2 * f * f) * x * y / rs.mean_ms / 1e9
                res[f"{f}|{x}x{y}|{c}"] = [rs.mean_ms, tf, rs.verification]
                print(f, x, y, c, f"{rs.mean_ms * 1e3:.1f} us {tf:.1f} TFLOP/s "
                      f"{8 * x * y / rs.mean_ms / 1e6:.0f} GB/s", rs.verification, flush=True)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    Path(ROOT / "gpurun_out" / "conv_size_probe.json").write_text(json.dumps(res))


if __name__ == "__main__":
    main()
