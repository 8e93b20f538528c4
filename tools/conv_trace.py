"""CTA timeline of tuned conv winners (run under gpurun): where a launch's
time goes (ramp, steady state, drain).

    python tools/conv_trace.py            # spawns a child with KTC_CONV_TRACE set

The diagnostic build (ptxgen_conv TRACE) stores each CTA's start/end
%globaltimer and SM id; one evaluation (warm-up + 1 flushed timed launch)
per case; the timed launch's trace is analysed: CTAs resident over time,
CTA lifetime in the first / middle / last tenth of the launch, time to the
first CTA end, and the drain after the last CTA start."""
import glob
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
CASES = [(7, 8192, 4096, "LOCAL=2;PAD=1;UNR=1;VW=8;XWG=8;XWPT=8;YWG=8;YWPT=4"),
         (7, 8192, 8192, "LOCAL=2;PAD=1;UNR=1;VW=8;XWG=8;XWPT=8;YWG=8;YWPT=4"),
         (3, 8192, 4096, "LOCAL=0;PAD=0;UNR=1;VW=4;XWG=32;XWPT=4;YWG=8;YWPT=4"),
         (11, 8192, 4096, "LOCAL=2;PAD=1;UNR=1;VW=8;XWG=8;XWPT=8;YWG=16;YWPT=4")]


def child(out_dir):
    sys.path.insert(0, str(ROOT))
    import paper_1703_06503_b200 as pkg

    be = pkg.CudaBackend(0)
    for i, (f, x, y, c) in enumerate(CASES):
        r = be.evaluate(pkg.conv_request(x, y, f, pkg.parse_canonical(c), reps=1))
        print(json.dumps({"case": i, "time_ms": r.time_ms, "verified": r.verification}), flush=True)


def analyse(path, time_ms):
    raw = Path(path).read_bytes()
    gx, gy = np.frombuffer(raw[:8], dtype=np.uint32)
    t = np.frombuffer(raw[8:], dtype=np.uint64).reshape(-1, 4).astype(np.float64)
    start, end, sm = t[:, 0], t[:, 1], t[:, 2].astype(int)
    t0 = start.min()
    start, end = (start - t0) / 1e3, (end - t0) / 1e3  # us
    span = end.max()
    life = end - start
    order = np.argsort(start)
    n = len(start)
    dec = lambda a: [float(np.mean(a[order[int(n * lo):int(n * hi)]])) for lo, hi in ((0, .1), (.45, .55), (.9, 1))]  # noqa
    grid = np.linspace(0, span, 200)
    resident = [int(np.sum((start <= g) & (end > g))) for g in grid]
    last_start = start.max()
    per_sm_end = np.array([end[sm == s].max() for s in np.unique(sm)])
    per_sm_first = np.array([start[sm == s].min() for s in np.unique(sm)])
    return {"grid": [int(gx), int(gy)], "ctas": n, "span_us": span, "event_time_us": time_ms * 1e3,
            "first_cta_end_us": float(end.min()), "last_cta_start_us": float(last_start),
            "drain_us": float(span - last_start),
            "sm_first_start_us": [float(per_sm_first.min()), float(per_sm_first.max())],
            "sm_last_end_us": [float(per_sm_end.min()), float(np.median(per_sm_end)), float(per_sm_end.max())],
            "lifetime_us_first_mid_last_tenth": dec(life),
            "max_resident": int(max(resident)),
            "resident_profile": resident[::10]}


def main():
    out = ROOT / "gpurun_out" / "conv_trace"
    out.mkdir(parents=True, exist_ok=True)
    for p in glob.glob(str(out / "*.bin")):
        os.unlink(p)
    env = dict(os.environ, KTC_CONV_TRACE=str(out))
    p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True,
                       timeout=900)
    if p.returncode:
        print(p.stderr[-2000:])
        sys.exit(1)
    runs = [json.loads(line) for line in p.stdout.splitlines() if line.startswith("{")]
    files = sorted(glob.glob(str(out / "conv_trace_*.bin")), key=lambda s: int(s.rsplit("_", 1)[1][:-4]))
    # one trace per evaluation: the buffer holds the last (timed) launch
    res = []
    for i, r in enumerate(runs):
        a = analyse(files[i], r["time_ms"])
        a.update({"filter": CASES[i][0], "image": f"{CASES[i][1]}x{CASES[i][2]}", "config": CASES[i][3]})
        res.append(a)
        print(json.dumps({k: v for k, v in a.items() if k != "resident_profile"}), flush=True)
        print("   resident:", a["resident_profile"], flush=True)
    (ROOT / "gpurun_out" / "conv_trace.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    if "--child" in sys.argv:
        child(None)
    else:
        main()
