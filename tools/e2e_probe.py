"""Where does a fresh tuning job's time go?  (run under gpurun)

Times, for a few fresh conv jobs of CHUNK configurations each (the bench's
e2e step): Tuner construction, Tune() wall, and the summary's compile and
device seconds.

  python tools/e2e_probe.py [--chunk 48] [--jobs 3]
"""
import argparse
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--chunk", type=int, default=48)
ap.add_argument("--jobs", type=int, default=3)
ap.add_argument("--filter", type=int, default=3)
a = ap.parse_args()
order = list(range(5104))
random.Random(99).shuffle(order)
reuse = pkg.Tuner.conv(8192, 4096, a.filter, devices=[0])
reuse.SetVerification(True)
reuse.SetRepetitions(3)
for j in range(a.jobs):
    reuse.SetSubset(order[(50 + j) * a.chunk:(51 + j) * a.chunk])
    t0 = time.perf_counter()
    s = reuse.Tune()
    t1 = time.perf_counter()
    print(f"same tuner, new units {j}: Tune {1e3 * (t1 - t0):.1f} ms (compile {s['compile_s']:.2f} s "
          f"summed, device {s['device_s']:.3f} s) -> {a.chunk / (t1 - t0):.1f} configs/s", flush=True)
for j in range(a.jobs):
    t0 = time.perf_counter()
    t = pkg.Tuner.conv(8192, 4096, a.filter, devices=[0])
    t.SetVerification(True)
    t.SetRepetitions(3)
    t.SetSubset(order[j * a.chunk:(j + 1) * a.chunk])
    t1 = time.perf_counter()
    s = t.Tune()
    t2 = time.perf_counter()
    rows = t.rows()
    t3 = time.perf_counter()
    del t
    t4 = time.perf_counter()
    print(f"job {j}: construct {1e3 * (t1 - t0):.1f} ms, Tune {1e3 * (t2 - t1):.1f} ms "
          f"(compile {s['compile_s']:.2f} s summed, device {s['device_s']:.3f} s), rows "
          f"{1e3 * (t3 - t2):.1f} ms, destroy {1e3 * (t4 - t3):.1f} ms -> "
          f"{len(rows) / (t4 - t0):.1f} configs/s", flush=True)
