"""Where does a warm-cache (device-bound) evaluation's time go?  (run under gpurun)

Evaluates 240 conv 3x3 configurations twice through CudaBackend (second pass:
every cubin cached) and prints the mean host-clock split per evaluation.
"""
import random
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402

t = pkg.Tuner.conv(8192, 4096, 3)
order = list(range(5104))
random.Random(5).shuffle(order)
cfgs = [pkg.parse_canonical(t.space_config(i)) for i in order[:240]]
be = pkg.CudaBackend(0)
reqs = [pkg.conv_request(8192, 4096, 3, c, reps=3) for c in cfgs]
for r in reqs:
    be.prefetch(r)
for p in range(2):
    acc = {"compile_ms": 0.0, "load_ms": 0.0, "run_ms": 0.0, "verify_ms": 0.0, "time_ms": 0.0}
    t0 = time.perf_counter()
    for r in reqs:
        res = be.evaluate(r)
        for k in acc:
            acc[k] += getattr(res, k)
    wall = time.perf_counter() - t0
    n = len(reqs)
    print(f"pass {p}: {n / wall:.0f} evals/s, per eval: wall {1e3 * wall / n:.3f} ms, " +
          ", ".join(f"{k} {v / n:.3f}" for k, v in acc.items()), flush=True)
