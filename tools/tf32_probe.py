"""TF32 tcgen05 variant: full search of its small space at several sizes (run under gpurun)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402

for m in [int(v) for v in (sys.argv[1:] or ["2048", "4096", "8192"])]:
    t = pkg.Tuner.gemm(m, m, m, tf32=True)
    t.SetVerification(True, rel_tol=1e-3)
    t.SetRepetitions(5)
    t.UseFullSearch()
    t0 = time.time()
    t.Tune()
    cfg, ms = t.GetBestResult()
    rows = sorted((r for r in t.rows() if r.time_ms and r.verified == "pass"), key=lambda r: r.time_ms)
    print(f"tf32 {m}^3: best {cfg} {ms:.4f} ms = {2 * m ** 3 / ms / 1e9:.1f} TFLOP/s "
          f"({len(rows)} verified rows, {time.time() - t0:.0f}s)", flush=True)
    for r in rows[:4]:
        print(f"   {r.time_ms:.4f} ms {2 * m ** 3 / r.time_ms / 1e9:7.1f} TF  {r.config}")
