"""Repro for the round-1 TF32 full-search crash (run under gpurun with KTC_SEGV_TRACE=1)."""
import faulthandler
import sys
from pathlib import Path

faulthandler.enable()
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402

for rnd in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t = pkg.Tuner.gemm(2048, 2048, 2048, tf32=(rnd % 2 == 1))
    t.SetVerification(True, rel_tol=1e-3)
    t.SetRepetitions(3)
    if rnd % 2:
        t.UseFullSearch()
    else:
        t.UseRandomSearch(1 / 8192)
    s = t.Tune()
    print(rnd, "rows", s["rows"], "best", t.GetBestResult(), flush=True)
    del t
print("ok")
