"""A/B of the SGEMM split-K tail (TAILK) on the tuned winners (run under gpurun).

    python tools/tail_ab.py            # spawns one process per mode

Times each winner of tuned/b200_winners.json (2048^3, 4096^3) with
KTC_GEMM_TAIL=0 and =1: best of 10 flushed launches and mean of 30
back-to-back launches, verified."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child():
    sys.path.insert(0, str(ROOT))
    import paper_1703_06503_b200 as pkg

    table = json.loads((ROOT / "tuned" / "b200_winners.json").read_text())
    be = pkg.CudaBackend(0)
    sus = pkg.CudaBackend(0, flush_l2=False, warmup=3)
    out = {}
    for size in ("2048", "4096"):
        m = int(size)
        cfg = pkg.parse_canonical(table["gemm"][size]["config"])
        req = pkg.gemm_request(m, m, m, cfg, reps=10)
        r = be.evaluate(req)
        req.repetitions = 30
        rs = sus.evaluate(req)
        out[size] = {"best_ms": r.time_ms, "mean_ms": rs.mean_ms, "verified": r.verification,
                     "tflops_mean": 2 * m ** 3 / rs.mean_ms / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
    else:
        res = {}
        for mode in ("0", "1"):
            env = dict(os.environ, KTC_GEMM_TAIL=mode)
            p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True,
                               text=True, timeout=600)
            res["tail=" + mode] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 \
                else p.stderr[-500:]
        print(json.dumps(res, indent=1))
