"""Evaluates the tuned winners once each (for ncu captures).

    ncu --set full -k regex:'conv2d_k|gemm_k|gemm_tf32_k' -c 4 -o prof python tools/profile_winners.py
    ncu --metrics gpu__time_duration.sum --csv python tools/profile_winners.py

Reads tuned/b200_winners.json (or gpurun_out/b200_winners.json).
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402


def main():
    which = sys.argv[1:] or ["conv3", "conv11", "gemm", "tf32"]
    for p in (ROOT / "tuned" / "b200_winners.json", ROOT / "gpurun_out" / "b200_winners.json"):
        if p.exists():
            table = json.loads(p.read_text())
            break
    else:
        raise SystemExit("no winners table")
    be = pkg.CudaBackend(0, warmup=1)
    for w in which:
        if w.startswith("conv"):
            f = int(w[4:])
            cfg = table["conv"][str(f)]["config"]
            r = be.evaluate(pkg.conv_request(8192, 4096, f, pkg.parse_canonical(cfg), reps=2))
        elif w.startswith("gemm:"):  # gemm:<size or MxNxK>:<canonical config>
            _, size, cfg = w.split(":", 2)
            m, n, k = (int(size),) * 3 if "x" not in size else (int(v) for v in size.split("x"))
            r = be.evaluate(pkg.gemm_request(m, n, k, pkg.parse_canonical(cfg), reps=2))
        elif w.startswith("tf32:"):  # tf32:<size>:<canonical config>
            _, size, cfg = w.split(":", 2)
            m = int(size)
            r = be.evaluate(pkg.gemm_request(m, m, m, pkg.parse_canonical(cfg), reps=2, tf32=True))
        elif w == "gemm":
            cfg = table["gemm"]["2048"]["config"]
            r = be.evaluate(pkg.gemm_request(2048, 2048, 2048, pkg.parse_canonical(cfg), reps=2))
        else:
            cfg = table["gemm_tf32"]["2048"]["config"]
            r = be.evaluate(pkg.gemm_request(2048, 2048, 2048, pkg.parse_canonical(cfg), reps=2,
                                             tf32=True))
        print(w, cfg, r.status, r.verification, f"{r.time_ms:.4f} ms", flush=True)
    be.close()


if __name__ == "__main__":
    main()
