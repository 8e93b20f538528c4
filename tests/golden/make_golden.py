"""Regenerates tests/golden/oracle_golden.json from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/libktune_ref.so, which
is compiled from the unmodified headers under /root/reference by
oracle/Makefile).  Everything here is the reference's own output:

  conv_digests   FNV digest of conv_reference, 8192x4096, w=1, seed 2026
                 (landscapes.hpp:146), f = 3..11
  gemm_digests   FNV digest of gemm_reference, alpha=1, beta=0, seed 2026
                 (landscapes.hpp:315); 2048^3 takes ~3 minutes on one core
                 and is included only with --full (the survey's value,
                 e2e6ec9ed745dcf0, is recorded otherwise and cross-checked by
                 the bit-identical C restatement in tests/test_oracle.py)
  small          conv / gemm digests at desk sizes with non-default weights,
                 alphas, betas and seeds
  counts         (raw, constrained, valid) of the composed spaces
  winners        the reference tuner's full search with its synthetic cost
                 model on the B200 device model: rows, best step, best config
"""
from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import oracle as O  # noqa: E402

B200 = {"name": "B200", "max_work_group_total": 1024, "max_work_group_dim": [1024, 1024, 64],
        "local_mem_bytes": 232448}


def main(full: bool) -> None:
    out = {"generator": "tests/golden/make_golden.py (reference headers via oracle/_ref)"}
    out["conv_digests"] = {}
    for f in (3, 5, 7, 9, 11):
        out["conv_digests"][str(f)] = O.digest(O.ref_conv_reference(8192, 4096, f))
        print("conv", f, out["conv_digests"][str(f)], flush=True)
    out["gemm_digests"] = {}
    for m in ((512, 1024, 2048) if full else (512, 1024)):
        out["gemm_digests"][str(m)] = O.digest(O.ref_gemm_reference(m, m, m))
        print("gemm", m, out["gemm_digests"][str(m)], flush=True)
    if not full:
        out["gemm_digests"]["2048"] = "e2e6ec9ed745dcf0"  # SURVEY 8(c), reference run 168 s
    out["small"] = []
    for (x, y, f, w, seed) in [(64, 64, 3, 1.0, 2026), (64, 64, 7, 1.0, 2026), (64, 64, 11, 1.0, 2026),
                               (16, 8, 3, 0.25, 99), (300, 70, 5, 0.5, 7), (1000, 3, 9, 2.0, 1)]:
        out["small"].append({"kind": "conv", "x": x, "y": y, "f": f, "w": w, "seed": seed,
                             "digest": O.digest(O.ref_conv_reference(x, y, f, w, seed))})
    for (m, n, k, a, b, seed) in [(8, 4, 16, 1.5, 0.5, 7), (8, 8, 8, 1.0, 0.0, 2026),
                                  (8, 8, 8, 0.0, 1.0, 2026), (96, 80, 64, 1.0, 0.0, 2026),
                                  (128, 256, 64, 0.5, 2.0, 5), (100, 30, 70, 1.0, 1.0, 3)]:
        out["small"].append({"kind": "gemm", "m": m, "n": n, "k": k, "alpha": a, "beta": b,
                             "seed": seed,
                             "digest": O.digest(O.ref_gemm_reference(m, n, k, a, b, seed))})
    out["counts"] = {}
    jobs = {
        "conv_f3_B200": {"template": "conv", "problem": {"filter": 3}, "device": B200},
        "conv_f11_B200": {"template": "conv", "problem": {"filter": 11}, "device": B200},
        "conv_f7_K40m": {"template": "conv", "problem": {"filter": 7}, "device": "K40m"},
        "conv_f11_K40m": {"template": "conv", "problem": {"filter": 11}, "device": "K40m"},
        "gemm_4096_B200": {"template": "gemm", "problem": {"m": 4096, "n": 4096, "k": 4096},
                           "device": B200},
        "gemm_2048_K40m": {"template": "gemm", "device": "K40m"},
        "gemm_2048_HD7970": {"template": "gemm", "device": "HD7970"},
    }
    for name, job in jobs.items():
        out["counts"][name] = list(O.ref_job_counts(json.dumps(job)))
        print("counts", name, out["counts"][name], flush=True)
    out["winners"] = {}
    with tempfile.TemporaryDirectory() as td:
        for name, job in [
            ("conv_f3_B200_conv_like", {"template": "conv", "problem": {"filter": 3}, "device": B200,
                                        "backend": {"kind": "synthetic", "model": "conv-like"},
                                        "strategy": {"kind": "full"}}),
            ("gemm_4096_B200_gemm_like", {"template": "gemm",
                                          "problem": {"m": 4096, "n": 4096, "k": 4096},
                                          "device": B200,
                                          "backend": {"kind": "synthetic", "model": "gemm-like"},
                                          "strategy": {"kind": "full"}}),
        ]:
            csv = Path(td) / "r.csv"
            idx, t = O.ref_job_run(json.dumps(job), td, str(csv))
            rows = csv.read_bytes().decode().split("\r\n")[1:-1]
            best = rows[idx].split(",")
            out["winners"][name] = {"rows": len(rows), "best_step": int(best[0]),
                                    "best_config": best[1], "best_time_ms": t}
            print("winner", name, out["winners"][name], flush=True)
    (HERE / "oracle_golden.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main("--full" in sys.argv)
