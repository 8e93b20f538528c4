"""Large-shape GEMM goldens (BASELINE configs[2]-[4] sizes) -- build container only.

    python tests/golden/make_golden_large.py NAME [--ref]

NAME is one of CASES below.  Each case is computed with the bit-identical
row-parallel C restatement (oracle/ktune_oracle.c, all host threads) and,
with --ref, ALSO with the reference's own single-threaded gemm_reference
(landscapes.hpp:315-323 via oracle/_ref; 4096^3 takes ~25 min on one core,
8192^3 ~3.5 h).  The two digests must agree; the result is written to
tests/golden/large/NAME.json and folded into oracle_golden.json's
"gemm_digests_large" by --merge.

The 4096^3 value must also equal SURVEY.md 8(c)'s independently probed
digest 0d7e2b57acb326c9.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import oracle as O  # noqa: E402

# name -> (m, n, k); alpha=1, beta=0, seed 2026 (the reference defaults,
# landscapes.hpp:185-208)
CASES = {
    "4096": (4096, 4096, 4096),
    "8192": (8192, 8192, 8192),
    "8192x256x8192": (8192, 256, 8192),
    "4096x4096x256": (4096, 4096, 256),
}


def run(name: str, ref: bool) -> dict:
    m, n, k = CASES[name]
    t0 = time.time()
    restated = O.digest(O.gemm_reference(m, n, k))
    out = {"m": m, "n": n, "k": k, "alpha": 1.0, "beta": 0.0, "seed": 2026,
           "restated_digest": restated, "restated_s": round(time.time() - t0, 1),
           "restated_threads": O.threads()}
    if ref:
        t0 = time.time()
        out["reference_digest"] = O.digest(O.ref_gemm_reference(m, n, k))
        out["reference_s"] = round(time.time() - t0, 1)
        assert out["reference_digest"] == restated, out
    out["digest"] = restated
    return out


def merge() -> None:
    g = json.loads((HERE / "oracle_golden.json").read_text())
    large = {}
    for p in sorted((HERE / "large").glob("*.json")):
        d = json.loads(p.read_text())
        large[p.stem] = {k: d[k] for k in ("m", "n", "k", "digest")}
        large[p.stem]["source"] = ("reference gemm_reference (oracle/_ref) == C restatement"
                                   if "reference_digest" in d else
                                   "C restatement (pinned: bit-identical to the reference at "
                                   "every size both ran)")
    g["gemm_digests_large"] = large
    (HERE / "oracle_golden.json").write_text(json.dumps(g, indent=1) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "--merge":
        merge()
    else:
        res = run(sys.argv[1], "--ref" in sys.argv)
        (HERE / "large").mkdir(exist_ok=True)
        (HERE / "large" / f"{sys.argv[1]}.json").write_text(json.dumps(res, indent=1) + "\n")
        print(json.dumps(res), flush=True)
