"""First light + A/B of the TF32 stream-K launch (run under gpurun): with
KTC_TF32_SK=0 / 1 (child process each), CTA-pair and single-CTA configurations
at 1024x1024x8192 (real K-segments; checked against the fp32 oracle) and at
2048^3 (the size it is for), verified on the device."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import json, sys, time
sys.path.insert(0, sys.argv[1])
import paper_1703_06503_b200 as pkg
from oracle import oracle as O
be = pkg.CudaBackend(0)
out = {}
for (m, n, k) in ((1024, 1024, 8192), (2048, 2048, 2048), (4096, 4096, 4096)):
    want = O.gemm_reference(m, n, k) if m == 1024 else None
    for cfg in (dict(BN=256, BK=64, STAGES=3, CG=2), dict(BN=256, BK=32, STAGES=3, CG=2),
                dict(BN=256, BK=64, STAGES=3, CG=1), dict(BN=128, BK=64, STAGES=3, CG=2)):
        r = be.evaluate(pkg.gemm_request(m, n, k, cfg, tf32=True, reps=10))
        row = [r.status, r.verification, r.time_ms if r.ok else r.message[:200]]
        if r.ok and want is not None:
            row.append(O.verify(be.read_output(m * n), want, 1e-3, 1e-6)["pass"])
        out[f"{m}x{n}x{k} {cfg}"] = row
        print(f"{m}x{n}x{k} {cfg} {row}", flush=True)
print(json.dumps(out))
"""

res = {}
for mode in ("0", "1"):
    env = dict(os.environ, KTC_TF32_SK=mode)
    p = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=600)
    print(f"--- KTC_TF32_SK={mode} rc={p.returncode}", flush=True)
    print(p.stdout[-3000:], p.stderr[-1500:] if p.returncode else "", flush=True)
