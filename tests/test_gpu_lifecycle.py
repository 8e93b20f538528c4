"""Job lifecycle on one device: a tuner that closes the last backend (and so
releases the primary context) must not invalidate what later jobs reuse.

Regression: the process-wide pinned copies of materialized recipes were
allocated in the primary context; destroying the last tuner released that
context, freed the pinned memory under the cache, and the next job's upload
failed (CUDA_ERROR_INVALID_VALUE) or crashed.  Runs in a subprocess so no
other handle in the test process keeps the context alive.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import paper_1703_06503_b200 as pkg
seq = [("gemm", 256), ("tf32", 256), ("gemm", 256), ("conv", 3), ("conv", 3), ("tf32", 256)]
for kind, size in seq:
    if kind == "conv":
        t = pkg.Tuner.conv(512, 256, size, devices=[0])
        t.SetSubset(list(range(0, 5104, 997)))
    else:
        t = pkg.Tuner.gemm(size, size, size, tf32=(kind == "tf32"), devices=[0])
        t.UseRandomSearch(1 / 4096 if kind == "gemm" else 1.0)
    t.SetVerification(True, rel_tol=1e-3 if kind == "tf32" else 1e-4)
    s = t.Tune()
    rows = t.rows()
    assert rows and all(r.verified in ("pass", "skipped") for r in rows if r.status == "ok"), kind
    assert any(r.status == "ok" and r.verified == "pass" for r in rows), kind
    print(kind, size, len(rows), flush=True)
    del t
print("lifecycle ok")
"""


@pytest.mark.gpu
def test_jobs_survive_primary_context_release():
    env = dict(os.environ, KTC_SEGV_TRACE="1")
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0 and "lifecycle ok" in p.stdout, (p.stdout[-2000:], p.stderr[-3000:])
