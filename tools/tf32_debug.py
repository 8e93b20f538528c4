"""Characterizes TF32 tcgen05 output errors on small problems (GPU)."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402
from oracle import oracle as O  # noqa: E402

be = pkg.CudaBackend(0)
for (m, n, k) in [(128, 64, 32), (128, 128, 64), (256, 256, 256), (2048, 2048, 2048)]:
    a = O.materialize("uniform:2026", k * m).reshape(k, m)
    b = O.materialize(f"uniform:{2026 ^ 0x9E3779B97F4A7C15}", k * n).reshape(k, n)
    want = (a.astype(np.float64).T @ b.astype(np.float64))
    for bn, bk, st in [(64, 32, 2), (128, 32, 3), (128, 64, 2), (256, 32, 2)]:
        if n % bn or k % bk:
            continue
        r = be.evaluate(pkg.gemm_request(m, n, k, dict(BN=bn, BK=bk, STAGES=st), tf32=True))
        got = be.read_output(m * n).reshape(m, n).astype(np.float64)
        err = np.abs(got - want)
        print(f"variant={os.environ.get('KTC_TF32_DESC_VARIANT', '0')} {m}x{n}x{k} BN={bn} BK={bk} "
              f"ST={st} {r.status} {r.verification} t={r.time_ms:.4f}ms "
              f"max_rel={np.max(err / np.abs(want)):.2e} mean_rel={np.mean(err / np.abs(want)):.2e}",
              flush=True)
        if m == 128 and r.verification == "fail":
            # which (row, col) blocks are wrong, and does got match a
            # transposed / partial-K product?
            bad = err > 1e-2 * np.abs(want)
            print("   bad fraction", bad.mean(), "bad rows", np.unique(np.nonzero(bad)[0])[:8],
                  "bad cols", np.unique(np.nonzero(bad)[1])[:8])
            for kk in (8, 16, 32):
                part = a[:kk].astype(np.float64).T @ b[:kk].astype(np.float64)
                print(f"   rel diff vs first {kk} k: {np.max(np.abs(got - part) / np.abs(want)):.2e}")
            print("   got[0,:4]", got[0, :4], "want", want[0, :4])
            print("   got[:4,0]", got[:4, 0], "want", want[:4, 0])
be.close()
