"""Per-segment timeline of the TF32 stream-K launch (diagnostic; run under
gpurun): KTC_TF32_SK=2 forces stream-K at 2048^3, KTC_TF32_SK_TRACE makes the
kernel record globaltimer stamps per CTA (start, per segment: MMA start, last
MMA issued, accumulator ready in the epilogue, TMEM handed back; end)."""
import glob
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def main():
    out = ROOT / "gpurun_out" / "sk_trace"
    out.mkdir(parents=True, exist_ok=True)
    for p in glob.glob(str(out / "*.bin")):
        os.unlink(p)
    code = ("import sys; sys.path.insert(0, '.')\n"
            "import paper_1703_06503_b200 as pkg\n"
            "be = pkg.CudaBackend(0)\n"
            "r = be.evaluate(pkg.gemm_request(2048, 2048, 2048, dict(BN=256, BK=64, STAGES=3, CG=2), tf32=True, reps=3))\n"
            "print(r.status, r.verification, r.time_ms)\n")
    env = dict(os.environ, KTC_TF32_SK="2", KTC_TF32_SK_TRACE=str(out))
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=str(ROOT))
    print(p.stdout, p.stderr[-2000:])
    f = sorted(glob.glob(str(out / "sk_trace_*.bin")))[-1]
    d = np.fromfile(f, dtype=np.uint64).reshape(-1, 16).astype(np.float64)
    t0 = d[:, 0][d[:, 0] > 0].min()
    rel = lambda x: (x - t0) / 1e3 if x > 0 else float("nan")  # noqa: E731
    rows = []
    for c in range(d.shape[0]):
        r = d[c]
        rows.append([c, int(r[15])] + [round(rel(r[i]), 2) for i in (0, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 14)])
    hdr = ["cta", "sm", "start", "mma0_start", "mma0_issued", "epi0_acc", "epi0_done", "mma1_start",
           "mma1_issued", "epi1_acc", "epi1_done", "mma2_start", "mma2_issued", "end"]
    print(" ".join(f"{h:>10s}" for h in hdr))
    for r in rows[:16] + rows[-8:]:
        print(" ".join(f"{v:>10}" for v in r))
    arr = np.array([r[2:] for r in rows], dtype=float)
    print("median per column:", dict(zip(hdr[2:], np.round(np.nanmedian(arr, axis=0), 2))))
    print("max per column:", dict(zip(hdr[2:], np.round(np.nanmax(arr, axis=0), 2))))
    Path(ROOT / "gpurun_out" / "sk_trace.json").write_text(json.dumps({"header": hdr, "rows": rows}))


if __name__ == "__main__":
    main()
