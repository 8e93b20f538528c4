"""Flag-rate probe for the verifier's fp32 screen on real kernel output (run under gpurun)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402

table = json.loads((ROOT / "tuned" / "b200_winners.json").read_text())
be = pkg.CudaBackend(0)
cfg = pkg.parse_canonical(table["conv"]["3"]["config"])
req = pkg.conv_request(8192, 4096, 3, cfg, reps=1)
r = be.evaluate(req)
cand = be.read_output(8192 * 4096)
ref, _ = be.read_reference(req, 8192 * 4096)
f32 = np.float32
df = np.abs(cand - ref)
mf = np.abs(ref)
ca = np.abs(cand)
pass_sure = df <= f32(0.5) * (f32(1e-4) * mf + f32(1e-6))
exact = ((cand >= 0) == (ref >= 0)) & (ca <= 2 * mf) & (mf <= 2 * ca)
print("n", cand.size, "pass_sure false", int((~pass_sure).sum()), "inexact", int((~exact).sum()),
      "df==0", int((df == 0).sum()), "max df", float(df.max()), "distinct df", len(np.unique(df)))
print("ref min/max", float(ref.min()), float(ref.max()), "mf==0", int((mf == 0).sum()))
# per-thread sequential emulation (lockstep over threads)
n = cand.size
T, blocks = 256, 592
chunk = ((n + blocks - 1) // blocks + 3) & ~3
flags = 0
max_abs = np.full((blocks, T), -1.0)
max_rel = np.full((blocks, T), -1.0)
b = np.arange(blocks)[:, None]
t = np.arange(T)[None, :]
step = 4 * T
k = 0
while True:
    base = b * chunk + 4 * t + k * step
    if base.min() >= n:
        break
    for lane in range(4):
        i = base + lane
        valid = (i < np.minimum(n, (b + 1) * chunk))
        ii = np.where(valid, i, 0)
        c = cand[ii].astype(np.float64)
        rr = ref[ii].astype(np.float64)
        D = np.abs(c - rr)
        M = np.abs(rr)
        dff = df[ii]
        abs_rd = max_abs.astype(np.float32)
        abs_skip = np.where(exact[ii], dff.astype(np.float64) <= max_abs, dff < (max_abs * (1 - 2**-20)))
        with np.errstate(divide="ignore", invalid="ignore"):
            rel = np.where(M > 0, D / M, 0.0)
        rel_skip = np.where((M > 0) & (D > 0), dff.astype(np.float64) < max_rel * (1 - 2**-20) * M,
                            max_rel >= 0)
        need = valid & (~pass_sure[ii] | ~abs_skip | ~rel_skip)
        flags += int(need.sum())
        max_abs = np.where(need & (D > max_abs), D, max_abs)
        max_rel = np.where(need & (rel > max_rel), rel, max_rel)
    k += 1
print("per-lane screen flags", flags, f"{flags / n:.3%}")
