"""First-light check of the TF32 CTA-pair kernel (CG=2), in its own process
(run under gpurun with a timeout): a few configurations at small and large
sizes, verified at rel 1e-3 on the device and against the fp32 oracle."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker)

be = pkg.CudaBackend(0)
for (m, n, k) in ((256, 256, 256), (512, 256, 1024), (2048, 2048, 2048)):
    want = O.gemm_reference(m, n, k) if m <= 512 else None
    for cfg in (dict(BN=128, BK=32, STAGES=4, CG=2), dict(BN=256, BK=32, STAGES=4, CG=2),
                dict(BN=64, BK=64, STAGES=3, CG=2), dict(BN=128, BK=32, STAGES=4, CG=1)):
        if n % cfg["BN"]:
            continue
        t0 = time.time()
        r = be.evaluate(pkg.gemm_request(m, n, k, cfg, tf32=True, reps=5))
        line = f"{m}x{n}x{k} {cfg}: {r.status} {r.verification} {r.time_ms if r.ok else r.message[:200]}"
        if r.ok and want is not None:
            rep = O.verify(be.read_output(m * n), want, 1e-3, 1e-6)
            line += f" oracle={'pass' if rep['pass'] else rep}"
        if r.ok and r.time_ms:
            line += f" {2 * m * n * k / r.time_ms / 1e9:.1f} TFLOP/s"
        print(line, f"({time.time() - t0:.1f}s)", flush=True)
