"""Evaluates a fixed set of configurations of every kernel family at small
shapes, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_configs.py

conv: LOCAL 0/1/2 (incl. the TMA + mbarrier halo path), PAD, UNR, VW,
ragged images (GUARD epilogue); SGEMM: SA/SB staging (cp.async double
buffer), STRM/STRN, VW; TF32 tcgen05 (TMA ring, mbarriers, TMEM); plus the
builtin kernels (device references, verifier, L2 flush).  Each row must be
ok + verified pass.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1703_06503_b200 as pkg  # noqa: E402

CONV = [
    dict(XWG=32, YWG=8, XWPT=1, YWPT=8, LOCAL=0, VW=1, PAD=0, UNR=1),
    dict(XWG=32, YWG=8, XWPT=4, YWPT=4, LOCAL=0, VW=4, PAD=0, UNR=1),
    dict(XWG=16, YWG=8, XWPT=2, YWPT=2, LOCAL=0, VW=2, PAD=0, UNR=0),
    dict(XWG=32, YWG=8, XWPT=2, YWPT=4, LOCAL=1, VW=2, PAD=0, UNR=1),
    dict(XWG=64, YWG=8, XWPT=8, YWPT=8, LOCAL=1, VW=8, PAD=1, UNR=0),
    dict(XWG=32, YWG=16, XWPT=2, YWPT=4, LOCAL=2, VW=2, PAD=1, UNR=1),
    dict(XWG=16, YWG=8, XWPT=4, YWPT=4, LOCAL=2, VW=4, PAD=0, UNR=1),
    dict(XWG=8, YWG=8, XWPT=8, YWPT=4, LOCAL=2, VW=8, PAD=1, UNR=1),
    dict(XWG=8, YWG=64, XWPT=8, YWPT=8, LOCAL=2, VW=4, PAD=0, UNR=1),
    dict(XWG=8, YWG=8, XWPT=1, YWPT=1, LOCAL=1, VW=1, PAD=1, UNR=0),
]
GEMM_NAMES = "MWG NWG KWG MDIMC NDIMC SA SB MDIMA NDIMB STRM STRN VWM VWN KWI".split()
GEMM = [(128, 128, 16, 16, 16, 1, 1, 32, 16, 1, 0, 2, 1, 8),
        (64, 64, 32, 8, 16, 1, 1, 32, 32, 1, 0, 2, 2, 8),
        (128, 128, 32, 16, 16, 1, 1, 32, 32, 0, 1, 4, 4, 2),
        (64, 64, 16, 8, 8, 1, 1, 8, 16, 1, 1, 4, 4, 8),
        (128, 128, 128, 8, 8, 1, 1, 8, 8, 1, 1, 8, 8, 8),
        (32, 32, 32, 32, 32, 0, 1, 32, 32, 0, 1, 1, 1, 2),
        (64, 64, 64, 16, 16, 1, 1, 16, 8, 0, 1, 4, 4, 8),
        (64, 128, 16, 8, 8, 1, 1, 8, 16, 1, 1, 4, 8, 8),
        (16, 16, 16, 8, 8, 0, 0, 8, 8, 0, 0, 1, 1, 2)]
TF32 = [dict(BN=64, BK=32, STAGES=2), dict(BN=128, BK=32, STAGES=4), dict(BN=256, BK=32, STAGES=2),
        dict(BN=128, BK=64, STAGES=3)]


def main() -> int:
    be = pkg.CudaBackend(0, warmup=0, flush_l2=False)
    bad = 0
    n = 0

    def run(req, what):
        nonlocal bad, n
        r = be.evaluate(req)
        n += 1
        ok = r.ok and r.verification == "pass"
        bad += not ok
        print(f"{'ok  ' if ok else 'FAIL'} {what} {r.status} {r.verification} {r.message[:120]}",
              flush=True)

    for (x, y, f) in [(256, 128, 3), (264, 72, 7), (512, 64, 11)]:
        for cfg in CONV:
            req = pkg.conv_request(x, y, f, cfg)
            req.global_size = (-(-x // cfg["XWPT"]), -(-y // cfg["YWPT"]))
            run(req, f"conv {x}x{y} f={f} {cfg}")
    for (m, nn, k) in [(256, 256, 128), (128, 384, 256)]:
        for row in GEMM:
            cfg = dict(zip(GEMM_NAMES, row))
            run(pkg.gemm_request(m, nn, k, cfg, alpha=1.5, beta=0.5), f"gemm {m}x{nn}x{k} {cfg}")
    for cfg in TF32:
        run(pkg.gemm_request(256, 256, 256, cfg, tf32=True), f"tf32 256^3 {cfg}")
    be.close()
    print(f"{n} evaluations, {bad} not ok/pass")
    return 1 if bad else 0


if __name__ == "__main__" and "--control" not in sys.argv:
    sys.exit(main())


CONTROL = r"""
extern "C" __global__ void oob(const int n, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= n) out[i] = 1.0f;   // i == n writes one element past the buffer
}
"""


def control() -> int:
    """Negative control: a custom kernel that writes one float past its
    output buffer.  Under memcheck this run must report an invalid write
    (proves the runtime-loaded cubins are instrumented)."""
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        src = Path(td) / "oob.cu"
        src.write_text(CONTROL)
        n = 1 << 20  # a whole number of blocks: out[n] lands right after the buffer
        t = pkg.Tuner(devices=[0], flush_l2=False)
        t.AddKernel(str(src), "oob", [n + 1], [1])
        t.AddParameter("LS", [128])
        t.MulLocalSize(["LS"])
        t.AddArgumentScalar(n, "i32")
        t.AddArgumentOutput(n, fill="constant:0")
        t.UseFullSearch()
        t.Tune()
        for r in t.rows():
            print("control row:", r.status, r.message[:160])
    return 0


if __name__ == "__main__" and "--control" in sys.argv:
    sys.exit(control())
