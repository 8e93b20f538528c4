"""The CLTune API on a user kernel (not a built-in template), on the B200:
AddKernel / AddParameter / Div/MulGlobal/LocalSize / AddArgument* /
SetReference (a reference kernel run once on the device) / UseFullSearch /
Tune / GetBestResult.  A deliberately wrong configuration must fail
verification; every other configuration must pass."""
import numpy as np
import pytest

import paper_1703_06503_b200 as pkg

KERNEL = r"""
extern "C" __global__ void axpy(const int n, const float a, const float* __restrict__ x,
                                const float* __restrict__ y, float* __restrict__ out) {
    const int base = (blockIdx.x * blockDim.x + threadIdx.x) * WPT;
#pragma unroll
    for (int w = 0; w < WPT; ++w) {
        const int i = base + w;
        if (i >= n) continue;
        if (BUG && WPT == 4 && w == 3) continue;  // a broken configuration
        out[i] = fmaf(a, x[i], y[i]);
    }
}
"""

REFERENCE = r"""
extern "C" __global__ void axpy_ref(const int n, const float a, const float* __restrict__ x,
                                    const float* __restrict__ y, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a * x[i] + y[i];
}
"""


def _tuner(tmp_path, n):
    src = tmp_path / "axpy.cu"
    src.write_text(KERNEL)
    ref = tmp_path / "axpy_ref.cu"
    ref.write_text(REFERENCE)
    t = pkg.Tuner(devices=[0])
    t.AddKernel(str(src), "axpy", [n], [1])
    t.AddParameter("WPT", [1, 2, 4])
    t.AddParameter("LS", [64, 128, 256])
    t.AddParameter("BUG", [0, 1])
    t.DivGlobalSize(["WPT"])
    t.MulLocalSize(["LS"])
    t.AddArgumentScalar(n, "i32")
    t.AddArgumentScalar(2.5, "f32")
    t.AddArgumentInput(n, fill="uniform:7")
    t.AddArgumentInput(n, fill="uniform:8")
    t.AddArgumentOutput(n, fill="constant:0")
    return t, ref


@pytest.mark.gpu
def test_custom_kernel_set_reference_full_search(tmp_path):
    n = 1 << 20
    t, ref = _tuner(tmp_path, n)
    t.SetReference(str(ref), "axpy_ref", [n], [128])
    t.SetVerification(True)
    t.SetRepetitions(3)
    t.UseFullSearch()
    t.Tune()
    rows = t.rows()
    assert len(rows) == 18
    for r in rows:
        p = pkg.parse_canonical(r.config)
        broken = p["BUG"] == 1 and p["WPT"] == 4
        assert r.status == "ok", r
        assert r.verified == ("fail" if broken else "pass"), r
    cfg, ms = t.GetBestResult()
    best = pkg.parse_canonical(cfg)
    assert ms > 0 and not (best["BUG"] == 1 and best["WPT"] == 4)


@pytest.mark.gpu
def test_custom_kernel_host_reference_outputs(tmp_path):
    """SetReferenceOutputs: the reference as host arrays (ktune's reference callback)."""
    n = 1 << 16
    t, _ = _tuner(tmp_path, n)
    # The same recipes the backend materializes (uniform:7, uniform:8).
    from oracle import oracle as O  # checker only

    x = O.materialize("uniform:7", n)
    y = O.materialize("uniform:8", n)
    t.SetReferenceOutputs([(np.float32(2.5) * x + y).astype(np.float32)])
    t.SetVerification(True)
    t.UseFullSearch()
    t.Tune()
    def expect(r):
        p = pkg.parse_canonical(r.config)
        return "fail" if p["BUG"] == 1 and p["WPT"] == 4 else "pass"

    bad = [r for r in t.rows() if r.verified != expect(r)]
    assert not bad, bad[:3]
