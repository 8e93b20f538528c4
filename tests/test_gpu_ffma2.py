"""Packed FFMA2 (gemm.cu F2, conv.cu CF2) is bit-identical to scalar FFMA.

Each FFMA2 lane is a round-to-nearest fp32 FMA, the same operation fmaf
performs, applied in the same per-output order -- so switching the
implementation must not change a single output bit.  The switch is read
once per process (KTC_GEMM_F2 / KTC_CONV_F2), so each variant runs in its
own subprocess and reports the FNV digests of its outputs.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import paper_1703_06503_b200 as pkg
be = pkg.CudaBackend(0, digest_outputs=True)
out = {}
convs = [(11, dict(XWG=16, YWG=8, XWPT=4, YWPT=4, LOCAL=2, VW=4, PAD=0, UNR=1)),
         (7, dict(XWG=8, YWG=8, XWPT=8, YWPT=4, LOCAL=2, VW=8, PAD=1, UNR=1)),
         (5, dict(XWG=32, YWG=8, XWPT=2, YWPT=8, LOCAL=0, VW=2, PAD=0, UNR=1)),
         (3, dict(XWG=16, YWG=16, XWPT=4, YWPT=2, LOCAL=1, VW=4, PAD=1, UNR=1))]
for f, cfg in convs:
    r = be.evaluate(pkg.conv_request(1024, 512, f, cfg))
    out[f"conv{f}"] = [r.status, r.verification, r.digests]
gemms = [dict(MWG=128, NWG=128, KWG=32, MDIMC=16, NDIMC=16, SA=1, SB=1, MDIMA=16, NDIMB=16,
              STRM=1, STRN=1, VWM=4, VWN=4, KWI=8),
         dict(MWG=64, NWG=32, KWG=16, MDIMC=8, NDIMC=32, SA=1, SB=0, MDIMA=16, NDIMB=16,
              STRM=0, STRN=1, VWM=2, VWN=1, KWI=2)]
for i, cfg in enumerate(gemms):
    r = be.evaluate(pkg.gemm_request(256, 384, 512, cfg, alpha=1.5, beta=0.5))
    out[f"gemm{i}"] = [r.status, r.verification, r.digests]
print(json.dumps(out))
"""


def run_variant(f2: str) -> dict:
    env = dict(os.environ, KTC_GEMM_F2=f2, KTC_CONV_F2=f2)
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_ffma2_outputs_bit_identical_to_scalar_fma():
    packed, scalar = run_variant("1"), run_variant("0")
    for k, (st, ver, dig) in packed.items():
        assert st == "ok" and ver == "pass", (k, st, ver)
        assert dig and dig == scalar[k][2], (k, dig, scalar[k])
