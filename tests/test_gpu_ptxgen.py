"""The direct PTX generators (ptxgen_conv.cpp / ptxgen_gemm.cpp, the default
tuning-time code paths) emit the same kernels as kernels/conv.cu and
kernels/gemm.cu through NVRTC: for every sampled configuration -- conv: all
LOCAL modes, UNR 0/1, vector widths, PAD, ragged images (GUARD); SGEMM: SA/SB,
DBUF and register staging, STRM/STRN, vector widths, alpha/beta, rectangular
shapes -- the output digests of the two builds are identical, and both pass
device verification.  The code path is chosen once per process
(KTC_CONV_CODEGEN / KTC_GEMM_CODEGEN), so each runs in its own subprocess.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import json, random, sys
sys.path.insert(0, sys.argv[1])
import paper_1703_06503_b200 as pkg
be = pkg.CudaBackend(0, digest_outputs=True)
out = {}
space = pkg.Tuner.conv(1024, 512, 3)
_, _, n = space.space_counts()
rng = random.Random(42)
idx = rng.sample(range(n), 40)
for f, (x, y) in ((3, (1024, 512)), (5, (520, 300)), (7, (1024, 512)), (11, (520, 300))):
    for i in idx:
        cfg = pkg.parse_canonical(space.space_config(i))
        req = pkg.conv_request(x, y, f, cfg)
        req.global_size = (-(-x // cfg["XWPT"]), -(-y // cfg["YWPT"]))
        r = be.evaluate(req)
        out[f"{f}|{x}x{y}|{space.space_config(i)}"] = [r.status, r.verification, r.digests]
gspace = pkg.Tuner.gemm(512, 512, 512)
_, _, gn = gspace.space_counts()
for i in rng.sample(range(gn), 60):
    cfg = pkg.parse_canonical(gspace.space_config(i))
    for (m, n, k, a, b) in ((512, 512, 512, 1.0, 0.0), (256, 384, 640, 1.5, 0.5)):
        if m % cfg["MWG"] or n % cfg["NWG"] or k % cfg["KWG"]:
            continue
        r = be.evaluate(pkg.gemm_request(m, n, k, cfg, alpha=a, beta=b))
        out[f"gemm|{m}x{n}x{k}|{a}|{b}|{gspace.space_config(i)}"] = [r.status, r.verification, r.digests]
print(json.dumps(out))
"""


def run(codegen: str) -> dict:
    # The split-K tail (a launch-time policy of the generated SGEMM only)
    # changes the accumulation order of split tiles; compare single chains.
    env = dict(os.environ, KTC_CONV_CODEGEN=codegen, KTC_GEMM_CODEGEN=codegen, KTC_GEMM_TAIL="0")
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=1500)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_ptx_codegen_matches_nvrtc_bit_for_bit():
    gen, ref = run("ptx"), run("nvrtc")
    assert gen.keys() == ref.keys()
    bad = []
    for k, (st, ver, dig) in gen.items():
        rst, rver, rdig = ref[k]
        if st != rst or ver != rver or dig != rdig:
            bad.append((k, (st, ver, dig), (rst, rver, rdig)))
        elif st == "ok" and ver != "pass":
            bad.append((k, "verification", ver))
    assert not bad, bad[:5]
    assert sum(1 for k, v in gen.items() if v[0] == "ok" and not k.startswith("gemm")) > 100
    assert sum(1 for k, v in gen.items() if v[0] == "ok" and k.startswith("gemm")) > 50

