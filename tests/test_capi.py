"""The C-ABI library (CPU): loads without a GPU driver, exports every entry
point include/ktc.h declares, compiles both kernel families with NVRTC for
sm_100a, and maps failures to codes instead of crashing."""
import re
import sys
from pathlib import Path

import pytest

import paper_1703_06503_b200 as pkg
from paper_1703_06503_b200 import _ktc as K

ROOT = Path(__file__).resolve().parent.parent
KERNELS = ROOT / "paper_1703_06503_b200" / "csrc" / "kernels"


def header_functions() -> list[str]:
    text = (ROOT / "include" / "ktc.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ktc_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(built):
    import ctypes as C

    lib = C.CDLL(str(K.LIB_PATH))
    names = header_functions()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers exactly the header
    assert sorted(K.exported_symbols()) == names


def test_no_device_is_an_error_code_not_a_crash(built):
    import ctypes as C

    if pkg.device_count() > 0:
        pytest.skip("host has a GPU")
    h = C.c_void_p()
    rc = pkg.lib().ktc_open(0, C.byref(h))
    assert rc == 2  # KTC_ERR_NO_DRIVER
    assert "libcuda" in K.last_error()


def _conv_defines(f, XWG, YWG, XWPT, YWPT, LOCAL, VW, PAD, UNR):
    H, TX, TY = (f - 1) // 2, XWG * XWPT, YWG * YWPT
    d = dict(FS=f, XWG=XWG, YWG=YWG, XWPT=XWPT, YWPT=YWPT, LOCAL=LOCAL, VW=VW,
             PAD=PAD if LOCAL else 0, UNR=UNR, GUARD=0, OUT_VEC=1)
    if LOCAL == 1:
        d["SP"] = TX + 2 * H + PAD
    if LOCAL == 2:
        pwo = min(TX, 128)
        bw = (pwo + 2 * H + 3) // 4 * 4 + 4 * PAD
        tr = TY + 2 * H
        nb = (tr + 255) // 256
        bh = ((tr + nb - 1) // nb + 7) // 8 * 8
        d.update(PWO=pwo, BW=bw, BH=bh, NB=nb, NP=TX // pwo, PF=bw * nb * bh)
    return [f"-D{k}={v}" for k, v in d.items()]


@pytest.mark.parametrize("cfg", [
    (3, 32, 8, 1, 8, 0, 1, 0, 1), (7, 32, 16, 2, 4, 2, 2, 1, 1), (5, 64, 8, 4, 4, 1, 4, 1, 0),
    (9, 8, 64, 8, 8, 2, 4, 0, 1), (3, 16, 16, 8, 2, 1, 8, 0, 1),
])
def test_nvrtc_compiles_conv_family_for_sm100a(built, cfg):
    cubin = K.compile_source((KERNELS / "conv.cu").read_text(), _conv_defines(*cfg))
    assert cubin[:4] == b"\x7fELF"


@pytest.mark.parametrize("row", [(128, 128, 16, 16, 16, 1, 1, 32, 16, 1, 0, 2, 1, 8),
                                 (16, 16, 16, 8, 8, 0, 0, 8, 8, 0, 0, 1, 1, 2),
                                 (64, 32, 64, 8, 32, 1, 0, 16, 8, 0, 1, 8, 1, 2)])
@pytest.mark.parametrize("dbuf", [0, 1])
def test_nvrtc_compiles_gemm_family_for_sm100a(built, row, dbuf):
    names = "MWG NWG KWG MDIMC NDIMC SA SB MDIMA NDIMB STRM STRN VWM VWN KWI".split()
    cubin = K.compile_source((KERNELS / "gemm.cu").read_text(),
                             [f"-D{k}={v}" for k, v in zip(names, row)] + [f"-DDBUF={dbuf}"])
    assert cubin[:4] == b"\x7fELF"


def test_compile_error_returns_log(built):
    with pytest.raises(K.KtcError) as e:
        K.compile_source("extern \"C\" __global__ void k() { undefined_thing(); }", [])
    assert e.value.code == 5 and "undefined_thing" in str(e.value)


def test_digest_matches_reference_format(built):
    import ctypes as C

    import numpy as np

    a = np.arange(10, dtype=np.float32)
    L = pkg.lib()
    d = L.ktc_digest_words(a.ctypes.data, a.size)
    buf = C.create_string_buffer(17)
    L.ktc_digest_hex(d, buf)
    from oracle import oracle as O

    assert buf.value.decode() == O.digest(a)


def _sass(cubin: bytes, tmp_path) -> str:
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    p = tmp_path / "k.cubin"
    p.write_bytes(cubin)
    return subprocess.run([tool, "-sass", str(p)], capture_output=True, text=True, check=True).stdout


@pytest.mark.parametrize("f2", [0, 1])
def test_gemm_outer_product_issues_packed_ffma2(built, tmp_path, f2):
    """F2=1 (the default): the 8x8 register tile is 32 FFMA2 per k step, not 64 FFMA."""
    names = "MWG NWG KWG MDIMC NDIMC SA SB MDIMA NDIMB STRM STRN VWM VWN KWI".split()
    row = (128, 128, 32, 16, 16, 1, 1, 16, 16, 1, 1, 4, 4, 8)
    cubin = K.compile_source((KERNELS / "gemm.cu").read_text(),
                             [f"-D{k}={v}" for k, v in zip(names, row)] + ["-DDBUF=1", f"-DF2={f2}"])
    sass = _sass(cubin, tmp_path)
    n2 = len(re.findall(r"\bFFMA2\b", sass))
    n1 = len(re.findall(r"\bFFMA\b", sass))
    if f2:
        assert n2 == 8 * 64 // 2 and n1 <= 64  # KWI=8 steps x 64 FMAs, paired; scalar only in the beta epilogue
    else:
        assert n2 == 0 and n1 >= 8 * 64


def test_conv_unrolled_rows_issue_packed_ffma2(built, tmp_path):
    """CF2=1 (default): 11x11 taps, YWPT=4 rows pair into FFMA2; edge tap rows stay scalar."""
    opts = _conv_defines(11, 16, 8, 4, 4, 2, 4, 0, 1)
    sass = _sass(K.compile_source((KERNELS / "conv.cu").read_text(), opts), tmp_path)
    n2 = len(re.findall(r"\bFFMA2\b", sass))
    n1 = len(re.findall(r"\bFFMA\b", sass))
    # 4 rows x 121 taps x 4 columns = 1936 FMAs: 2 row pairs x 10 inner tap rows
    # x 11 x 4 = 880 FFMA2 and 2 x 2 edge rows x 11 x 4 = 176 FFMA.
    assert (n2, n1) == (880, 176)
    sass0 = _sass(K.compile_source((KERNELS / "conv.cu").read_text(), opts + ["-DCF2=0"]), tmp_path)
    assert len(re.findall(r"\bFFMA2\b", sass0)) == 0


@pytest.mark.parametrize("cfg", [
    (3, 32, 8, 1, 8, 0, 1, 0, 1), (7, 32, 16, 2, 4, 2, 2, 1, 1), (5, 64, 8, 4, 4, 1, 4, 1, 0),
    (9, 8, 64, 8, 8, 2, 4, 0, 1), (3, 16, 16, 8, 2, 1, 8, 0, 1), (11, 16, 8, 4, 4, 2, 4, 0, 1),
    (11, 8, 8, 2, 2, 2, 2, 1, 0), (3, 64, 8, 8, 8, 2, 8, 1, 1),
])
def test_conv_ptx_codegen_compiles_and_matches_fma_counts(built, tmp_path, cfg):
    """The direct PTX generator (the conv family's tuning-time code path)
    compiles every mode with ptxas and issues the same FFMA/FFMA2 as conv.cu."""
    d = _conv_defines(*cfg)
    gen, ptx = K.codegen_conv([x[2:] for x in d])
    assert gen[:4] == b"\x7fELF" and ".entry conv2d_k0" in ptx
    ref = K.compile_source((KERNELS / "conv.cu").read_text(), d)
    count = lambda s, op: len(re.findall(rf"\b{op}\b", s))  # noqa: E731
    sg, sr = _sass(gen, tmp_path), _sass(ref, tmp_path)
    assert (count(sg, "FFMA2"), count(sg, "FFMA")) == (count(sr, "FFMA2"), count(sr, "FFMA"))


@pytest.mark.parametrize("row", [(128, 128, 16, 16, 16, 1, 1, 32, 16, 1, 0, 2, 1, 8),
                                 (16, 16, 16, 8, 8, 0, 0, 8, 8, 0, 0, 1, 1, 2),
                                 (64, 32, 64, 8, 32, 1, 0, 16, 8, 0, 1, 8, 1, 2),
                                 (64, 64, 32, 16, 8, 1, 1, 32, 8, 0, 1, 4, 4, 8)])
@pytest.mark.parametrize("dbuf", [0, 1])
def test_gemm_ptx_codegen_matches_instruction_mix(built, tmp_path, row, dbuf):
    """ptxgen_gemm emits the gemm.cu kernel: same FFMA2 / FFMA / cp.async counts."""
    names = "MWG NWG KWG MDIMC NDIMC SA SB MDIMA NDIMB STRM STRN VWM VWN KWI".split()
    d = [f"{k}={v}" for k, v in zip(names, row)] + [f"DBUF={dbuf}", "OCC=1", "F2=1"]
    gen, ptx = K.codegen_gemm(d)
    assert gen[:4] == b"\x7fELF" and ".entry gemm_k0" in ptx
    ref = K.compile_source((KERNELS / "gemm.cu").read_text(), ["-D" + x for x in d])
    count = lambda s, op: len(re.findall(rf"\b{op}\b", s))  # noqa: E731
    sg, sr = _sass(gen, tmp_path), _sass(ref, tmp_path)
    for op in ("FFMA2", "FFMA", "LDGSTS"):
        assert count(sg, op) == count(sr, op), op


@pytest.mark.parametrize("n,seed", [(0, 1), (1000, 7), (4 * 2**20 - 1, 2026), (4 * 2**20, 2026),
                                    (9 * 2**20 + 17, 12345),
                                    (8194 * 4098, 2026),                      # configs[0] image
                                    (2**22, 2026 ^ 0x9E3779B97F4A7C15)])       # GEMM B recipe
def test_parallel_uniform_recipe_is_bit_identical(built, n, seed):
    """ktc_fill_uniform_f32 (mt19937_64 jump-ahead over host threads) equals
    the sequential reference stream (arguments.hpp:126-180) bit for bit."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as O

    out = np.empty(max(1, n), np.float32)
    for threads in (1, 3, 16):
        assert pkg.lib().ktc_fill_uniform_f32(seed & (2**64 - 1), out.ctypes.data, n, threads) == 0
        want = O.materialize(f"uniform:{seed}", n)
        assert np.array_equal(out[:n].view(np.uint32), want.view(np.uint32)), threads


def test_isolated_backend_worker_starts_and_reports_no_device(built):
    """The isolated backend spawns ktc-worker; without a GPU the worker's
    backend_open fails and the parent returns that error (no hang, no crash)."""
    import subprocess

    worker = Path(pkg.lib()._name).parent / "ktc-worker"
    assert worker.exists()
    if pkg.device_count() > 0:
        pytest.skip("covered by the GPU fault tests")
    code = ("import paper_1703_06503_b200 as p\n"
            "try:\n    p.CudaBackend(0, isolate=True)\n    print('opened')\n"
            "except p.KtcError as e:\n    print('error', e)\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                         cwd=str(Path(__file__).resolve().parent.parent))
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("error"), out.stdout
