"""The C-ABI library (CPU): loads without a GPU driver, exports every entry
point include/ktc.h declares, compiles both kernel families with NVRTC for
sm_100a, and maps failures to codes instead of crashing."""
import re
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
