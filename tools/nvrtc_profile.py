"""Where does the tuning-time NVRTC compile go?  (CPU only; no GPU needed.)

Assembles the same batched program libktc builds for a batch of conv
configurations (compile_service.cpp assemble(), backend.cpp plan_conv()) and
times nvrtcCompileProgram under option variants, optionally with NVRTC's
--time phase breakdown.

  python tools/nvrtc_profile.py --filter 11 --batch 8 --reps 2
"""
import argparse
import ctypes
import random
import re
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
nv = ctypes.CDLL("/usr/local/cuda/lib64/libnvrtc.so")
MARK = "//@@KTC_BODY@@"


def conv_defines(F, X, Y, c):
    XWG, YWG, XWPT, YWPT, LOCAL, VW, PAD, UNR = (c[k] for k in
                                                 ("XWG", "YWG", "XWPT", "YWPT", "LOCAL", "VW", "PAD", "UNR"))
    H, TX, TY = (F - 1) // 2, XWG * XWPT, YWG * YWPT
    d = dict(XWG=XWG, YWG=YWG, XWPT=XWPT, YWPT=YWPT, LOCAL=LOCAL, VW=VW, PAD=PAD if LOCAL else 0,
             UNR=UNR, GUARD=int(X % TX != 0 or Y % TY != 0), OUT_VEC=int(X % VW == 0))
    if LOCAL == 1:
        d["SP"] = TX + 2 * H + PAD
    elif LOCAL == 2:
        PWO = min(TX, 128)
        BW = (PWO + 2 * H + 3) // 4 * 4 + 4 * PAD
        TR = TY + 2 * H
        NB = (TR + 255) // 256
        BH = ((TR + NB - 1) // NB + 7) // 8 * 8
        d.update(PWO=PWO, BW=BW, BH=BH, NB=NB, NP=TX // PWO, PF=BW * NB * BH)
    return d


def space(rng, n):
    out = []
    while len(out) < n:
        c = dict(XWG=rng.choice([8, 16, 32]), YWG=rng.choice([4, 8, 16]), XWPT=rng.choice([1, 2, 4, 8]),
                 YWPT=rng.choice([1, 2, 4, 8]), LOCAL=rng.choice([0, 1, 2]), VW=rng.choice([1, 2, 4, 8]),
                 PAD=rng.choice([0, 1]), UNR=rng.choice([0, 1]))
        if c["XWPT"] % c["VW"] == 0 and c["XWG"] * c["YWG"] <= 1024:
            out.append(c)
    return out


def assemble(text, base, cfgs):
    at = text.index(MARK)
    pre, body = text[:at], text[at:]
    s = [pre]
    for i, d in enumerate(cfgs):
        s.append(f"namespace ktc_k{i} {{")
        s += [f"#define {k} {v}" for k, v in d.items()]
        s.append(f"#define KTC_ENTRY {base}_k{i}")
        s.append(body)
        s += [f"#undef {k}" for k in d] + ["#undef KTC_ENTRY", "}"]
    return "\n".join(s)


def compile_(src, opts):
    prog = ctypes.c_void_p()
    assert nv.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), b"k.cu", 0, None, None) == 0
    arr = (ctypes.c_char_p * len(opts))(*[o.encode() for o in opts])
    t0 = time.perf_counter()
    rc = nv.nvrtcCompileProgram(prog, len(opts), arr)
    dt = time.perf_counter() - t0
    if rc:
        n = ctypes.c_size_t()
        nv.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
        log = ctypes.create_string_buffer(n.value)
        nv.nvrtcGetProgramLog(prog, log)
        raise RuntimeError(log.value.decode()[-2000:])
    n = ctypes.c_size_t()
    nv.nvrtcGetCUBINSize(prog, ctypes.byref(n))
    nv.nvrtcDestroyProgram(ctypes.byref(prog))
    return dt, n.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--filter", type=int, default=3)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--time", action="store_true")
    a = ap.parse_args()
    text = (ROOT / "paper_1703_06503_b200/csrc/kernels/conv.cu").read_bytes().decode()
    rng = random.Random(a.seed)
    base = ["--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true", f"-DFS={a.filter}"]
    variants = {
        "current": base,
        "no-lineinfo": [o for o in base if o != "-lineinfo"],
        "ptx-only(compute_100a)": ["--gpu-architecture=compute_100a"] + base[1:],
        "minimal": base + ["--minimal"],
        "dopt-off?": base + ["--dopt=off"] if False else None,
    }
    cfgs = [conv_defines(a.filter, 8192, 4096, c) for c in space(rng, a.batch * a.reps)]
    for name, opts in variants.items():
        if opts is None:
            continue
        tot = 0.0
        try:
            for r in range(a.reps):
                src = assemble(text, "conv", cfgs[r * a.batch:(r + 1) * a.batch])
                dt, nbytes = compile_(src, opts)
                tot += dt
        except RuntimeError as e:
            print(f"{name:28s} FAILED: {str(e)[:200]}")
            continue
        print(f"{name:28s} {1e3 * tot / (a.reps * a.batch):8.1f} ms/config")
    if a.time:
        src = assemble(text, "conv", cfgs[:a.batch])
        compile_(src, base + ["--time=/tmp/nvrtc_time.csv"])
        print(Path("/tmp/nvrtc_time.csv").read_text()[-3000:])
    # singles vs batch
    t1 = sum(compile_(assemble(text, "conv", [c]), base)[0] for c in cfgs[:a.batch])
    print(f"{'unbatched':28s} {1e3 * t1 / a.batch:8.1f} ms/config")


if __name__ == "__main__":
    main()
