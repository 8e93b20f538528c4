"""Stream-K A/B for the SGEMM family (run under gpurun): the N fastest
2048^3 full-search configurations of every (MWG, NWG) tile shape, timed with
KTC_GEMM_SK=0 (whole tiles) and =1 (stream-K where tiles land unevenly on
the SMs), best of 5 flushed launches, verified, at each shape given.

    python tools/sk_probe.py [--per-tile 8] [--shapes 2048x2048x2048,...]
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(shape, idx):
    sys.path.insert(0, str(ROOT))
    import paper_1703_06503_b200 as pkg

    m, n, k = shape
    space = pkg.Tuner.gemm(2048, 2048, 2048)
    be = pkg.CudaBackend(0)
    out = []
    for i in idx:
        cfg = pkg.parse_canonical(space.space_config(i))
        if m % cfg["MWG"] or n % cfg["NWG"] or k % cfg["KWG"]:
            continue
        r = be.evaluate(pkg.gemm_request(m, n, k, cfg, reps=5))
        out.append([i, r.time_ms if r.ok else None, r.verification])
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--per-tile", type=int, default=8)
    ap.add_argument("--shapes", default="2048x2048x2048")
    ap.add_argument("--variants", default="0:KTC_GEMM_SK=0;1:KTC_GEMM_SK=1",
                    help='"name:ENV=V,ENV2=V;name2:..." (default: stream-K off / on)')
    ap.add_argument("--child", nargs=2)
    a = ap.parse_args()
    if a.child:
        child(tuple(int(v) for v in a.child[0].split("x")), json.loads(a.child[1]))
        return
    import numpy as np

    sys.path.insert(0, str(ROOT))
    import paper_1703_06503_b200 as pkg

    t = np.load(ROOT / "profiles/fullsearch_r01/gemm2048_times.npz")["times"]
    order = np.argsort(np.nan_to_num(t, nan=1e9))
    space = pkg.Tuner.gemm(2048, 2048, 2048)
    count, idx = {}, []
    for i in order[:200000]:
        c = pkg.parse_canonical(space.space_config(int(i)))
        key = (c["MWG"], c["NWG"])
        if count.get(key, 0) < a.per_tile:
            count[key] = count.get(key, 0) + 1
            idx.append(int(i))
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    for shape in a.shapes.split(","):
        m, n, k = (int(v) for v in shape.split("x"))
        res = {}
        variants = {}
        for item in a.variants.split(";"):
            name, _, envs = item.partition(":")
            variants[name] = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
        for mode, extra in variants.items():
            env = dict(os.environ, **extra)
            p = subprocess.run([sys.executable, __file__, "--child", shape, json.dumps(idx)], env=env,
                               capture_output=True, text=True, timeout=1800)
            res[mode] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-800:]
        per = {}
        for mode, rows in res.items():
            if isinstance(rows, str):
                continue
            for i, ms, v in rows:
                c = pkg.parse_canonical(space.space_config(i))
                key = f"{c['MWG']}x{c['NWG']}"
                if ms is not None and v == "pass":
                    per.setdefault(key, {}).setdefault(mode, []).append((ms, i))
        summ = {key: {mode: {"best_ms": min(v)[0], "index": min(v)[1],
                             "tflops": 2 * m * n * k / min(v)[0] / 1e9} for mode, v in d.items()}
                for key, d in per.items()}
        bad = {mode: [r for r in rows if r[2] != "pass"] for mode, rows in res.items()
               if not isinstance(rows, str)}
        errs = {mode: rows for mode, rows in res.items() if isinstance(rows, str)}
        rec = {"shape": shape, "per_tile": summ, "not_verified": bad, "errors": errs, "results": res}
        Path(ROOT / "gpurun_out" / f"sk_probe_{shape}.json").write_text(json.dumps(rec))
        print(json.dumps({"shape": shape, "per_tile": summ, "not_verified": bad, "errors": errs}), flush=True)


if __name__ == "__main__":
    main()
