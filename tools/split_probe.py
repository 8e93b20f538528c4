"""Probe of K-splitting every SGEMM tile (run under gpurun).

    python tools/split_probe.py [--top 200] [--sizes 2048,...]

For the fastest configurations of the 2048^3 full search (or the tuned
winners at other sizes) times each with the TAILK launch policy and with every
tile cut into s K-ranges (KTC_GEMM_SPLIT=s, one child process per s), best of 5
flushed launches, verified.  Prints one JSON object per (shape, s)."""
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
    ap.add_argument("--top", type=int, default=200)
    ap.add_argument("--shapes", default="2048x2048x2048")
    ap.add_argument("--splits", default="0,1,2,3,4,6,8")
    ap.add_argument("--per-tile", type=int, default=0,
                    help="instead of --top: the N fastest configurations of each (MWG, NWG) tile shape")
    ap.add_argument("--child", nargs=2)
    a = ap.parse_args()
    if a.child:
        child(tuple(int(v) for v in a.child[0].split("x")), json.loads(a.child[1]))
        return
    import numpy as np

    t = np.load(ROOT / "profiles/fullsearch_r01/gemm2048_times.npz")["times"]
    order = np.argsort(np.nan_to_num(t, nan=1e9))
    idx = [int(i) for i in order[:a.top]]
    if a.per_tile:
        sys.path.insert(0, str(ROOT))
        import paper_1703_06503_b200 as pkg

        space = pkg.Tuner.gemm(2048, 2048, 2048)
        count, idx = {}, []
        for i in order[:100000]:
            c = pkg.parse_canonical(space.space_config(int(i)))
            key = (c["MWG"], c["NWG"])
            if count.get(key, 0) < a.per_tile:
                count[key] = count.get(key, 0) + 1
                idx.append(int(i))
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    for shape in a.shapes.split(","):
        m, n, k = (int(v) for v in shape.split("x"))
        res = {}
        for s in a.splits.split(","):
            env = dict(os.environ)
            env.pop("KTC_GEMM_SPLIT", None)
            if s != "0":
                env["KTC_GEMM_SPLIT"] = s
            p = subprocess.run([sys.executable, __file__, "--child", shape, json.dumps(idx)], env=env,
                               capture_output=True, text=True, timeout=1800)
            res[s] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-800:]
        rec = {"shape": shape, "results": res}
        summ = {}
        for s, rows in res.items():
            if isinstance(rows, str):
                summ[s] = rows[-200:]
                continue
            ok = [(ms, i) for i, ms, v in rows if ms is not None and v == "pass"]
            best = min(ok) if ok else None
            summ[s] = {"n": len(rows), "ok": len(ok), "best_ms": best[0] if best else None,
                       "best_index": best[1] if best else None,
                       "tflops": 2 * m * n * k / best[0] / 1e9 if best else None}
        rec["summary"] = summ
        Path(ROOT / "gpurun_out" / f"split_probe_{shape}.json").write_text(json.dumps(rec))
        print(json.dumps({"shape": shape, "summary": summ}), flush=True)


if __name__ == "__main__":
    main()
