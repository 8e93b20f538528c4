"""Time a curated SGEMM configuration set (run under gpurun): code-generation A/B.

The set: the 48 fastest rows of the round-1 2048^3 random search
(profiles/sweep_r01/gemm_2048_replay.csv) plus every register-heavy
configuration (MWI*NWI >= 32) with SA=SB=1, STRM=STRN=1 and KWI=8 -- the
region where the winners live.  Env knobs (KTC_GEMM_*) select the variant.

  python tools/gemm_probe.py --size 2048 --out gpurun_out/probe_a.json
  python tools/gemm_probe.py --compare gpurun_out/probe_a.json gpurun_out/probe_b.json
"""
from __future__ import annotations

import argparse
import csv
import itertools
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def valid(c: dict) -> bool:
    MWG, NWG, KWG, MDIMC, NDIMC, MDIMA, NDIMB = (c[k] for k in
                                                 ("MWG", "NWG", "KWG", "MDIMC", "NDIMC", "MDIMA", "NDIMB"))
    VWM, VWN, KWI = c["VWM"], c["VWN"], c["KWI"]
    if MWG % MDIMC or NWG % NDIMC or (MWG // MDIMC) % VWM or (NWG // NDIMC) % VWN or KWG % KWI:
        return False
    nt = MDIMC * NDIMC
    if nt % MDIMA or nt % NDIMB or KWG % (nt // MDIMA) or KWG % (nt // NDIMB):
        return False
    if MWG % (MDIMA * VWM) or NWG % (NDIMB * VWN):
        return False
    return True


def configs() -> list[str]:
    out = []
    rows = [(r["config"], float(r["time_ms"])) for r in
            csv.DictReader(open(ROOT / "profiles" / "sweep_r01" / "gemm_2048_replay.csv"))
            if r["time_ms"] not in ("", "inf", "nan")]
    rows.sort(key=lambda r: r[1])
    out += [c for c, _ in rows[:48]]
    for MWG, NWG, KWG, MDIMC, NDIMC, MDIMA, NDIMB, VWM, VWN in itertools.product(
            (64, 128), (64, 128), (16, 32), (8, 16), (8, 16), (16, 32), (16, 32), (2, 4), (4,)):
        if MDIMA != NDIMB:
            continue
        c = dict(KWG=KWG, KWI=8, MDIMA=MDIMA, MDIMC=MDIMC, MWG=MWG, NDIMB=NDIMB, NDIMC=NDIMC,
                 NWG=NWG, SA=1, SB=1, STRM=1, STRN=1, VWM=VWM, VWN=VWN)
        if (MWG // MDIMC) * (NWG // NDIMC) < 32 or not valid(c):
            continue
        s = ";".join(f"{k}={v}" for k, v in sorted(c.items()))
        if s not in out:
            out.append(s)
    return out


def run(size: int, out: str, limit: int) -> None:
    import paper_1703_06503_b200 as pkg

    be = pkg.CudaBackend(0)
    cfgs = configs()[:limit] if limit else configs()
    mk = lambda c: pkg.gemm_request(size, size, size, pkg.parse_canonical(c), reps=5)  # noqa: E731
    for c in cfgs:
        be.prefetch(mk(c))
    rows = {}
    t0 = time.time()
    for c in cfgs:
        r = be.evaluate(mk(c))
        rows[c] = r.time_ms if r.ok and r.verification == "pass" else None
    wall = time.time() - t0
    ok = {c: t for c, t in rows.items() if t}
    best = min(ok, key=ok.get)
    print(f"size {size}: {len(rows)} configs, {len(ok)} ok, wall {wall:.0f}s, best {best} "
          f"{ok[best]:.4f} ms = {2 * size ** 3 / ok[best] / 1e9:.1f} TFLOP/s", flush=True)
    top = sorted(ok, key=ok.get)[:8]
    for c in top:
        print(f"  {ok[c]:.4f} ms {2 * size ** 3 / ok[c] / 1e9:6.1f} TF  {c}")
    Path(out).write_text(json.dumps({"size": size, "rows": rows, "wall_s": wall}))


def compare(a: str, b: str) -> None:
    A, B = json.loads(Path(a).read_text()), json.loads(Path(b).read_text())
    n = A["size"]
    r = [A["rows"][c] / B["rows"][c] for c in A["rows"] if A["rows"][c] and B["rows"].get(c)]
    ba = min(t for t in A["rows"].values() if t)
    bb = min(t for t in B["rows"].values() if t)
    print(f"best A {2 * n ** 3 / ba / 1e9:.1f} TF  B {2 * n ** 3 / bb / 1e9:.1f} TF; per-config A/B "
          f"median {statistics.median(r):.3f}, B faster on {sum(x > 1.01 for x in r)}, slower on "
          f"{sum(x < 0.99 for x in r)} of {len(r)}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=2048)
    ap.add_argument("--out")
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--compare", nargs=2)
    a = ap.parse_args()
    if a.compare:
        compare(*a.compare)
    else:
        run(a.size, a.out, a.limit)
