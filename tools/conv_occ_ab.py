"""Conv register-budget A/B (run under gpurun): the 12 fastest configurations
per filter (profiles/sweep_r01c) timed with each KTC_CONV_MINCTA /
KTC_CONV_BH_EXACT variant (one child process per variant), sustained mean of
30 back-to-back launches and best of 10 flushed, verified.

    python tools/conv_occ_ab.py [--filters 5,7,9,11] [--n 12]
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
VARIANTS = {"base": {}, "mincta": {"KTC_CONV_MINCTA": "1"},
            "mincta+bh": {"KTC_CONV_MINCTA": "1", "KTC_CONV_BH_EXACT": "1"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--filters", default="5,7,9,11")
    ap.add_argument("--n", type=int, default=12)
    ap.add_argument("--variants", help='e.g. "base:;persist:KTC_CONV_PERSIST=1,KTC_CONV_MINCTA=16"')
    a = ap.parse_args()
    variants = VARIANTS
    if a.variants:
        variants = {}
        for item in a.variants.split(";"):
            name, _, envs = item.partition(":")
            variants[name] = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    res = {}
    for name, env in variants.items():
        out = ROOT / "gpurun_out" / f"conv_occ_{name}.json"
        e = dict(os.environ, **env)
        p = subprocess.run([sys.executable, str(ROOT / "tools" / "conv_sustained_ab.py"), "--out", str(out),
                            "--filters", a.filters, "--n", str(a.n)], env=e, capture_output=True,
                           text=True, timeout=1500)
        print(name, p.stdout.strip()[-1500:], p.stderr.strip()[-800:] if p.returncode else "", flush=True)
        res[name] = json.loads(out.read_text()) if out.exists() else None
    for f in a.filters.split(","):
        line = [f"f={f}"]
        for name, r in res.items():
            if not r:
                continue
            ks = [k for k in r if k.startswith(f + "|")]
            bad = sum(1 for k in ks if r[k][2] != "pass")
            line.append(f"{name}: sus {min(r[k][1] for k in ks) * 1e3:.1f} us, "
                        f"flushed {min(r[k][0] for k in ks) * 1e3:.1f} us" + (f" ({bad} NOT VERIFIED)" if bad else ""))
        print(" | ".join(line), flush=True)


if __name__ == "__main__":
    main()
