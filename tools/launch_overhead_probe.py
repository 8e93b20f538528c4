"""How much of a tuned kernel's event time is launch overhead? (run under gpurun)

    python tools/launch_overhead_probe.py

For each winner of tuned/b200_winners.json (conv filters at 8192x4096, SGEMM
and TF32 at their sizes) and for a one-wave conv (64x64) as the floor:
  flushed   best of 10 launches, each after an L2 flush, own event pair (tuner)
  per_event mean of 30 back-to-back launches, own event pair each (round-1/2 roofline)
  stream    mean of 30 back-to-back launches between ONE event pair (flush_l2=2)
The conv trace (tools/conv_trace.py) showed the CTAs of one 7x7 launch span
57.1 us of a 63.4 us event time."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1703_06503_b200 as pkg  # noqa: E402


def main():
    table = json.loads((ROOT / "tuned" / "b200_winners.json").read_text())
    fl = pkg.CudaBackend(0)
    pe = pkg.CudaBackend(0, flush_l2=False, warmup=3)
    st = pkg.CudaBackend(0, warmup=3, stream_timing=True)
    cases = [("conv3_64x64", pkg.conv_request(64, 64, 3, pkg.parse_canonical(table["conv"]["3"]["config"])))]
    for f in ("3", "5", "7", "9", "11"):
        cases.append((f"conv{f}", pkg.conv_request(8192, 4096, int(f), pkg.parse_canonical(table["conv"][f]["config"]))))
    for size, g in table["gemm"].items():
        m, n, k = ((int(size),) * 3) if "x" not in size else tuple(int(v) for v in size.split("x"))
        cases.append((f"sgemm_{size}", pkg.gemm_request(m, n, k, pkg.parse_canonical(g["config"]))))
    for size, g in table.get("gemm_tf32", {}).items():
        m = int(size)
        cases.append((f"tf32_{size}", pkg.gemm_request(m, m, m, pkg.parse_canonical(g["config"]), tf32=True)))
    out = {}
    for name, req in cases:
        row = {}
        for label, be, reps in (("flushed", fl, 10), ("per_event", pe, 30), ("stream", st, 30)):
            req.repetitions = reps if "8192" not in name else max(3, reps // 3)
            r = be.evaluate(req)
            row[label] = (r.time_ms if label == "flushed" else r.mean_ms) * 1e3 if r.ok else r.message[:100]
        row["verified"] = r.verification
        out[name] = row
        print(name, json.dumps(row), flush=True)
    (ROOT / "gpurun_out" / "launch_overhead.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
