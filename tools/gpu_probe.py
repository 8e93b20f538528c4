"""Box probe: host cores, device limits, NVRTC throughput, a short tuning sample."""
import json, os, subprocess, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1703_06503_b200 as pkg

print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
print(subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total", "--format=csv"], capture_output=True, text=True).stdout)
be = pkg.CudaBackend(0)
L = be.limits()
print({f: (getattr(L, f)[:] if hasattr(getattr(L, f), "__len__") and not isinstance(getattr(L, f), bytes) else getattr(L, f)) for f, _ in L._fields_})
t = pkg.Tuner.conv(8192, 4096, 3)
_, _, valid = t.space_counts()
import random
rng = random.Random(0)
idx = sorted(rng.sample(range(valid), 256))
for threads in [len(os.sched_getaffinity(0))]:
    tt = pkg.Tuner.conv(8192, 4096, 3, compile_threads=threads)
    tt.SetVerification(True)
    tt.SetRepetitions(3)
    tt.SetSubset(idx)
    t0 = time.time(); s = tt.Tune(); dt = time.time() - t0
    rows = tt.rows()
    ok = sum(r.status == "ok" and r.verified == "pass" for r in rows)
    print(json.dumps({k: s[k] for k in ("rows", "wall_s", "configs_per_s", "compile_s", "device_s", "best_time_ms", "kernel_launches")}), "ok", ok)
    best = sorted([r for r in rows if r.time_ms], key=lambda r: r.time_ms)[:8]
    for r in best:
        print(f"  {r.time_ms:.4f} ms  {268.435456/r.time_ms:.1f} GB/s  {r.config}")
    bad = [(r.config, r.status, r.message[:200]) for r in rows if not (r.status == "ok" and r.verified == "pass")]
    print("bad", len(bad), bad[:10])
