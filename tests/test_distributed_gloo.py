"""Multi-process sharding (CPU, gloo, world_size 2): two ranks tune disjoint
chunks of a full search on replayed per-configuration times, rank 0 merges
the gathered rows; the merged outcome must equal the reference tuner's
sequential full search on the same table (rows, best index, best time)."""
import json
import os
import socket
from pathlib import Path

import pytest
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

JOB = {"template": "conv", "problem": {"filter": 7},
       "device": {"name": "B200", "max_work_group_total": 1024,
                  "max_work_group_dim": [1024, 1024, 64], "local_mem_bytes": 232448}}


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, tmp, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1703_06503_b200 as pkg
    from paper_1703_06503_b200 import distributed as D

    job = dict(JOB, backend={"kind": "replay", "path": "table.csv"})
    t = pkg.Tuner.from_job(json.dumps(job), tmp)
    _, _, valid = t.space_counts()
    rows = D.tune_shard(t, list(range(valid)), rank, world, chunk=37)
    merged = D.gather_merge(rows, world)
    if rank == 0:
        Path(out_path).write_text(json.dumps({
            "rows": [[r[1], r[2], r[3]] for r in merged.rows],
            "best_index": merged.best_index, "best_time_ms": merged.best_time_ms}))
    dist.destroy_process_group()


def test_two_ranks_reproduce_reference_full_search(tmp_path):
    j = dict(JOB, backend={"kind": "synthetic", "model": "conv-like", "failure_rate": 0.05})
    O.ref_job_price_table(json.dumps(j), str(tmp_path / "table.csv"))
    ref_job = dict(JOB, backend={"kind": "replay", "path": "table.csv"}, strategy={"kind": "full"})
    bi, bt = O.ref_job_run(json.dumps(ref_job), str(tmp_path), str(tmp_path / "ref.csv"))
    ref_rows = [ln.split(",") for ln in
                (tmp_path / "ref.csv").read_bytes().decode().split("\r\n")[1:-1]]

    out = tmp_path / "merged.json"
    mp.spawn(_rank, args=(2, free_port(), str(tmp_path), str(out)), nprocs=2, join=True)
    got = json.loads(out.read_text())
    assert got["best_index"] == bi and got["best_time_ms"] == bt
    assert len(got["rows"]) == len(ref_rows)
    for (cfg, status, t), ref in zip(got["rows"], ref_rows):
        assert cfg == ref[1] and status == ref[2]
        assert (t is None and ref[3] == "") or float(ref[3]) == t


def _stats_rank(rank, world, port, tmp):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1703_06503_b200 as pkg
    from paper_1703_06503_b200 import distributed as D

    job = dict(JOB, backend={"kind": "replay", "path": "table.csv"},
               strategy={"kind": "annealing", "fraction": "1/64", "temperature": 4})
    t = pkg.Tuner.from_job(json.dumps(job), tmp)
    runs = D.gather_runs(D.stats_replicas(t, 10, 5, rank, world), world)
    # Whole-space distribution: one full sweep sharded over the ranks.
    t.UseFullSearch()
    _, _, valid = t.space_counts()
    merged = D.gather_merge(D.tune_shard(t, list(range(valid)), rank, world, chunk=53), world)
    if rank == 0:
        times = [r[3] for r in merged.rows if r[2] == "ok" and r[4] != "fail" and r[3] is not None]
        D.write_stats_reports(runs, str(Path(tmp) / "mine.csv"), times)
    dist.destroy_process_group()


def test_two_ranks_stats_replicas_match_reference(tmp_path):
    """SA replicas dealt over two processes (one per GPU in production);
    rank 0's reports equal the reference's `ktune stats` byte for byte."""
    j = dict(JOB, backend={"kind": "synthetic", "model": "conv-like", "failure_rate": 0.05})
    O.ref_job_price_table(json.dumps(j), str(tmp_path / "table.csv"))
    ref_job = dict(JOB, backend={"kind": "replay", "path": "table.csv"},
                   strategy={"kind": "annealing", "fraction": "1/64", "temperature": 4})
    O.ref_job_stats(json.dumps(ref_job), str(tmp_path), 10, 5, str(tmp_path / "ref.csv"))
    mp.spawn(_stats_rank, args=(2, free_port(), str(tmp_path)), nprocs=2, join=True)
    for suffix in ("", "_runs", "_space"):
        assert (tmp_path / f"mine{suffix}.csv").read_bytes() == \
            (tmp_path / f"ref{suffix}.csv").read_bytes(), suffix
