"""Repeated-search statistics (`ktune stats`, tools/ktune.cpp:120-258) against
the reference's own stats code (stats.hpp, report.hpp:80-112) on the same
per-configuration times.  The three reports -- best-of-run statistics with
their density grid, the per-run table and the whole-space distribution -- must
be byte-identical, whether the runs execute on one worker or as replicas over
several (annealing / PSO chains do not shard, K of them do)."""
import json
from pathlib import Path

import pytest

import paper_1703_06503_b200 as pkg
from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

B200 = {"name": "B200", "max_work_group_total": 1024, "max_work_group_dim": [1024, 1024, 64],
        "local_mem_bytes": 232448}
CONV = {"template": "conv", "problem": {"filter": 7}, "device": B200}


@pytest.fixture(scope="module")
def table(tmp_path_factory):
    d = tmp_path_factory.mktemp("stats")
    j = dict(CONV, backend={"kind": "synthetic", "model": "conv-like", "failure_rate": 0.07})
    O.ref_job_price_table(json.dumps(j), str(d / "table.csv"))
    return d


def both(d: Path, job: dict, runs: int, seed: int, devices=(0,)):
    text = json.dumps(job)
    O.ref_job_stats(text, str(d), runs, seed, str(d / "ref.csv"))
    t = pkg.Tuner.from_job(text, str(d), devices=list(devices))
    s = t.Stats(runs, seed, str(d / "mine.csv"))
    return s


def same(d: Path, suffix: str) -> bool:
    a, b = d / f"ref{suffix}.csv", d / f"mine{suffix}.csv"
    assert a.exists() == b.exists(), suffix
    return not a.exists() or a.read_bytes() == b.read_bytes()


@pytest.mark.parametrize("strategy", [
    {"kind": "random", "fraction": "1/32"},
    {"kind": "annealing", "fraction": "1/32", "temperature": 4},
    {"kind": "pso", "fraction": "1/32"},
])
@pytest.mark.parametrize("devices", [(0,), (0, 1, 2)])
def test_stats_reports_byte_identical(table, strategy, devices):
    job = dict(CONV, backend={"kind": "replay", "path": "table.csv"}, strategy=strategy)
    s = both(table, job, 24, 5, devices)
    for suffix in ("", "_runs", "_space"):
        assert same(table, suffix), (strategy, suffix)
    assert s["runs"] == 24 and s["space_written"] == 1
    assert s["min"] >= s["space_min"] and s["space_count"] > 4000
    runs = (table / "mine_runs.csv").read_bytes().decode().split("\r\n")
    assert runs[0] == "run,seed,best_time_ms,best_config" and runs[1].startswith("0,5,")
    stats = (table / "mine.csv").read_bytes().decode().split("\r\n")
    assert stats[:2] == ["statistic,value", "count,24"] and stats[6] == "density_x,density_y"
    assert len(stats) == 7 + 256 + 1


def test_stats_degenerate_samples(table):
    # One run: zero deviation and IQR -> the fixed 0.25 bandwidth over
    # [min-1, max+1] (stats.hpp:103-110).
    job = dict(CONV, backend={"kind": "replay", "path": "table.csv"},
               strategy={"kind": "random", "fraction": "1/64"})
    s = both(table, job, 1, 9)
    assert s["stddev"] == 0.0 and s["min"] == s["max"]
    for suffix in ("", "_runs", "_space"):
        assert same(table, suffix), suffix


def test_stats_large_space_skips_space_distribution(tmp_path):
    job = {"template": "gemm", "problem": {"m": 1024, "n": 1024, "k": 1024}, "device": "K40m"}
    O.ref_job_price_table(json.dumps(dict(job, backend={"kind": "synthetic",
                                                        "model": "gemm-like"})),
                          str(tmp_path / "table.csv"))
    job.update(backend={"kind": "replay", "path": "table.csv"},
               strategy={"kind": "annealing", "fraction": "1/16384", "temperature": 4})
    s = both(tmp_path, job, 6, 1, devices=(0, 1))
    assert s["space_written"] == 0
    assert same(tmp_path, "") and same(tmp_path, "_runs") and same(tmp_path, "_space")


def test_stats_run_without_success_is_an_error(tmp_path):
    (tmp_path / "empty.csv").write_text("config,time_ms\n")
    job = dict(CONV, backend={"kind": "replay", "path": "empty.csv"},
               strategy={"kind": "random", "fraction": "1/512"})
    t = pkg.Tuner.from_job(json.dumps(job), str(tmp_path))
    with pytest.raises(Exception, match="no successful configuration"):
        t.Stats(2, 1, str(tmp_path / "s.csv"))
