"""`ktune-b200`: the reference's command line (proj/tools/ktune.cpp -- tune,
stats, enumerate) over libktc.  On replay jobs its report files must be
byte-identical to the reference tuner's (run through oracle/_ref), reruns
must reproduce them byte for byte (the reference's acceptance criterion 12,
acceptance.cpp:710-767), and the exit codes follow ktune.cpp:284-298
(1 error, 2 empty space)."""
import json
import subprocess
from pathlib import Path

import pytest

import paper_1703_06503_b200 as pkg
from oracle import oracle as O

CLI = Path(pkg.__file__).resolve().parent / "ktune-b200"
pytestmark = pytest.mark.skipif(not CLI.exists() or not O.ref_available(),
                                reason="ktune-b200 / oracle/_ref not built")

B200 = {"name": "B200", "max_work_group_total": 1024, "max_work_group_dim": [1024, 1024, 64],
        "local_mem_bytes": 232448}


def cli(*args, cwd):
    return subprocess.run([str(CLI), *map(str, args)], cwd=cwd, capture_output=True, text=True,
                          timeout=600)


@pytest.fixture(scope="module")
def wd(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli")
    job = {"template": "conv", "problem": {"filter": 5}, "device": B200}
    O.ref_job_price_table(json.dumps(dict(job, backend={"kind": "synthetic", "model": "conv-like",
                                                        "failure_rate": 0.05})),
                          str(d / "table.csv"))
    return d


def write_job(d: Path, name: str, strategy: dict, **extra) -> dict:
    job = {"template": "conv", "problem": {"filter": 5}, "device": B200,
           "backend": {"kind": "replay", "path": "table.csv"}, "strategy": strategy, **extra}
    (d / name).write_text(json.dumps(job))
    return job


@pytest.mark.parametrize("strategy,gpus", [({"kind": "full"}, 4),
                                           ({"kind": "random", "fraction": "1/16"}, 2),
                                           ({"kind": "annealing", "fraction": "1/32"}, 1),
                                           ({"kind": "pso", "fraction": "1/32"}, 1)])
def test_tune_matches_reference_tuner(wd, strategy, gpus):
    job = write_job(wd, "tune.json", strategy, seed=1)
    p = cli("tune", "tune.json", "--seed", 7, "--out", "mine.csv", "--gpus", gpus, cwd=wd)
    assert p.returncode == 0, p.stderr
    bi, bt = O.ref_job_run(json.dumps(dict(job, seed=7)), str(wd), str(wd / "ref.csv"))
    assert (wd / "mine.csv").read_bytes() == (wd / "ref.csv").read_bytes()
    lines = p.stdout.splitlines()
    assert lines[0] == "kernel: conv on B200 via replay"
    assert lines[1] == "space: 5104 valid configurations"
    assert f"(step {bi + 1}," in lines[4] and lines[-1] == "wrote mine.csv"


def test_tune_uses_the_jobs_output_field(wd):
    write_job(wd, "out.json", {"kind": "random", "fraction": "1/64"}, output="from_job.csv")
    p = cli("tune", "out.json", cwd=wd)
    assert p.returncode == 0 and (wd / "from_job.csv").exists(), p.stderr


def test_stats_matches_reference_and_reruns_identically(wd):
    job = write_job(wd, "stats.json", {"kind": "annealing", "fraction": "1/64", "temperature": 4})
    O.ref_job_stats(json.dumps(job), str(wd), 10, 5, str(wd / "ref.csv"))
    for rnd, extra in enumerate((["--parallel", 3], ["--gpus", 2], [])):
        p = cli("stats", "stats.json", "--runs", 10, "--base-seed", 5, "--out", f"s{rnd}.csv",
                *extra, cwd=wd)
        assert p.returncode == 0, p.stderr
        assert p.stdout.splitlines()[0] == "runs: 10 (seeds 5..14)"
        for suffix in ("", "_runs", "_space"):
            assert (wd / f"s{rnd}{suffix}.csv").read_bytes() == \
                (wd / f"ref{suffix}.csv").read_bytes(), (rnd, suffix)


def test_enumerate_counts_and_list(wd):
    write_job(wd, "enum.json", {"kind": "full"})
    p = cli("enumerate", "enum.json", cwd=wd)
    assert p.returncode == 0
    assert p.stdout.splitlines() == ["raw: 12288", "constrained: 6400", "device-rejected: 1296",
                                     "valid: 5104"]
    p = cli("enumerate", "enum.json", "--list", cwd=wd)
    listed = p.stdout.splitlines()[4:]
    job = json.loads((wd / "enum.json").read_text())
    del job["backend"]
    want = O.ref_job_enumerate(json.dumps(job), wd / "e.txt")
    assert listed == want


def test_exit_codes(wd):
    write_job(wd, "empty.json", {"kind": "full"}, space={"constraints": ["XWG > 1000"]})
    assert cli("enumerate", "empty.json", cwd=wd).returncode == 2
    assert cli("tune", "empty.json", cwd=wd).returncode == 2
    (wd / "bad.json").write_text(json.dumps({"template": "conv", "backend": {"kind": "opencl"}}))
    p = cli("tune", "bad.json", cwd=wd)
    assert p.returncode == 1 and "error" in p.stderr
    assert cli("stats", "stats.json", cwd=wd).returncode == 1  # --runs missing
    assert cli("frobnicate", "x.json", cwd=wd).returncode == 1
    assert cli("tune", "missing.json", cwd=wd).returncode == 1


@pytest.mark.gpu
def test_cli_cuda_backend_tune_and_stats(tmp_path):
    """The reference's job format with backend kind "cuda" on the B200:
    every row ok and verified; stats replicas run whole searches."""
    job = {"template": "conv", "problem": {"x": 1024, "y": 512, "filter": 3}, "device": B200,
           "backend": {"kind": "cuda"}, "strategy": {"kind": "random", "fraction": "1/128"},
           "verify": True, "repetitions": 2}
    (tmp_path / "job.json").write_text(json.dumps(job))
    p = cli("tune", "job.json", "--out", "r.csv", "--gpus", 1, cwd=tmp_path)
    assert p.returncode == 0, p.stderr
    rows = [ln.split(",") for ln in (tmp_path / "r.csv").read_bytes().decode().split("\r\n")[1:-1]]
    assert len(rows) == 5104 // 128
    assert all(r[2] == "ok" and r[7] == "pass" for r in rows), rows[:3]
    assert "cuda" in p.stdout.splitlines()[0]
    job["strategy"] = {"kind": "annealing", "fraction": "1/256"}
    (tmp_path / "sa.json").write_text(json.dumps(job))
    # Two replicas sharing the one GPU of the test box (one per device in
    # production: --gpus N).
    p = cli("stats", "sa.json", "--runs", 3, "--out", "s.csv", "--devices", "0,0", cwd=tmp_path)
    assert p.returncode == 0, p.stderr
    runs = (tmp_path / "s_runs.csv").read_bytes().decode().split("\r\n")[1:-1]
    assert len(runs) == 3 and (tmp_path / "s_space.csv").exists()


@pytest.mark.gpu
def test_cli_exits_cleanly_with_speculative_compiles_queued(tmp_path):
    """Annealing prefetches every neighbour of the current GEMM configuration
    into the compile pool; at exit the queued compiles are dropped and the
    running ones drained before static destructors (was: free() abort)."""
    job = {"template": "gemm", "problem": {"m": 1024, "n": 1024, "k": 1024}, "device": B200,
           "backend": {"kind": "cuda"}, "verify": True,
           "strategy": {"kind": "annealing", "fraction": "1/8192", "temperature": 4}}
    (tmp_path / "sa.json").write_text(json.dumps(job))
    p = cli("stats", "sa.json", "--runs", 2, "--out", "s.csv", cwd=tmp_path)
    assert p.returncode == 0, p.stderr[-2000:]
    assert len((tmp_path / "s_runs.csv").read_bytes().decode().split("\r\n")) == 4


@pytest.mark.gpu
def test_cli_exits_cleanly_tf32_annealing(tmp_path):
    """Same exit path for an NVRTC family (TF32): pool workers still inside
    NVRTC at exit read the leaked option vector, never a destroyed static
    (base_options() was destroyed before the quiesce handler ran)."""
    job = {"template": "gemm_tf32", "problem": {"m": 1024, "n": 1024, "k": 1024}, "device": B200,
           "backend": {"kind": "cuda"}, "verify": True,
           "strategy": {"kind": "annealing", "fraction": "1/4", "temperature": 4}}
    (tmp_path / "sa.json").write_text(json.dumps(job))
    for _ in range(3):
        p = cli("stats", "sa.json", "--runs", 2, "--out", "s.csv", cwd=tmp_path)
        assert p.returncode == 0, p.stderr[-2000:]
        assert len((tmp_path / "s_runs.csv").read_bytes().decode().split("\r\n")) == 4
