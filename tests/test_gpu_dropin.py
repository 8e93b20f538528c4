"""Drop-in proof (GPU): the reference's OWN tuner (run_tuning, jobfile,
write_results_csv -- compiled unmodified from /root/reference into
oracle/_ref/ref_tune_cuda) evaluates on the B200 through
include/ktune_cuda_backend.hpp -> libktc's C ABI.  Every row must be `ok`
and verified `pass` by the reference tuner's own verification rule, and the
configurations it visits must be exactly the ones this framework's tuner
visits for the same job and seed."""
import json
import subprocess
from pathlib import Path

import pytest

import paper_1703_06503_b200 as pkg
from oracle import oracle as O

pytestmark = pytest.mark.gpu

BIN = Path(O.__file__).resolve().parent / "_ref" / "ref_tune_cuda"
B200 = {"name": "B200", "max_work_group_total": 1024, "max_work_group_dim": [1024, 1024, 64],
        "local_mem_bytes": 232448}


def run_ref(tmp, job, mode=None):
    (tmp / "job.json").write_text(json.dumps(job))
    cmd = [str(BIN), str(tmp / "job.json"), str(tmp / "ref.csv")] + ([mode] if mode else [])
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr
    lines = (tmp / "ref.csv").read_bytes().decode().split("\r\n")[1:-1]
    return [ln.split(",") for ln in lines], p.stdout


@pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/ref_tune_cuda not built")
def test_reference_tuner_on_b200_device_verdict(built, tmp_path):
    job = {"template": "conv", "problem": {"x": 2048, "y": 1024, "filter": 7}, "device": B200,
           "strategy": {"kind": "random", "fraction": "1/64"}, "seed": 5, "verify": True,
           "repetitions": 2}
    rows, out = run_ref(tmp_path, job)
    assert len(rows) == 5104 // 64
    assert all(r[2] == "ok" and r[7] == "pass" for r in rows), [r for r in rows if r[7] != "pass"][:3]
    mine = pkg.Tuner.from_job(json.dumps(dict(job, backend={"kind": "cuda"})), str(tmp_path))
    mine.Tune()
    assert [r.config for r in mine.rows()] == [r[1] for r in rows]


@pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/ref_tune_cuda not built")
def test_reference_tuner_on_b200_host_verification(built, tmp_path):
    job = {"template": "gemm", "problem": {"m": 256, "n": 256, "k": 256}, "device": B200,
           "strategy": {"kind": "annealing", "fraction": "1/32768"}, "seed": 3, "verify": True}
    rows, _ = run_ref(tmp_path, job, "host")
    assert len(rows) == 852608 // 32768
    assert all(r[2] == "ok" and r[7] == "pass" for r in rows), rows[:3]


RUNNER = Path(pkg.__file__).resolve().parent / "ktune-cuda-runner"


@pytest.mark.skipif(not O.ref_available() or not RUNNER.exists(), reason="runner / oracle not built")
def test_reference_external_backend_drives_b200_runner(built, tmp_path):
    """Zero-change integration: the reference's own ExternalBackend
    (external.hpp) spawns ktune-cuda-runner per evaluation; every row comes
    back ok and verified through the protocol's output digests."""
    job = {"template": "conv", "problem": {"x": 512, "y": 256, "filter": 5}, "device": B200,
           "strategy": {"kind": "random", "fraction": "1/512"}, "seed": 3, "verify": True,
           "backend": {"kind": "external", "argv": [str(RUNNER)], "timeout_ms": 120000}}
    import os

    os.environ["KTC_CACHE_DIR"] = str(tmp_path / "cubins")
    bi, bt = O.ref_job_run(json.dumps(job), str(tmp_path), str(tmp_path / "ref.csv"))
    rows = [ln.split(",") for ln in (tmp_path / "ref.csv").read_bytes().decode().split("\r\n")[1:-1]]
    assert len(rows) == 5104 // 512
    assert all(r[2] == "ok" and r[7] == "pass" for r in rows), rows
    assert bi >= 0 and bt > 0


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_measured_times_replay_through_reference_full_search(built, tmp_path):
    """a full search measured on the B200 is saved as a replay
    table and re-run through the reference's own run_full on its
    ReplayBackend (backend.hpp:485-592): same best index, same best time."""
    job = {"template": "conv", "problem": {"x": 1024, "y": 512, "filter": 5}, "device": B200,
           "strategy": {"kind": "full"}, "verify": True, "repetitions": 2}
    t = pkg.Tuner.from_job(json.dumps(dict(job, backend={"kind": "cuda"})), str(tmp_path))
    s = t.Tune()
    assert s["rows"] == 5104
    t.write_replay(str(tmp_path / "measured.csv"))
    rjob = dict(job, verify=False, backend={"kind": "replay", "path": "measured.csv"})
    bi, bt = O.ref_job_run(json.dumps(rjob), str(tmp_path), str(tmp_path / "ref.csv"))
    assert bi == s["best_index"] and bt == s["best_time_ms"]
