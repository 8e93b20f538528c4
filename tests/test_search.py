"""Search layer parity with the reference tuner (CPU).

Both tuners run the SAME job (the reference's JSON format) on the SAME
per-configuration times: a replay table priced by the reference's own
synthetic cost model (with injected failures, which replay as `missing`).
The results CSVs must be byte-identical: same enumeration order, same RNG
consumption in random / annealing / PSO, same cache and tie rules, same
running bests and report format.  The sharded executor (several workers,
dynamic chunks) must reproduce the sequential CSV exactly.
"""
import json
from pathlib import Path

import pytest

import paper_1703_06503_b200 as pkg
from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

B200 = {"name": "B200", "max_work_group_total": 1024, "max_work_group_dim": [1024, 1024, 64],
        "local_mem_bytes": 232448}


def price(tmp: Path, job: dict, model: str, failure_rate=0.0, name="table.csv") -> str:
    j = dict(job)
    j["backend"] = {"kind": "synthetic", "model": model, "failure_rate": failure_rate}
    O.ref_job_price_table(json.dumps(j), str(tmp / name))
    return name


def run_both(tmp: Path, job: dict, devices=(0,)):
    text = json.dumps(job)
    ref_csv = tmp / "ref.csv"
    bi, bt = O.ref_job_run(text, str(tmp), str(ref_csv))
    t = pkg.Tuner.from_job(text, str(tmp), devices=list(devices))
    t.Tune()
    mine_csv = tmp / "mine.csv"
    t.write_csv(str(mine_csv))
    return ref_csv.read_bytes(), mine_csv.read_bytes(), (bi, bt), t


CONV = {"template": "conv", "problem": {"filter": 5}, "device": B200}


@pytest.fixture(scope="module")
def conv_table(tmp_path_factory):
    d = tmp_path_factory.mktemp("conv")
    price(d, CONV, "conv-like", failure_rate=0.07)
    return d


@pytest.mark.parametrize("strategy", [
    {"kind": "full"},
    {"kind": "random", "fraction": "1/32"},
    {"kind": "random", "fraction": 0.25},
    {"kind": "annealing", "fraction": "1/64", "temperature": 4},
    {"kind": "annealing", "fraction": "1/16", "temperature": 0.5},
    {"kind": "pso", "fraction": "1/64"},
    {"kind": "pso", "fraction": "1/32", "swarm": 5, "alpha": 0.3, "beta": 0.3, "gamma": 0.3},
])
@pytest.mark.parametrize("seed", [1, 7])
def test_conv_strategies_byte_identical(conv_table, strategy, seed):
    job = dict(CONV, backend={"kind": "replay", "path": "table.csv"}, strategy=strategy, seed=seed)
    ref, mine, (bi, bt), t = run_both(conv_table, job)
    assert mine == ref
    s = t.summary()
    assert s["best_index"] == bi and s["best_time_ms"] == bt


@pytest.mark.parametrize("strategy", [{"kind": "full"}, {"kind": "random", "fraction": "1/8"}])
@pytest.mark.parametrize("devices", [(0, 1), (0, 1, 2, 3), tuple(range(8))])
def test_sharded_executor_reproduces_sequential(conv_table, strategy, devices):
    job = dict(CONV, backend={"kind": "replay", "path": "table.csv"}, strategy=strategy, seed=3)
    ref, mine, (bi, _), t = run_both(conv_table, job, devices=devices)
    assert mine == ref
    assert t.summary()["best_index"] == bi


def test_golden_conv_winner_full_search(tmp_path, golden):
    # conv f=3, B200 limits, reference synthetic conv-like model.
    job = {"template": "conv", "problem": {"filter": 3}, "device": B200}
    price(tmp_path, job, "conv-like")
    job.update(backend={"kind": "replay", "path": "table.csv"}, strategy={"kind": "full"})
    t = pkg.Tuner.from_job(json.dumps(job), str(tmp_path), devices=[0, 1, 2, 3])
    s = t.Tune()
    w = golden["winners"]["conv_f3_B200_conv_like"]
    assert s["rows"] == w["rows"]
    assert s["best_index"] + 1 == w["best_step"]
    assert t.GetBestResult()[0] == w["best_config"]


@pytest.mark.slow
def test_golden_gemm_winner_full_search_852k(tmp_path, golden):
    # 852,608-row full search of the GEMM space at 4096^3, sharded 8 ways.
    job = {"template": "gemm", "problem": {"m": 4096, "n": 4096, "k": 4096}, "device": B200}
    price(tmp_path, job, "gemm-like")
    job.update(backend={"kind": "replay", "path": "table.csv"}, strategy={"kind": "full"})
    t = pkg.Tuner.from_job(json.dumps(job), str(tmp_path), devices=list(range(8)))
    s = t.Tune()
    w = golden["winners"]["gemm_4096_B200_gemm_like"]
    assert s["rows"] == w["rows"] == 852608
    assert s["best_index"] + 1 == w["best_step"]
    cfg, ms = t.GetBestResult()
    assert cfg == w["best_config"] and ms == w["best_time_ms"]


def test_gemm_random_and_annealing_byte_identical(tmp_path):
    job = {"template": "gemm", "problem": {"m": 1024, "n": 1024, "k": 1024}, "device": "K40m",
           "space": {"constraints": ["MWG >= 64", "NWG >= 64", "KWI == 8"]}}
    price(tmp_path, job, "gemm-like", failure_rate=0.05)
    for strategy in ({"kind": "random", "fraction": "1/256"},
                     {"kind": "annealing", "fraction": "1/2048", "temperature": 4},
                     {"kind": "pso", "fraction": "1/2048"}):
        j = dict(job, backend={"kind": "replay", "path": "table.csv"}, strategy=strategy, seed=2)
        ref, mine, _, _ = run_both(tmp_path, j)
        assert mine == ref, strategy


def test_custom_kernel_space_byte_identical(tmp_path):
    job = {
        "kernel": {"name": "copy", "source_ref": "copy.cu", "global": [4096, 64], "local": [1, 1],
                   "modifiers": [{"target": "global", "op": "divide", "factors": ["WPT", "1"]},
                                 {"target": "local", "op": "multiply", "factors": ["TBX", "TBY"]}],
                   "local_mem": "4 * TBX * TBY * (PAD + 1)",
                   "arguments": [{"role": "input", "type": "f32", "length": 4096, "fill": "ramp"},
                                 {"role": "output", "type": "f32", "length": 4096}]},
        "space": {"parameters": {"WPT": [1, 2, 3, 4, 8], "TBX": [8, 16, 32, 64, 128],
                                 "TBY": [1, 2, 4, 8], "PAD": [0, 1, 2]},
                  "constraints": ["TBX * TBY <= 256 || PAD == 0", "!(WPT == 8 && TBY > 2)",
                                  "(WPT + TBX) % 3 != 1 || TBY == 1"]},
        "device": {"name": "tiny", "max_work_group_total": 512,
                   "max_work_group_dim": [256, 4, 1], "local_mem_bytes": 4096},
    }
    price(tmp_path, job, "hash-random", failure_rate=0.1)
    for strategy in ({"kind": "full"}, {"kind": "random", "fraction": "1/3"},
                     {"kind": "annealing", "fraction": "1/4"}, {"kind": "pso", "fraction": "1/4"}):
        j = dict(job, backend={"kind": "replay", "path": "table.csv"}, strategy=strategy)
        ref, mine, _, _ = run_both(tmp_path, j)
        assert mine == ref, strategy


def test_enumeration_order_matches_reference(tmp_path):
    job = {"template": "conv", "problem": {"filter": 9}, "device": "K40m"}
    want = O.ref_job_enumerate(json.dumps(job), tmp_path / "e.txt")
    t = pkg.Tuner.from_job(json.dumps(job), str(tmp_path))
    assert [t.space_config(i) for i in range(len(want))] == want
    job = {"template": "gemm", "device": "HD7970"}
    want = O.ref_job_enumerate(json.dumps(job), tmp_path / "g.txt")
    t = pkg.Tuner.from_job(json.dumps(job), str(tmp_path))
    assert len(want) == t.space_counts()[2] == 639368
    for i in list(range(0, len(want), 9973)) + [len(want) - 1]:
        assert t.space_config(i) == want[i]


def test_space_counts_golden(golden):
    jobs = {
        "conv_f3_B200": {"template": "conv", "problem": {"filter": 3}, "device": B200},
        "conv_f11_K40m": {"template": "conv", "problem": {"filter": 11}, "device": "K40m"},
        "gemm_4096_B200": {"template": "gemm", "problem": {"m": 4096, "n": 4096, "k": 4096},
                           "device": B200},
        "gemm_2048_HD7970": {"template": "gemm", "device": "HD7970"},
    }
    for name, job in jobs.items():
        t = pkg.Tuner.from_job(json.dumps(job), ".")
        assert list(t.space_counts()) == golden["counts"][name], name


def test_checkpoint_resume_reproduces_full_search(conv_table, tmp_path):
    """An interrupted full search resumed from its checkpoint gives the
    same results CSV as an uninterrupted one."""
    job = dict(CONV, backend={"kind": "replay", "path": "table.csv"}, strategy={"kind": "full"})
    text = json.dumps(job)
    ckpt = tmp_path / "ckpt.csv"
    first = pkg.Tuner.from_job(text, str(conv_table))
    _, _, valid = first.space_counts()
    first.SetCheckpoint(str(ckpt))
    first.SetSubset(list(range(valid // 3)))  # "interrupted" after a third
    first.Tune()
    logged = ckpt.read_text().splitlines()
    assert logged[0] == "config,time_ms" and len(logged) > 1
    # Resume against an EMPTY replay table: recorded rows come from the
    # checkpoint, everything else is `missing`.
    (tmp_path / "empty.csv").write_text("config,time_ms\n")
    job2 = dict(job, backend={"kind": "replay", "path": "empty.csv"})
    resumed = pkg.Tuner.from_job(json.dumps(job2), str(tmp_path))
    resumed.SetCheckpoint(str(ckpt))
    resumed.Tune()
    rows = resumed.rows()
    served = [r for r in rows if r.message == "resumed from checkpoint"]
    assert len(served) == len(logged) - 1
    # Resume with the real table: byte-identical to the reference's run.
    again = pkg.Tuner.from_job(text, str(conv_table))
    again.SetCheckpoint(str(ckpt))
    again.Tune()
    again.write_csv(str(tmp_path / "mine.csv"))
    O.ref_job_run(text, str(conv_table), str(tmp_path / "ref.csv"))
    assert (tmp_path / "mine.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()


def test_random_search_above_enumeration_limit_matches_reference(tmp_path):
    """A custom space whose raw size (8 parameters x 8 values = 16.7M) is over
    the enumeration limit: random search samples by rejection, exactly as the
    reference's sample_unique does (space.hpp:443-460) -- same configurations,
    same order (the sharded path used to refuse the space)."""
    params = {f"P{i}": list(range(1, 9)) for i in range(8)}
    job = {
        "kernel": {"name": "copy", "source_ref": "copy.cu", "global": [4096], "local": [1],
                   "arguments": [{"role": "output", "type": "f32", "length": 4096}]},
        "space": {"parameters": params, "constraints": ["P0 + P1 != 3"]},
        "device": {"name": "big", "max_work_group_total": 1024,
                   "max_work_group_dim": [1024, 1024, 64], "local_mem_bytes": 49152},
        "backend": {"kind": "replay", "path": "empty.csv"},
        "strategy": {"kind": "random", "fraction": 1e-5},
    }
    (tmp_path / "empty.csv").write_text("config,time_ms\n")
    ref, mine, _, t = run_both(tmp_path, job, devices=(0, 0))
    assert mine == ref
    assert len(t.rows()) > 100


def test_checkpoint_refuses_a_different_job(conv_table, tmp_path):
    """A checkpoint is bound to the job that wrote it: resuming a
    different problem with the same configuration keys is an error, not a
    silent reuse of the other problem's times."""
    job = dict(CONV, backend={"kind": "replay", "path": "table.csv"}, strategy={"kind": "full"})
    ckpt = tmp_path / "ckpt.csv"
    first = pkg.Tuner.from_job(json.dumps(job), str(conv_table))
    first.SetCheckpoint(str(ckpt))
    first.SetSubset(list(range(50)))
    first.Tune()
    assert (tmp_path / "ckpt.csv.job").exists()
    other = dict(job, problem={"filter": 5, "x": 4096})
    t = pkg.Tuner.from_job(json.dumps(other), str(conv_table))
    t.SetCheckpoint(str(ckpt))
    t.SetSubset(list(range(50)))
    with pytest.raises(Exception, match="different job"):
        t.Tune()
    # the same job resumes fine
    again = pkg.Tuner.from_job(json.dumps(job), str(conv_table))
    again.SetCheckpoint(str(ckpt))
    again.SetSubset(list(range(50)))
    again.Tune()
    assert all(r.message == "resumed from checkpoint" for r in again.rows() if r.status == "ok")


@pytest.mark.parametrize("body", [
    "",                                             # empty file
    "cfg,time\nA=1,2\n",                            # wrong header
    "config,time_ms\r\nLOCAL=0,abc\r\n",            # unparsable time (CRLF)
    "config,time_ms\nLOCAL=0,1e999\n",              # out of range
    "config,time_ms\nLOCAL=0,-2.5\n",               # non-positive
    "config,time_ms\nLOCAL=0,nan\n",                # NaN
    "config,time_ms\nLOCAL=0,1.5\nLOCAL=0,2.5\n",   # duplicate key
    "config,time_ms\n,1.5\n",                       # empty key
    "config,time_ms\nLOCAL=0 1.5\n",                # no comma
])
def test_malformed_replay_tables_fail_like_the_reference(tmp_path, body):
    (tmp_path / "t.csv").write_bytes(body.encode())
    job = dict(CONV, backend={"kind": "replay", "path": "t.csv"},
               strategy={"kind": "random", "fraction": "1/512"})
    text = json.dumps(job)
    with pytest.raises(Exception) as ref_err:
        O.ref_job_run(text, str(tmp_path), str(tmp_path / "r.csv"))
    with pytest.raises(Exception) as mine_err:
        pkg.Tuner.from_job(text, str(tmp_path)).Tune()
    # the reference's job loader prefixes "job file error: " (it loads the
    # table while parsing the job); the diagnostic itself must be the same
    want = str(ref_err.value).strip().removeprefix("job file error: ")
    assert want in str(mine_err.value), (str(ref_err.value), str(mine_err.value))


@pytest.mark.parametrize("values", [[5, 7, 7, 5], [3, -1, 3], [-2, 4, -2], [1, 2, 3, 2, 1], [0, -5]])
def test_parameter_value_errors_match_the_reference(tmp_path, values):
    job = {"kernel": {"name": "k", "source_ref": "k.cu", "global": [64], "local": [1],
                      "arguments": [{"role": "output", "type": "f32", "length": 64}]},
           "space": {"parameters": {"P": values}}, "device": "K40m"}
    text = json.dumps(job)
    with pytest.raises(Exception) as ref_err:
        O.ref_job_counts(text)
    with pytest.raises(Exception) as mine_err:
        pkg.Tuner.from_job(text, str(tmp_path)).space_counts()
    want = str(ref_err.value).strip().removeprefix("job file error: ")
    assert want in str(mine_err.value), (str(ref_err.value), str(mine_err.value))


def test_tf32_space_counts_follow_the_local_memory_expression():
    """The TF32 variant's space (BN x BK x STAGES x CG = 48 points) keeps the
    configurations whose shared memory, STAGES*4*BK*(128 + BN/CG) + 2048
    bytes (a CTA pair stages half of B per CTA), fits the B200's 232,448 B."""
    t = pkg.Tuner.gemm(2048, 2048, 2048, tf32=True)
    want = sum(1 for bn in (64, 128, 256) for bk in (32, 64) for st in (2, 3, 4, 6) for cg in (1, 2)
               if st * 4 * bk * (128 + bn // cg) + 2048 <= 232448)
    assert t.space_counts() == (48, 48, want)
    valid = {t.space_config(i) for i in range(want)}
    assert "BK=32;BN=256;CG=2;STAGES=6" in valid  # 6 x 32 KiB stages per CTA of a pair
    assert "BK=32;BN=256;CG=1;STAGES=6" not in valid


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_full_search_4096_replays_to_the_same_best_index(tmp_path):
    """configs[4]: the measured times of the whole 852,608-configuration
    SGEMM space at 4096^3 (profiles/fullsearch_4096, six GPU ranges of the
    enumeration order) merged with the executor's rule give the same best
    index and time as the reference's own run_full replaying them on its
    ReplayBackend (backend.hpp:485-592)."""
    import numpy as np

    root = Path(__file__).resolve().parent.parent
    times = np.load(root / "profiles" / "fullsearch_4096" / "gemm4096_times.npz")["times"]
    t = pkg.Tuner.gemm(4096, 4096, 4096)
    assert t.space_counts()[2] == len(times) == 852608 and np.isfinite(times).all()
    best = int(np.argmin(times))  # first minimum = earliest index
    with open(tmp_path / "measured.csv", "w") as f:
        f.write("config,time_ms\n")
        for i in range(len(times)):
            f.write(f"{t.space_config(i)},{float(times[i])!r}\n")
    job = {"template": "gemm", "problem": {"m": 4096, "n": 4096, "k": 4096}, "device": B200,
           "strategy": {"kind": "full"}, "verify": False,
           "backend": {"kind": "replay", "path": "measured.csv"}}
    bi, bt = O.ref_job_run(json.dumps(job), str(tmp_path), str(tmp_path / "ref.csv"))
    assert (bi, bt) == (best, float(times[best])) == (442805, float(times[442805]))
