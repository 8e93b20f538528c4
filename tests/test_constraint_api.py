"""Constraint language and CLTune-named API (CPU).

Mirrors the reference's test_constraint.cpp (precedence, short-circuit,
division-by-zero spans, syntax-error offsets, depth limit) through the
public API, and checks the CLTune facade builds the same composed spaces as
the reference's job loader."""
import json
import re

import pytest

import paper_1703_06503_b200 as pkg
from paper_1703_06503_b200 import _ktc as K
from oracle import oracle as O


def count(params: dict, constraints: list[str]) -> int:
    t = pkg.Tuner(device="K40m")
    t.AddKernel("k.cu", "k", [64], [1])
    for name, vals in params.items():
        t.AddParameter(name, vals)
    for c in constraints:
        t.AddConstraint(c)
    return t.space_counts()[1]


def brute(params: dict, pred) -> int:
    import itertools

    names = list(params)
    return sum(1 for vals in itertools.product(*params.values()) if pred(dict(zip(names, vals))))


@pytest.mark.parametrize("expr,fn", [
    ("A + B * C == 14", lambda v: v["A"] + v["B"] * v["C"] == 14),
    ("(A + B) * C >= 20", lambda v: (v["A"] + v["B"]) * v["C"] >= 20),
    ("A - B - C > 0", lambda v: v["A"] - v["B"] - v["C"] > 0),
    ("A * B % 4 == 2", lambda v: (v["A"] * v["B"]) % 4 == 2),
    ("C / 2 * 2 == C", lambda v: (v["C"] // 2) * 2 == v["C"]),
    ("A < B || A > C && B != 0", lambda v: v["A"] < v["B"] or (v["A"] > v["C"] and v["B"] != 0)),
    ("!(A == B) && !!C", lambda v: v["A"] != v["B"] and v["C"] != 0),
    ("(A >= 1) * 4 + (B < 2) == 4", lambda v: (v["A"] >= 1) * 4 + (v["B"] < 2) == 4),
    ("B != 0 && A % B == 0", lambda v: v["B"] != 0 and v["A"] % v["B"] == 0),
    ("B == 0 || C / B >= 1", lambda v: v["B"] == 0 or v["C"] // v["B"] >= 1),
])
def test_constraint_semantics_match_brute_force(built, expr, fn):
    params = {"A": [0, 1, 2, 3, 4, 5, 6], "B": [0, 1, 2, 3], "C": [0, 1, 2, 4, 5, 8]}
    assert count(params, [expr]) == brute(params, fn)


def _err(expr: str) -> str:
    t = pkg.Tuner(device="K40m")
    t.AddKernel("k.cu", "k", [64], [1])
    t.AddParameter("Xwg", [1, 2])
    t.AddParameter("Ywg", [1, 2])
    with pytest.raises(K.KtcError) as e:
        t.AddConstraint(expr)
    return str(e.value)


@pytest.mark.parametrize("expr,offset", [
    ("Xwg &* 2", 4), ("", 0), (")", 0), ("(1", 2), ("1 +", 3), ("-1", 0), ("1 < 2 < 3", 6),
    ("Xwg = 1", 4), ("Xwg | 2", 4), ("2 # 2", 2), ("99999999999999999999999", 0),
])
def test_syntax_error_offsets(built, expr, offset):
    msg = _err(expr)
    m = re.search(r"syntax error at offset (\d+)", msg)
    assert m and int(m.group(1)) == offset, msg


def test_unknown_identifier_and_depth_limit(built):
    assert 'unknown parameter: "Zwg"' in _err("Xwg + Zwg")
    assert "nested too deeply" in _err("(" * 1000 + "1" + ")" * 1000)


def test_division_by_zero_reports_subexpression(built):
    t = pkg.Tuner(device="K40m")
    t.AddKernel("k.cu", "k", [64], [1])
    t.AddParameter("A", [12])
    t.AddParameter("B", [0])
    t.AddConstraint("A % B == 0")
    with pytest.raises(K.KtcError) as e:
        t.space_counts()
    assert 'division by zero in subexpression "A % B"' in str(e.value)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_cltune_facade_matches_reference_job(built):
    """Tuner.AddKernel/AddParameter/MulLocalSize/DivGlobalSize/... builds the
    same composed space (counts and enumeration) as the reference's job
    loader on the equivalent JSON job."""
    t = pkg.Tuner(device="HD7970")
    t.AddKernel("copy.cu", "copy", [4096, 64], [1, 1])
    t.AddParameter("WPT", [1, 2, 3, 4, 8])
    t.AddParameter("TBX", [8, 16, 32, 64, 128, 256, 512])
    t.AddParameter("TBY", [1, 2, 4])
    t.DivGlobalSize(["WPT", "1"])
    t.MulLocalSize(["TBX", "TBY"])
    t.SetLocalMemoryUsage("4 * TBX * TBY * WPT")
    t.AddConstraint("TBX * TBY <= 512")
    job = {"kernel": {"name": "copy", "source_ref": "copy.cu", "global": [4096, 64],
                      "local": [1, 1],
                      "modifiers": [{"target": "global", "op": "divide", "factors": ["WPT", "1"]},
                                    {"target": "local", "op": "multiply",
                                     "factors": ["TBX", "TBY"]}],
                      "local_mem": "4 * TBX * TBY * WPT"},
           "space": {"parameters": {"WPT": [1, 2, 3, 4, 8], "TBX": [8, 16, 32, 64, 128, 256, 512],
                                    "TBY": [1, 2, 4]},
                     "constraints": ["TBX * TBY <= 512"]},
           "device": "HD7970"}
    assert t.space_counts() == O.ref_job_counts(json.dumps(job))
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        want = O.ref_job_enumerate(json.dumps(job), f"{d}/e.txt")
    assert [t.space_config(i) for i in range(len(want))] == want


def test_device_presets(built):
    dm = K.DeviceModel()
    import ctypes as C

    K.check(pkg.lib().ktc_device_preset(b"B200", C.byref(dm)))
    assert dm.local_mem_bytes == 232448 and dm.max_work_group_total == 1024
    assert abs(dm.peak_gflops - 148 * 128 * 2 * 1.965) < 1e-6
    with pytest.raises(K.KtcError):
        K.check(pkg.lib().ktc_device_preset(b"GTX9000", C.byref(dm)))


def test_cltune_reporting_names(built, tmp_path, capsys):
    """PrintToScreen / PrintToFile / SetNumRuns on a replayed search (no GPU)."""
    table = tmp_path / "t.csv"
    rows = ["config,time_ms"] + [f"WPT={w},1.{w}" for w in (1, 2, 4)]
    table.write_text("\n".join(rows) + "\n")
    t = pkg.Tuner(device=None, backend=f"replay:{table}")
    t.SetDevice({"name": "tiny", "max_work_group_total": 256, "local_mem_bytes": 4096})
    t.AddKernel("k.cu", "k", [64], [1])
    t.AddParameter("WPT", [1, 2, 4])
    t.DivGlobalSize(["WPT"])
    t.AddArgumentOutput(64)
    t.SetNumRuns(3)
    t.UseFullSearch()
    t.Tune()
    t.PrintToScreen()
    out = capsys.readouterr().out
    assert "WPT=1" in out and "[ best ]" in out and "1.1000 ms" in out
    t.PrintToFile(str(tmp_path / "r.csv"))
    assert (tmp_path / "r.csv").read_text().count("\n") >= 4
