"""Parity of the B200 path with the oracle (GPU).

* the device reference kernels are BIT-EXACT with the reference's CPU
  oracle (FNV digests vs the golden digests the reference produced);
* every evaluated configuration of both kernel families matches the oracle
  within the stated fp32 tolerance (rel 1e-4, abs 1e-6: the reference
  defaults, tuner.hpp:148-149), checked on the device AND re-checked here on
  the host against the C oracle;
* the device verifier reproduces verify_outputs' report field for field.
"""
import random

import numpy as np
import pytest

import paper_1703_06503_b200 as pkg
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def conv_configs(f, n, seed, device="B200"):
    t = pkg.Tuner.conv(512, 256, f, device=device)
    _, _, valid = t.space_counts()
    rng = random.Random(seed)
    return [pkg.parse_canonical(t.space_config(i)) for i in sorted(rng.sample(range(valid), n))]


def gemm_configs(n, seed, m=256):
    t = pkg.Tuner.gemm(m, m, m, device="B200")
    _, _, valid = t.space_counts()
    rng = random.Random(seed)
    return [pkg.parse_canonical(t.space_config(i)) for i in sorted(rng.sample(range(valid), n))]


# --------------------------------------------------------------- references
@pytest.mark.parametrize("f", [3, 5, 7, 9, 11])
def test_device_conv_reference_bit_exact(backend, golden, f):
    cfg = dict(XWG=32, YWG=8, XWPT=1, YWPT=1, LOCAL=0, VW=1, PAD=0, UNR=1)
    req = pkg.conv_request(8192, 4096, f, cfg)
    _, dig = backend.read_reference(req, 8192 * 4096)
    assert dig == golden["conv_digests"][str(f)]


@pytest.mark.parametrize("m", [512, 1024, 2048])
def test_device_gemm_reference_bit_exact(backend, golden, m):
    cfg = dict(MWG=64, NWG=64, KWG=16, MDIMC=16, NDIMC=16, SA=1, SB=1, MDIMA=16, NDIMB=16,
               STRM=0, STRN=0, VWM=1, VWN=1, KWI=2)
    _, dig = backend.read_reference(pkg.gemm_request(m, m, m, cfg), m * m)
    assert dig == golden["gemm_digests"][str(m)]


def test_device_reference_small_cases(backend, golden):
    for case in golden["small"]:
        if case["kind"] == "conv":
            x, y, f = case["x"], case["y"], case["f"]
            cfg = dict(XWG=8, YWG=8, XWPT=1, YWPT=1, LOCAL=0, VW=1, PAD=0, UNR=0)
            req = pkg.conv_request(x, y, f, cfg, w=case["w"], seed=case["seed"])
            _, dig = backend.read_reference(req, x * y)
        else:
            m, n, k = case["m"], case["n"], case["k"]
            cfg = dict(MWG=16, NWG=16, KWG=16, MDIMC=8, NDIMC=8, SA=0, SB=0, MDIMA=8, NDIMB=8,
                       STRM=0, STRN=0, VWM=1, VWN=1, KWI=2)
            req = pkg.gemm_request(m, n, k, cfg, alpha=case["alpha"], beta=case["beta"],
                                   seed=case["seed"])
            _, dig = backend.read_reference(req, m * n)
        assert dig == case["digest"], case


# ------------------------------------------------------------- conv family
@pytest.mark.parametrize("f", [3, 5, 7, 9, 11])
def test_conv_configs_match_oracle(backend, f):
    x, y = 512, 256
    want = O.conv_reference(x, y, f)
    bad = []
    for cfg in conv_configs(f, 40, seed=f):
        r = backend.evaluate(pkg.conv_request(x, y, f, cfg))
        if not (r.ok and r.verification == "pass"):
            bad.append((cfg, r.status, r.verification, r.message))
            continue
        rep = O.verify(backend.read_output(x * y), want)
        if not rep["pass"]:
            bad.append((cfg, "host", rep))
    assert not bad, bad[:5]


def test_conv_paper_rows_and_edge_tiles(backend):
    """Table II rows plus the extreme tile shapes, incl. ragged images (GUARD)."""
    rows = [
        dict(XWG=32, YWG=8, XWPT=1, YWPT=8, LOCAL=0, VW=1, PAD=0, UNR=1),
        dict(XWG=32, YWG=16, XWPT=2, YWPT=4, LOCAL=2, VW=2, PAD=1, UNR=1),
        dict(XWG=32, YWG=8, XWPT=2, YWPT=8, LOCAL=2, VW=2, PAD=1, UNR=1),
        dict(XWG=64, YWG=8, XWPT=1, YWPT=4, LOCAL=0, VW=1, PAD=0, UNR=1),
        dict(XWG=32, YWG=8, XWPT=2, YWPT=4, LOCAL=1, VW=2, PAD=0, UNR=1),
        dict(XWG=64, YWG=8, XWPT=8, YWPT=8, LOCAL=2, VW=8, PAD=1, UNR=1),    # 512-wide, 4 panels
        dict(XWG=8, YWG=64, XWPT=8, YWPT=8, LOCAL=2, VW=4, PAD=0, UNR=1),    # 512-tall, 3 boxes
        dict(XWG=64, YWG=8, XWPT=8, YWPT=8, LOCAL=1, VW=8, PAD=1, UNR=0),
        dict(XWG=8, YWG=8, XWPT=1, YWPT=1, LOCAL=1, VW=1, PAD=1, UNR=0),
    ]
    for (x, y, f) in [(512, 512, 3), (1024, 512, 11), (520, 300, 7)]:
        want = O.conv_reference(x, y, f)
        for cfg in rows:
            gx = -(-x // cfg["XWPT"])
            gy = -(-y // cfg["YWPT"])
            req = pkg.conv_request(x, y, f, cfg)
            req.global_size = (gx, gy)
            r = backend.evaluate(req)
            assert r.ok and r.verification == "pass", (x, y, f, cfg, r)
            assert O.verify(backend.read_output(x * y), want)["pass"], (x, y, f, cfg)


def test_conv_full_size_best_known(backend):
    for f, cfg in [(3, dict(XWG=32, YWG=8, XWPT=1, YWPT=8, LOCAL=0, VW=1, PAD=0, UNR=1)),
                   (11, dict(XWG=32, YWG=8, XWPT=2, YWPT=8, LOCAL=2, VW=2, PAD=1, UNR=1))]:
        r = backend.evaluate(pkg.conv_request(8192, 4096, f, cfg, reps=3))
        assert r.ok and r.verification == "pass", r
        assert r.report["elements_compared"] == 8192 * 4096
        assert r.report["max_rel_error"] < 1e-4


# ------------------------------------------------------------- gemm family
def test_gemm_configs_match_oracle(backend):
    m = 256
    want = O.gemm_reference(m, m, m)
    bad = []
    for cfg in gemm_configs(60, seed=1, m=m):
        r = backend.evaluate(pkg.gemm_request(m, m, m, cfg))
        if not (r.ok and r.verification == "pass"):
            bad.append((cfg, r.status, r.verification, r.message))
            continue
        if not O.verify(backend.read_output(m * m), want)["pass"]:
            bad.append((cfg, "host"))
    assert not bad, bad[:5]


def test_gemm_paper_rows_beta_and_rectangular(backend):
    rows = [(128, 128, 16, 16, 16, 1, 1, 32, 16, 1, 0, 2, 1, 8),
            (64, 64, 32, 8, 16, 1, 1, 32, 32, 1, 0, 2, 2, 8),
            (128, 128, 32, 16, 16, 1, 1, 32, 32, 0, 1, 4, 4, 2),
            (64, 64, 16, 8, 8, 1, 1, 8, 16, 1, 1, 4, 4, 8),
            (128, 128, 128, 8, 8, 1, 1, 8, 8, 1, 1, 8, 8, 8),
            (32, 32, 32, 32, 32, 0, 1, 32, 32, 0, 1, 1, 1, 2)]
    names = "MWG NWG KWG MDIMC NDIMC SA SB MDIMA NDIMB STRM STRN VWM VWN KWI".split()
    for (m, n, k, a, b) in [(256, 384, 128, 1.0, 0.0), (512, 128, 256, 1.5, 0.5)]:
        want = O.gemm_reference(m, n, k, a, b)
        for row in rows:
            cfg = dict(zip(names, row))
            r = backend.evaluate(pkg.gemm_request(m, n, k, cfg, alpha=a, beta=b))
            assert r.ok and r.verification == "pass", (cfg, r)
            assert O.verify(backend.read_output(m * n), want)["pass"], cfg


def test_gemm_indivisible_problem_is_runtime_error(backend):
    cfg = dict(MWG=128, NWG=128, KWG=16, MDIMC=16, NDIMC=16, SA=1, SB=1, MDIMA=16, NDIMB=16,
               STRM=1, STRN=1, VWM=4, VWN=4, KWI=8)
    req = pkg.gemm_request(256, 256, 256, cfg)
    req.args = pkg.backend.gemm_args(200, 256, 256)
    req.global_size = (200 * 16 // 128, 256 * 16 // 128)
    r = backend.evaluate(req)
    assert r.status == "runtime_error" and "multiple" in r.message


# --------------------------------------------------- device verifier parity
def _cases():
    rng = np.random.default_rng(5)
    ref = rng.random(100_003, dtype=np.float32) * 4 - 2
    c0 = ref.copy()
    c1 = ref * (1 + 5e-5)                          # passes
    c2 = ref.copy(); c2[777] += 1.0                # fails at 777
    c3 = ref.copy(); c3[5] = np.nan                # NaN mid-buffer
    c4 = ref.copy(); c4[-1] = np.nan               # NaN last -> max is NaN
    c5 = ref.copy(); c5[10] = np.nan; c5[99_000] = np.nan; c5[99_001] += 3.0
    z = np.zeros(1000, np.float32)
    z1 = z.copy(); z1[3] = 5e-7                    # abs tolerance near zero: pass
    z2 = z.copy(); z2[3] = 2e-6                    # fail
    inf = ref.copy(); inf[42] = np.inf
    ties = ref.copy(); ties[100] += 1e-5; ties[200] += 1e-5   # argmax tie -> first index
    return [(c0, ref), (c1, ref), (c2, ref), (c3, ref), (c4, ref), (c5, ref), (z1, z), (z2, z),
            (inf, ref), (ties.astype(np.float32), ref), (np.zeros(0, np.float32), np.zeros(0, np.float32))]


def test_device_verifier_matches_host_rule(backend):
    for cand, ref in _cases():
        cand = np.ascontiguousarray(cand, np.float32)
        want = O.verify(cand, ref)
        got = backend.verify_pair(cand, ref)
        for key in ("pass", "buffer_index", "element_index", "elements_compared"):
            assert got[key] == want[key], (key, got, want)
        for key in ("max_abs_error", "max_rel_error"):
            a, b = got[key], want[key]
            assert (np.isnan(a) and np.isnan(b)) or a == b, (key, got, want)


def _screen_cases():
    """Adversarial cases for the verifier's fp32 screen: errors straddling the
    tolerance, records set late, ties, denormal / zero references, and
    tolerances at the edges of float range."""
    rng = np.random.default_rng(11)
    n = 2_000_003
    ref = (rng.random(n, dtype=np.float32) * 2 - 1) * np.float32(3.0)
    ref[::97] = 0.0
    ref[5::101] = np.float32(1e-40)  # denormal references
    out = []
    # relative errors spread across the 1e-4 threshold (some pass, some fail)
    e = rng.uniform(-2e-4, 2e-4, n).astype(np.float32)
    out.append(((ref * (1 + e)).astype(np.float32), ref, 1e-4, 1e-6))
    # exactly at / around the tolerance boundary, all in the same buffer
    c = ref.copy()
    idx = rng.choice(n, 5000, replace=False)
    t = (1e-6 + 1e-4 * np.abs(ref[idx].astype(np.float64)))
    c[idx] = (ref[idx].astype(np.float64) + t * rng.choice([0.999999, 1.0, 1.000001], 5000)).astype(np.float32)
    out.append((c, ref, 1e-4, 1e-6))
    # a monotonically growing error (a new record on every element)
    g = ref + np.linspace(0, 1e-3, n, dtype=np.float32)
    out.append((g.astype(np.float32), ref, 1e-4, 1e-6))
    # many exact ties of the maximum error
    tie = ref.copy()
    tie[rng.choice(n, 1000, replace=False)] += np.float32(0.5)
    out.append((tie, ref, 1e-4, 1e-6))
    # zero tolerances, and tolerances beyond float range
    out.append(((ref * (1 + e)).astype(np.float32), ref, 0.0, 0.0))
    out.append(((ref * (1 + e)).astype(np.float32), ref, 1e40, 1e-6))
    out.append(((ref * (1 + e)).astype(np.float32), ref, 1e-4, 1e40))
    return out


def test_device_verifier_screen_is_exact(backend):
    for cand, ref, rel, abs_ in _screen_cases():
        want = O.verify(cand, ref, rel, abs_)
        got = backend.verify_pair(cand, ref, rel, abs_)
        for key in ("pass", "buffer_index", "element_index", "elements_compared"):
            assert got[key] == want[key], (key, rel, abs_, got, want)
        for key in ("max_abs_error", "max_rel_error"):
            a, b = got[key], want[key]
            assert (np.isnan(a) and np.isnan(b)) or a == b, (key, rel, abs_, got, want)


def test_device_verifier_i32(backend):
    ref = np.arange(5000, dtype=np.int32)
    cand = ref.copy(); cand[1234] += 2
    got = backend.verify_pair(cand, ref)
    want = O.verify(cand, ref)
    assert got == want


# ----------------------------------------------------- tuner end-to-end
def test_tuner_random_search_conv_verified(built):
    t = pkg.Tuner.conv(1024, 512, 5, devices=[0])
    t.UseRandomSearch(1 / 128)
    t.SetVerification(True)
    s = t.Tune()
    rows = t.rows()
    assert s["rows"] == len(rows) == s["budget"] == 5104 // 128
    assert all(r.status == "ok" and r.verified == "pass" for r in rows), \
        [(r.config, r.status, r.message) for r in rows if r.status != "ok" or r.verified != "pass"]
    best, ms = t.GetBestResult()
    assert ms == min(r.time_ms for r in rows)
    assert s["kernel_launches"] > 0


# ------------------------------------------------- TF32 tcgen05 variant
@pytest.mark.parametrize("m,n,k", [(256, 256, 256), (512, 384, 640), (2048, 2048, 2048)])
def test_gemm_tf32_tcgen05_configs(backend, m, n, k):
    """Every TF32 configuration that fits the problem verifies at rel 1e-3
    (the variant's stated tolerance) against the fp32 oracle."""
    want = O.gemm_reference(m, n, k)
    seen = 0
    for cg in (1, 2):  # 2: CTA pair, tcgen05.mma.cta_group::2 (M = 256)
        for bn in (64, 128, 256):
            for bk in (32, 64):
                for st in (2, 3, 4, 6):
                    if m % (128 * cg) or n % bn or k % bk or \
                            st * 4 * bk * (128 + bn // cg) + 2048 > 232448:
                        continue
                    cfg = dict(BN=bn, BK=bk, STAGES=st, CG=cg)
                    r = backend.evaluate(pkg.gemm_request(m, n, k, cfg, tf32=True))
                    assert r.ok and r.verification == "pass", (cfg, r)
                    assert r.report["max_rel_error"] < 1e-3
                    rep = O.verify(backend.read_output(m * n), want, 1e-3, 1e-6)
                    assert rep["pass"], (cfg, rep)
                    seen += 1
    assert seen >= 12


def test_gemm_tf32_epilogues_alpha_beta(backend):
    """Both TF32 epilogues: beta == 0 goes through the TMA-store path (chunks
    staged in the operand ring, bulk tensor stores), beta != 0 through the
    register path that reads Cin -- each against the fp32 oracle (rel 1e-3)."""
    m, n, k = 512, 512, 1024
    for (a, b) in [(1.0, 0.0), (1.5, 0.0), (1.5, 0.5), (-0.5, 2.0)]:
        want = O.gemm_reference(m, n, k, a, b)
        for cfg in (dict(BN=256, BK=32, STAGES=3, CG=2), dict(BN=64, BK=64, STAGES=2, CG=1)):
            r = backend.evaluate(pkg.gemm_request(m, n, k, cfg, alpha=a, beta=b, tf32=True, reps=2))
            assert r.ok and r.verification == "pass", (a, b, cfg, r)
            rep = O.verify(backend.read_output(m * n), want, 1e-3, 1e-6)
            assert rep["pass"], (a, b, cfg, rep)


def test_gemm_tf32_stream_k_matches_oracle(backend):
    """TF32 stream-K (long K, fewer (pair-)tiles than SMs): the persistent
    clusters' partial 128 x BN tiles meet in the workspace (column-major, one
    line per warp access) and the last segment sums them in segment order;
    CTA pairs and single CTAs, alpha/beta, repeated launches -- rel 1e-3
    against the fp32 oracle."""
    for (m, n, k, a, b) in [(1024, 1024, 8192, 1.0, 0.0), (1024, 768, 8192, 1.5, 0.5)]:
        want = O.gemm_reference(m, n, k, a, b)
        for cfg in (dict(BN=256, BK=64, STAGES=3, CG=2), dict(BN=128, BK=32, STAGES=4, CG=2),
                    dict(BN=128, BK=64, STAGES=3, CG=1)):
            if m % (128 * cfg["CG"]) or n % cfg["BN"]:
                continue
            r = backend.evaluate(pkg.gemm_request(m, n, k, cfg, alpha=a, beta=b, tf32=True, reps=3))
            assert r.ok and r.verification == "pass", (m, n, k, cfg, r)
            rep = O.verify(backend.read_output(m * n), want, 1e-3, 1e-6)
            assert rep["pass"], (m, n, k, cfg, rep)


def test_prune_factor_early_out_keeps_winner_and_verification(built):
    """prune_factor (ktc.h): slow configurations are timed once, still verified;
    the winner's time is unaffected (it is never pruned: its first launch is
    within the factor of the best seen)."""
    def run(prune):
        t = pkg.Tuner.gemm(1024, 1024, 1024, devices=[0])
        t.UseRandomSearch(1 / 4096)
        t.SetVerification(True)
        t.SetRepetitions(3)
        if prune:
            t.SetPruning(prune)
        s = t.Tune()
        return t, s

    full, s_full = run(0.0)
    pruned, s_pruned = run(1.5)
    rows_f, rows_p = full.rows(), pruned.rows()
    assert [r.config for r in rows_f] == [r.config for r in rows_p]
    assert all(r.verified == "pass" for r in rows_p if r.status == "ok")
    assert s_pruned["kernel_launches"] < s_full["kernel_launches"]
    _, best_f = full.GetBestResult()
    _, best_p = pruned.GetBestResult()
    assert abs(best_p - best_f) / best_f < 0.05, (best_f, best_p)


def test_sharded_executor_two_workers_on_one_device(built):
    """run_tuning_sharded with two device workers (both on cuda:0 here; one per
    GPU on a multi-GPU box): every unit evaluated once and verified, rows in
    unit order with running bests, best = first minimum (CachedEvaluator's
    strict <, search.hpp:203-208)."""
    t = pkg.Tuner.conv(1024, 512, 5, devices=[0, 0])
    _, _, n = t.space_counts()
    units = list(range(0, n, 41))
    t.SetSubset(units)
    t.SetVerification(True)
    t.Tune()
    rows = t.rows()
    assert [r.space_index for r in rows] == units
    assert [r.step for r in rows] == list(range(1, len(units) + 1))
    assert all(r.status == "ok" and r.verified == "pass" for r in rows)
    times = [r.time_ms for r in rows]
    best_i = min(range(len(times)), key=lambda i: (times[i], i))
    cfg, ms = t.GetBestResult()
    assert cfg == rows[best_i].config and ms == times[best_i]
    run_best = None
    for r in rows:
        run_best = r.time_ms if run_best is None else min(run_best, r.time_ms)
        assert r.best_so_far == run_best


def test_gemm_stream_k_matches_oracle(backend):
    """Stream-K (SK): where whole tiles would land unevenly on the SMs the
    tiles x K-tiles units are dealt to the resident CTAs as contiguous
    ranges; partial tiles meet in a workspace and the last segment sums them
    in segment order.  Shapes with many segments per tile (few tiles, short
    per-CTA ranges), tiles spanning CTA boundaries, alpha/beta, repeated
    launches (counters reset) -- all match the oracle."""
    names = "MWG NWG KWG MDIMC NDIMC SA SB MDIMA NDIMB STRM STRN VWM VWN KWI".split()
    rows = [(64, 64, 32, 16, 16, 1, 1, 16, 16, 0, 1, 4, 4, 8),
            (128, 128, 32, 16, 16, 1, 1, 16, 16, 0, 1, 4, 4, 8),
            (64, 128, 16, 8, 8, 1, 1, 8, 16, 1, 1, 4, 8, 8)]
    # fewer than 2 tiles per SM and K >= 2048 -> stream-K (a CTA's share of
    # K >= 1024, or whole tiles per CTA, both paths covered)
    for (m, n, k, a, b) in [(1024, 512, 8192, 1.0, 0.0), (2048, 1024, 4096, 1.5, 0.5),
                            (512, 256, 2048, 1.0, 0.0)]:
        want = O.gemm_reference(m, n, k, a, b)
        for row in rows:
            cfg = dict(zip(names, row))
            r = backend.evaluate(pkg.gemm_request(m, n, k, cfg, alpha=a, beta=b, reps=3))
            assert r.ok and r.verification == "pass", (m, n, k, cfg, r)
            assert O.verify(backend.read_output(m * n), want)["pass"], (m, n, k, cfg)


def test_gemm_split_k_tail_matches_oracle(backend, monkeypatch):
    """The split-K launch (TAILK): few tiles, long K -> the launch cuts every
    tile's K range across CTAs, reduces the partials in split order and runs
    the alpha/beta epilogue; outputs match the oracle (incl. beta != 0) and
    the counters are reset so repeated launches stay correct.  Covers the
    launch policy (K >= 4096) and forced split counts (KTC_GEMM_SPLIT, read
    at every launch)."""
    names = "MWG NWG KWG MDIMC NDIMC SA SB MDIMA NDIMB STRM STRN VWM VWN KWI".split()
    rows = [(64, 64, 32, 16, 16, 1, 1, 16, 16, 0, 1, 4, 4, 8),
            (128, 64, 16, 16, 8, 1, 1, 16, 8, 1, 1, 4, 2, 8),
            (32, 32, 32, 8, 8, 0, 1, 8, 8, 0, 1, 2, 2, 2)]
    for (m, n, k, a, b, force) in [(512, 512, 2048, 1.0, 0.0, "3"), (256, 384, 4096, 1.5, 0.5, None),
                                   (256, 384, 4096, 1.5, 0.5, "2"), (512, 256, 8192, 1.0, 0.0, None)]:
        if force:
            monkeypatch.setenv("KTC_GEMM_SPLIT", force)
        else:
            monkeypatch.delenv("KTC_GEMM_SPLIT", raising=False)
        want = O.gemm_reference(m, n, k, a, b)
        for row in rows:
            cfg = dict(zip(names, row))
            r = backend.evaluate(pkg.gemm_request(m, n, k, cfg, alpha=a, beta=b, reps=3))
            assert r.ok and r.verification == "pass", (cfg, r)
            assert O.verify(backend.read_output(m * n), want)["pass"], cfg
