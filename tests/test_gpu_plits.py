"""PLITS on the GPU (paper_2103_10453_b200/csrc/plits.cu) vs the C oracle's canonical
rule (or_plits, OR_TIE_CANON), bit-exact, through the C ABI.

The oracle's REF policy is pinned to the reference's plits_run and its CANON
policy to its own specification (tests/test_oracle_plits.py), so equality here
pins the kernel: final colourings, f, iteration counts (both phases), the
per-step trace (move, delta, N, tenure, active-set size, f, c, best 2F) and the
algorithmic byte counter; then the MPMA run() end to end.
"""
import re

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CASES = [(5, 0.5, 61), (10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (60, 0.5, 12345), (70, 0.6, 12345)]


def _offspring(orc, grid, g, p, seed):
    off = orc.init_population(grid, p, seed)
    rng = np.random.default_rng(seed)
    for i in range(1, p, 4):  # some partial (uncoloured) inputs, some legal ones
        off[i][rng.random(g.vertex_count) < 0.3] = 0
    for i in range(2, p, 4):
        off[i] = orc.repair(grid, off[i])
    return off


@pytest.mark.parametrize("n,r,s", CASES)
@pytest.mark.parametrize("b1,b2", [(1, 1), (37, 5), (600, 0), (0, 0)])
def test_plits_improve_matches_oracle(plse, orc, n, r, s, b1, b2):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p = 16
    cfg = plse.SolverConfig(p=p, master_seed=5, phase1_iters=b1, phase2_iters=b2, variant=plse.MPMA)
    dp = plse.DevicePopulation(g, cfg)
    off = _offspring(orc, grid, g, p, 5)
    dp.offspring = off
    gen = 2
    it, bf, bi = dp.improve(gen)
    imp = dp.improved
    f, c, iters = dp.stats(plse.IMPROVED)
    stop_f = 1 if g.l == 1 else 0
    tot, want_bytes = 0, 0.0
    for i in range(p):
        o = orc.plits(grid, off[i], orc.derive_seed(5, 2, gen * p + i), b1, b2, 0.6, stop_f, tie=oracle.TIE_CANON)
        assert iters[i] == o["iterations"], (i, iters[i], o["iterations"])
        assert np.array_equal(imp[i], o["best"]), i
        assert f[i] == o["final_f"] and c[i] == 0
        tot += o["iterations"]
        want_bytes += o["alg_bytes"]
    assert it == tot
    assert bf == min(f) and bi == int(np.argmin(f))
    assert dp.counters().alg_bytes == want_bytes


@pytest.mark.parametrize("n,r,s", [(10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (70, 0.6, 12345)])
def test_plits_per_step_trace_matches_oracle(plse, orc, n, r, s):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p = 3
    b1, b2 = 3000, 200
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=13, phase1_iters=b1, phase2_iters=b2,
                                                    variant=plse.MPMA))
    off = _offspring(orc, grid, g, p, 13)
    dp.offspring = off
    stop_f = 1 if g.l == 1 else 0
    for idx in range(p):
        steps, n_it = dp.trace(idx, 4, b1 + b2)
        o = orc.plits(grid, off[idx], orc.derive_seed(13, 2, 4 * p + idx), b1, b2, 0.6, stop_f,
                      tie=oracle.TIE_CANON, trace_cap=b1 + b2)
        assert n_it == o["iterations"]
        for a, e in zip(steps, o["trace"]):
            want = dict(step=e["step"], v=e["v"], k=e["k"] if e["v"] >= 0 else 0, e=e["phase"],
                        ev0=e["from_"] if e["v"] >= 0 else 0, ev1=e["active"], f_before=e["f"], f_after=e["c"],
                        best_f=e["best_scaled"], tenure=e["tenure"], n_adm=e["n_adm"] if e["v"] >= 0 else 0,
                        level=e["delta"] if e["v"] >= 0 else 0)
            assert a == want, (idx, a, want)


@pytest.mark.parametrize("alpha", [0.0, 0.3, 1.5])
def test_plits_alpha_and_l1(plse, orc, alpha):
    """alpha changes every tenure; an instance with l == 1 stops at f <= 1 (engine.hpp:134)."""
    for n, r, s in [(20, 0.6, 9), (12, 0.45, 4)]:
        grid = orc.generate_instance(n, r, s)
        g = plse.preprocess(grid)
        p = 12
        dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=8, alpha=alpha, phase1_iters=900,
                                                        variant=plse.MPMA))
        off = _offspring(orc, grid, g, p, 8)
        dp.offspring = off
        dp.improve(1)
        imp = dp.improved
        for i in range(p):
            o = orc.plits(grid, off[i], orc.derive_seed(8, 2, p + i), 900, 0, alpha, 1 if g.l == 1 else 0,
                          tie=oracle.TIE_CANON)
            assert np.array_equal(imp[i], o["best"]), (n, i)


@pytest.mark.parametrize("n,r,s,p", [(10, 0.5, 3, 8), (20, 0.6, 9, 12), (30, 0.5, 4, 16), (60, 0.5, 12345, 24)])
def test_mpma_run_matches_oracle(plse, orc, n, r, s, p):
    grid = orc.generate_instance(n, r, s)
    res = plse.run(grid, plse.SolverConfig(p=p, master_seed=s, generation_limit=3, phase1_iters=500,
                                           variant=plse.MPMA))
    o = orc.run(grid, p=p, seed=s, generation_limit=3, phase1_iters=500, tie=oracle.TIE_CANON, variant=0)
    for k in ("best_f", "best_score", "stop_reason", "generations", "total_iterations", "l", "upper_bound"):
        assert getattr(res, k) == o[k], k
    assert np.array_equal(res.best_solution, o["best_colors"])


def test_mpma_cli_json_reports_variant(plse, orc, tmp_path):
    import json
    import subprocess
    import sys
    import os
    grid = orc.generate_instance(12, 0.6, 88)
    inst = tmp_path / "i.txt"
    inst.write_text(plse.serialize_instance(grid))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "paper_2103_10453_b200", "solve", str(inst), "--seed", "31337",
                        "--pop", "16", "--gen-limit", "5", "--workers", "2"], capture_output=True, text=True,
                       cwd=root, timeout=600)
    assert r.returncode in (0, 2), r.stderr
    j = json.loads(r.stdout)
    assert j["config"]["variant"] == "mpma"
    o = orc.run(grid, p=16, seed=31337, generation_limit=5, tie=oracle.TIE_CANON, variant=0)
    assert (j["f"], j["total_iterations"], j["generations"]) == (o["best_f"], o["total_iterations"],
                                                                 o["generations"])


@pytest.mark.parametrize("cap", [32, 8])
def test_plits_register_mode_transitions(plse, orc, capfd, monkeypatch, cap):
    """The register-resident active list (|active| <= 32) is entered and left inside searches and the
    results stay equal to the oracle's.  PLSE_PROFILE=1 runs the instrumented kernel, which counts the
    transitions; PLSE_PLITS_CAP shrinks its list capacity so that the searches leave the mode too (with 32
    lanes the active set rarely outgrows the list once it has shrunk into it)."""
    monkeypatch.setenv("PLSE_PROFILE", "1")
    monkeypatch.setenv("PLSE_PLITS_CAP", str(cap))
    entries = exits = 0
    for n, r, s in [(30, 0.5, 12345), (60, 0.5, 12345), (70, 0.6, 12345)]:
        grid = orc.generate_instance(n, r, s)
        g = plse.preprocess(grid)
        p, b1, b2 = 16, 3000, 300
        dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=21, phase1_iters=b1, phase2_iters=b2,
                                                        variant=plse.MPMA))
        off = _offspring(orc, grid, g, p, 21)
        dp.offspring = off
        dp.improve(3)
        imp = dp.improved
        _, _, iters = dp.stats(plse.IMPROVED)
        stop_f = 1 if g.l == 1 else 0
        for i in range(p):
            o = orc.plits(grid, off[i], orc.derive_seed(21, 2, 3 * p + i), b1, b2, 0.6, stop_f, tie=oracle.TIE_CANON)
            assert iters[i] == o["iterations"] and np.array_equal(imp[i], o["best"]), (n, i)
        err = capfd.readouterr().err
        m = re.search(r"register mode: (\d+) entries, (\d+) exits", err)
        assert m, err[-500:]
        entries += int(m.group(1))
        exits += int(m.group(2))
    assert entries > 0
    if cap < 32:
        assert exits > 0
