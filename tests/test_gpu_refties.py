"""The reference tie-break on the GPU (tie_mode = TIE_REF, csrc/improve_ref.cu) against the
UNMODIFIED reference compiled in place (oracle/_ref), bit for bit:

* partial_mpma_improve per individual: best colouring, iteration count, best f;
* the per-step trace equals the oracle's OR_TIE_REF trace (itself pinned to the reference);
* run() end to end: best f / score, stop reason, generations, total iterations and the best
  solution equal the reference's run() (engine.hpp:114-262) -- every phase of the generation
  (init, improve, distances, update, matching, crossover) is the reference's.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CASES = [(5, 0.5, 61), (10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (60, 0.5, 12345), (70, 0.6, 12345)]


@pytest.mark.parametrize("n,r,s", CASES)
@pytest.mark.parametrize("budget", [1, 9, 500, 0])
def test_ref_ties_improve_equals_reference(plse, orc, ref, n, r, s, budget):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p = 16
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=3, phase1_iters=budget, tie_mode=plse.TIE_REF))
    off = orc.init_population(grid, p, 3)
    for i in range(0, p, 3):
        off[i] = orc.repair(grid, off[i])
    dp.offspring = off
    gen = 2
    it, bf, bi = dp.improve(gen)
    imp = dp.improved
    f, c, iters = dp.stats(plse.IMPROVED)
    eff = budget if budget > 0 else 100 * g.vertex_count
    stop_f = 1 if g.l == 1 else 0
    for i in range(p):
        seed = orc.derive_seed(3, 2, gen * p + i)
        want = ref.improve(grid, off[i], seed, eff, stop_f=stop_f)
        assert iters[i] == want["iterations"], (i, iters[i], want["iterations"])
        assert np.array_equal(imp[i], want["best"]), i
        assert f[i] == want["best_f"]
    o_bytes = sum(orc.improve(grid, off[i], orc.derive_seed(3, 2, gen * p + i), eff, stop_f=stop_f,
                              tie=oracle.TIE_REF)["alg_bytes"] for i in range(p))
    assert dp.counters().alg_bytes == o_bytes


@pytest.mark.parametrize("n,r,s", [(10, 0.3, 606), (30, 0.5, 12345), (70, 0.6, 12345)])
def test_ref_ties_trace_equals_oracle_ref(plse, orc, n, r, s):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p = 3
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=11, phase1_iters=8000, tie_mode=plse.TIE_REF))
    off = orc.init_population(grid, p, 11)
    dp.offspring = off
    for idx in range(p):
        steps, n_it = dp.trace(idx, 2, 8000)
        o = orc.improve(grid, off[idx], orc.derive_seed(11, 2, 2 * p + idx), 8000, stop_f=1 if g.l == 1 else 0,
                        tie=oracle.TIE_REF, trace_cap=8000)
        assert n_it == o["iterations"]
        for a, b in zip(steps, o["trace"]):
            assert a == b, (idx, a, b)


@pytest.mark.parametrize("n,r,s,p", [(10, 0.5, 3, 16), (20, 0.7, 505, 16), (30, 0.5, 12345, 16),
                                     (12, 0.6, 88, 24)])
def test_ref_ties_run_equals_reference_run(plse, orc, ref, n, r, s, p):
    grid = orc.generate_instance(n, r, s)
    res = plse.run(grid, plse.SolverConfig(p=p, master_seed=7, generation_limit=5, tie_mode=plse.TIE_REF))
    want = ref.run(grid, p=p, seed=7, generation_limit=5, workers=2)
    for k in ("best_f", "best_score", "stop_reason", "generations", "total_iterations", "l", "upper_bound",
              "vertex_count"):
        assert getattr(res, k) == want[k], k
    assert np.array_equal(res.best_solution, want["best_colors"])


def test_ref_ties_run_golden(plse):
    """the same without the compiled reference: tests/golden runs (workers = 1)"""
    import os
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.npz"))
    for row in G["runs"]:
        n, pp, bf, score, opt, stop, gens, its = (int(x) for x in row)
        res = plse.run(G[f"run_inst_{n}"], plse.SolverConfig(p=pp, master_seed=7, generation_limit=5,
                                                             tie_mode=plse.TIE_REF))
        assert (res.best_f, res.best_score, res.generations, res.total_iterations) == (bf, score, gens, its)
        assert np.array_equal(res.best_solution, G[f"run_best_{n}"])


def test_cli_json_with_ref_ties_equals_reference_json(plse, orc, ref, tmp_path):
    """The drop-in claim end to end: `solve --variant partial --tie ref` prints the JSON the reference's
    run() + result_to_json(...).dump(2) print for the same instance, seed and flags."""
    import subprocess
    import sys
    import os
    if not ref.has_result_json():
        pytest.skip("nlohmann/json not found when oracle/_ref was built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    grid = orc.generate_instance(12, 0.6, 88)
    inst = tmp_path / "instance.txt"
    inst.write_text(plse.serialize_instance(grid))
    out = subprocess.run([sys.executable, "-m", "paper_2103_10453_b200", "solve", str(inst), "--seed", "31337",
                          "--pop", "16", "--gen-limit", "5", "--workers", "2", "--variant", "partial", "--tie", "ref"],
                         capture_output=True, text=True, cwd=root, timeout=600)
    assert out.returncode in (0, 2), out.stderr
    r = ref.run(grid, p=16, seed=31337, generation_limit=5, workers=2)
    want = ref.result_json("instance.txt", 12, r, r["stop_reason"], 16, 0.6, 10.0, 20.0, 0, 0, 1, 0, 0, 0, 31337, 2,
                           0.0, 0, 5)
    assert out.stdout == want + "\n"


# ---- PLITS (the MPMA variant) with the reference tie-break, against plits_run / run() themselves

def _plits_offspring(orc, grid, g, p, seed):
    off = orc.init_population(grid, p, seed)
    rng = np.random.default_rng(seed)
    for i in range(1, p, 4):
        off[i][rng.random(g.vertex_count) < 0.3] = 0
    for i in range(2, p, 4):
        off[i] = orc.repair(grid, off[i])
    return off


@pytest.mark.parametrize("n,r,s", CASES)
@pytest.mark.parametrize("b1,b2", [(1, 1), (37, 5), (600, 0), (0, 0)])
def test_ref_ties_plits_equals_plits_run(plse, orc, ref, n, r, s, b1, b2):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p = 12
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=5, phase1_iters=b1, phase2_iters=b2,
                                                    variant=plse.MPMA, tie_mode=plse.TIE_REF))
    off = _plits_offspring(orc, grid, g, p, 5)
    dp.offspring = off
    gen = 2
    dp.improve(gen)
    imp = dp.improved
    f, c, iters = dp.stats(plse.IMPROVED)
    stop_f = 1 if g.l == 1 else 0
    want_bytes = 0.0
    for i in range(p):
        seed = orc.derive_seed(5, 2, gen * p + i)
        best, its = ref.plits(grid, off[i], seed, b1, b2, 0.6, stop_f)
        assert iters[i] == its, (i, iters[i], its)
        assert np.array_equal(imp[i], best), i
        want_bytes += orc.plits(grid, off[i], seed, b1, b2, 0.6, stop_f, tie=oracle.TIE_REF)["alg_bytes"]
    assert dp.counters().alg_bytes == want_bytes


@pytest.mark.parametrize("n,r,s", [(10, 0.3, 606), (30, 0.5, 12345), (70, 0.6, 12345)])
def test_ref_ties_plits_trace_equals_oracle_ref(plse, orc, n, r, s):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p, b1, b2 = 3, 2500, 150
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=13, phase1_iters=b1, phase2_iters=b2,
                                                    variant=plse.MPMA, tie_mode=plse.TIE_REF))
    off = _plits_offspring(orc, grid, g, p, 13)
    dp.offspring = off
    for idx in range(p):
        steps, n_it = dp.trace(idx, 4, b1 + b2)
        o = orc.plits(grid, off[idx], orc.derive_seed(13, 2, 4 * p + idx), b1, b2, 0.6, 1 if g.l == 1 else 0,
                      tie=oracle.TIE_REF, trace_cap=b1 + b2)
        assert n_it == o["iterations"]
        for a_, e in zip(steps, o["trace"]):
            want = dict(step=e["step"], v=e["v"], k=e["k"] if e["v"] >= 0 else 0, e=e["phase"],
                        ev0=e["from_"] if e["v"] >= 0 else 0, ev1=e["active"], f_before=e["f"], f_after=e["c"],
                        best_f=e["best_scaled"], tenure=e["tenure"], n_adm=e["n_adm"] if e["v"] >= 0 else 0,
                        level=e["delta"] if e["v"] >= 0 else 0)
            assert a_ == want, (idx, a_, want)


@pytest.mark.parametrize("n,r,s,p", [(10, 0.5, 3, 8), (20, 0.6, 9, 12), (30, 0.5, 4, 16), (12, 0.6, 88, 16)])
def test_ref_ties_mpma_run_equals_reference_run(plse, orc, ref, n, r, s, p):
    grid = orc.generate_instance(n, r, s)
    res = plse.run(grid, plse.SolverConfig(p=p, master_seed=s, generation_limit=4, phase1_iters=500,
                                           variant=plse.MPMA, tie_mode=plse.TIE_REF))
    want = ref.run(grid, p=p, seed=s, generation_limit=4, phase1_iters=500, variant=0, workers=2)
    for k in ("best_f", "best_score", "stop_reason", "generations", "total_iterations"):
        assert getattr(res, k) == want[k], k
    assert np.array_equal(res.best_solution, want["best_colors"])
