"""GPU edge cases the reference's own tests exercise (test_lsgraph.cpp, test_oracle.cpp,
test_engine.cpp, acceptance c3): l = 1 instances, empty grids, the 64-colour mask
boundary, tiny graphs, every crossover / matching / exclusion mode, tabu-heavy alpha.
Each is compared bit-exactly with the oracle's canonical run."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _same_run(plse, orc, grid, **kw):
    res = plse.run(grid, plse.SolverConfig(**kw))
    o = orc.run(grid, tie=oracle.TIE_CANON, p=kw["p"], seed=kw.get("master_seed", 0),
                alpha=kw.get("alpha", 0.6), gamma=kw.get("gamma", 10.0), beta=kw.get("beta", 20.0),
                phase1_iters=kw.get("phase1_iters", 0), crossover=kw.get("crossover", 0),
                matching=kw.get("matching", 0), exclusion=kw.get("exclusion", 0),
                generation_limit=kw.get("generation_limit", 0), iteration_limit=kw.get("iteration_limit", 0))
    for k in ("best_f", "best_score", "stop_reason", "generations", "total_iterations", "l", "upper_bound"):
        assert getattr(res, k) == o[k], (k, getattr(res, k), o[k])
    assert bool(res.proven_optimal) == bool(o["proven_optimal"])
    assert np.array_equal(res.best_solution, o["best_colors"])
    return res


def test_fig1_instance_l1_bound_7(plse, orc):
    """acceptance c3 / test_oracle.cpp:9-18: l = 1, upper bound n^2 - 2 = 7, optimum 7, stop_f = 1"""
    grid = np.array([[1, 0, 0], [2, 0, 0], [0, 0, 3]], np.uint16)
    res = _same_run(plse, orc, grid, p=8, master_seed=1, generation_limit=5)
    assert res.l == 1 and res.upper_bound == 7 and res.best_score == 7 and res.proven_optimal


@pytest.mark.parametrize("n", [2, 3, 5])
def test_empty_grids(plse, orc, n):
    res = _same_run(plse, orc, np.zeros((n, n), np.uint16), p=8, master_seed=2, generation_limit=4)
    assert res.best_score == n * n


@pytest.mark.parametrize("n,r,s", [(63, 0.5, 1), (64, 0.5, 2), (65, 0.6, 3), (127, 0.8, 4)])
def test_mask_word_boundaries(plse, orc, n, r, s):
    """W = 1 for n <= 63, W = 2 for 64 <= n <= 127"""
    grid = orc.generate_instance(n, r, s)
    _same_run(plse, orc, grid, p=8, master_seed=3, generation_limit=2, phase1_iters=3000)


def test_order_128_is_outside_the_device_envelope(plse):
    with pytest.raises(NotImplementedError):
        plse.run(np.zeros((128, 128), np.uint16), plse.SolverConfig(p=4, generation_limit=1))


@pytest.mark.parametrize("n,r,s,p", [(4, 0.3, 7, 5), (5, 0.6, 11, 37), (6, 0.8, 3, 16)])
def test_tiny_graphs_odd_populations(plse, orc, n, r, s, p):
    grid = orc.generate_instance(n, r, s)
    _same_run(plse, orc, grid, p=p, master_seed=4, generation_limit=6)


@pytest.mark.parametrize("x,m,e", [(0, 0, 0), (0, 0, 1), (0, 0, 2), (0, 1, 0), (1, 0, 0), (1, 1, 2), (2, 0, 0)])
def test_every_offspring_mode(plse, orc, x, m, e):
    grid = orc.generate_instance(12, 0.6, 77)
    _same_run(plse, orc, grid, p=24, master_seed=5, generation_limit=5, crossover=x, matching=m, exclusion=e,
              phase1_iters=600)


@pytest.mark.parametrize("alpha", [0.0, 1.0])
def test_tenure_extremes(plse, orc, alpha):
    """alpha = 0 (tenure L only) and alpha = 1 (the largest tenure with reference-equivalent tabu reuse)"""
    grid = orc.generate_instance(20, 0.5, 9)
    _same_run(plse, orc, grid, p=16, master_seed=6, generation_limit=3, alpha=alpha, phase1_iters=4000)


def test_iteration_limit_and_spacing_params(plse, orc):
    grid = orc.generate_instance(15, 0.5, 21)
    _same_run(plse, orc, grid, p=16, master_seed=7, iteration_limit=20000, gamma=4.0, beta=6.0,
              phase1_iters=2500)


def test_lsc_instance_run(plse, orc):
    grid = orc.lsc_instance(20, 0.4, 7)
    _same_run(plse, orc, grid, p=16, master_seed=8, generation_limit=2, phase1_iters=5000)


@pytest.mark.parametrize("variant,tie", [("partial", 0), ("partial", 1), ("mpma", 0), ("mpma", 1)])
def test_results_do_not_depend_on_launch_geometry(plse, orc, monkeypatch, variant, tie):
    """Warp slots keep tabu state across individuals (monotone clocks, possibly-tabu masks) and the
    block shape follows the population size: the same population improved under different block
    shapes (one-warp CTAs, 8-warp CTAs, the 28-warp CTA of k_improve, the default) -- so different
    individual -> slot assignments, with p = 6000 above the resident slot count so that slots are reused
    inside one launch -- must give identical colourings and iteration counts.  (compute-sanitizer is closed
    on this GPU pool; this, the trace parity and the oracle comparisons are the race evidence.)"""
    grid = orc.generate_instance(20, 0.5, 9)
    g = plse.preprocess(grid)
    outs = []
    shapes = ("1", "8", "28", "0") if (variant, tie) == ("partial", 0) else ("1", "8", "0")
    for wpc in shapes:
        monkeypatch.setenv("PLSE_IMPROVE_WPC", wpc)
        dp = plse.DevicePopulation(g, plse.SolverConfig(
            p=6000, master_seed=4, phase1_iters=3000 if variant == "partial" else 800, tie_mode=tie,
            variant=plse.MPMA if variant == "mpma" else plse.PARTIAL))
        if wpc != "0":
            assert dp.counters().slots < 6000
        dp.initialize_population()
        dp.offspring = dp.members
        res = []
        for gen in (1, 2, 3):  # slots are reused across launches too
            dp.improve(gen)
            f, c, it = dp.stats(plse.IMPROVED)
            res.append((dp.improved.copy(), f.copy(), it.copy()))
        outs.append(res)
        dp.close()
    for other in outs[1:]:
        for (a_col, a_f, a_it), (b_col, b_f, b_it) in zip(outs[0], other):
            assert np.array_equal(a_col, b_col) and np.array_equal(a_f, b_f) and np.array_equal(a_it, b_it)


def test_two_word_masks_in_the_28_warp_cta(plse, orc, monkeypatch):
    """n = 70 (two mask words per vertex, the C4 instance) in k_improve's 28-warp CTA -- the shape whose
    shared memory now fits n = 70 (its 32-warp CTA did not) -- with p = 6000 above the resident slot count:
    sampled individuals, including ones served by a reused slot, equal the oracle's."""
    monkeypatch.setenv("PLSE_IMPROVE_WPC", "28")
    grid = orc.generate_instance(70, 0.6, 12345)
    g = plse.preprocess(grid)
    p, budget = 6000, 2000
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=6, phase1_iters=budget))
    assert dp.counters().slots < p
    dp.initialize_population()
    off = dp.members
    dp.offspring = off
    dp.improve(1)
    imp = dp.improved
    _, _, iters = dp.stats(plse.IMPROVED)
    for i in (0, 1, 147, 148 * 27 + 5, 4200, 5999):
        o = orc.improve(grid, off[i], orc.derive_seed(6, 2, p + i), budget, 0.6, 0, oracle.TIE_CANON)
        assert iters[i] == o["iterations"] and np.array_equal(imp[i], o["best"]), i
    dp.close()
