"""GPU (canonical tie-break) vs the C oracle, bit-exact, through the C ABI.

Parity bar (north star): gamma-derived moves, chosen moves, tabu tenures,
offspring and distance matrices bit-exact per step; final colourings, best f
and iteration counts identical for a fixed seed.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

# BASELINE configs C1 (30, 0.5), C2 (50, 0.4), C3 (60, 0.5), C4 (70, 0.6) at the instance seed 12345, and C5's
# order-70 LSC stand-in builders::lsc_instance(70, 0.4, 7) (|V| = 2940, two mask words), plus small edge cases
CASES = [(5, 0.5, 61), (10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (50, 0.4, 12345), (60, 0.5, 12345),
         (70, 0.6, 12345), (70, 0.4, "lsc7")]


def _grid(orc, n, r, s):
    if isinstance(s, str) and s.startswith("lsc"):
        return orc.lsc_instance(n, r, int(s[3:]))
    return orc.generate_instance(n, r, s)


def _pop(P, grid, p, seed=7, **kw):
    g = P.preprocess(grid)
    cfg = P.SolverConfig(p=p, master_seed=seed, **kw)
    return g, P.DevicePopulation(g, cfg)


@pytest.mark.parametrize("n,r,s", CASES)
def test_init_population_matches_reference_stream(plse, orc, n, r, s):
    grid = _grid(orc, n, r, s)
    g, dp = _pop(plse, grid, 16, seed=99)
    dp.initialize_population()
    mem = orc.init_population(grid, 16, 99)
    assert np.array_equal(dp.members, mem)
    assert np.array_equal(dp.dist, orc.full_distances(mem))
    f, c, _ = dp.stats()
    for i in range(16):
        assert (f[i], c[i]) == orc.eval(grid, mem[i])


@pytest.mark.parametrize("n,r,s", CASES)
@pytest.mark.parametrize("budget", [1, 7, 300, 0])
def test_improve_matches_oracle(plse, orc, n, r, s, budget):
    grid = _grid(orc, n, r, s)
    g = plse.preprocess(grid)
    p = 24
    cfg = plse.SolverConfig(p=p, master_seed=3, phase1_iters=budget)
    dp = plse.DevicePopulation(g, cfg)
    dp.initialize_population()
    off = orc.init_population(grid, p, 3)
    # mix fully random (heavy repair) and legal partial inputs
    for i in range(0, p, 3):
        off[i] = orc.repair(grid, off[i])
    dp.offspring = off
    gen = 1
    it, bf, bi = dp.improve(gen)
    imp = dp.improved
    f, c, iters = dp.stats(plse.IMPROVED)
    tot = 0
    want_bytes = 0.0
    eff_budget = budget if budget > 0 else 100 * g.vertex_count
    stop_f = 1 if g.l == 1 else 0
    for i in range(p):
        seed = orc.derive_seed(3, 2, gen * p + i)
        o = orc.improve(grid, off[i], seed, eff_budget, stop_f=stop_f, tie=oracle.TIE_CANON)
        assert iters[i] == o["iterations"], (i, iters[i], o["iterations"])
        assert f[i] == o["best_f"]
        assert np.array_equal(imp[i], o["best"]), i
        tot += o["iterations"]
        want_bytes += o["alg_bytes"]
    assert it == tot
    assert bf == min(f)
    assert bi == int(np.argmin(f))
    assert dp.counters().alg_bytes == want_bytes


@pytest.mark.parametrize("n,r,s", [(20, 0.7, 505), (30, 0.5, 12345), (60, 0.5, 12345), (70, 0.6, 12345)])
def test_per_step_trace_matches_oracle(plse, orc, n, r, s):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p = 4
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=11, phase1_iters=20000))
    dp.initialize_population()
    off = orc.init_population(grid, p, 11)
    dp.offspring = off
    for idx in range(p):
        steps, n_it = dp.trace(idx, 2, 20000)
        o = orc.improve(grid, off[idx], orc.derive_seed(11, 2, 2 * p + idx), 20000,
                        stop_f=1 if g.l == 1 else 0, trace_cap=20000)
        assert n_it == o["iterations"]
        assert len(steps) == len(o["trace"])
        for a, b in zip(steps, o["trace"]):
            assert a == b, (idx, a, b)


@pytest.mark.parametrize("n,r,s", [(10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345)])
def test_population_phases_match_reference(plse, orc, ref, n, r, s):
    """distances, update (incl. shortfall), matching + AUX crossover over several generations."""
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p = 32
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=55, phase1_iters=2000))
    dp.initialize_population()
    mem, dist = ref.init_population(grid, p, 55)
    off = mem.copy()
    ex = ref.new_exclusion(p)
    dp.offspring = off
    for gen in range(1, 6):
        dp.improve(gen)
        imp = dp.improved
        for i in range(p):
            o = orc.improve(grid, off[i], orc.derive_seed(55, 2, gen * p + i), 2000, stop_f=1 if g.l == 1 else 0)
            assert np.array_equal(imp[i], o["best"])
        dp.compute_cross_distances()
        cr, fr = ref.cross_distances(grid, mem, imp)
        assert np.array_equal(dp.get_dist(plse.CROSS), cr)
        assert np.array_equal(dp.get_dist(plse.FRESH), fr)
        info = dp.update_population()
        u = ref.update(grid, mem, dist, imp, cr, fr)
        assert info.pool_best_f == u["pool_best_f"]
        assert info.shortfall_slots == u["shortfall_slots"]
        mem, dist = u["members"], u["dist"]
        assert np.array_equal(dp.members, mem)
        assert np.array_equal(dp.dist, dist)
        dp.build_offspring(gen)
        off = ref.offspring(grid, mem, dist, ex, 55, gen)
        assert np.array_equal(dp.offspring, off), gen


@pytest.mark.parametrize("mode", [(1, 1, 0), (2, 0, 0), (0, 0, 2), (0, 1, 1), (0, 0, 1)])
def test_offspring_modes_match_reference(plse, orc, ref, mode):
    x, m, e = mode
    grid = orc.generate_instance(20, 0.7, 505)
    g = plse.preprocess(grid)
    p = 32
    dp = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=9, crossover=x, matching=m, exclusion=e))
    mem = np.stack([orc.repair(grid, c) for c in orc.init_population(grid, p, 9)])
    dist = orc.full_distances(mem)
    dp.members = mem
    dp.dist = dist
    ex = ref.new_exclusion(p)
    for gen in range(1, 5):
        if e == 1:
            dp.reset_exclusion()
            ref.lib.ref_excl_reset(ex, p)
        dp.build_offspring(gen)
        want = ref.offspring(grid, mem, dist, ex, 9, gen, crossover=x, matching=m, exclusion=e)
        assert np.array_equal(dp.offspring, want), (mode, gen)


@pytest.mark.parametrize("n,r,s,p", [(10, 0.5, 3, 16), (20, 0.7, 505, 16), (30, 0.5, 12345, 16)])
def test_run_matches_oracle(plse, orc, n, r, s, p):
    grid = orc.generate_instance(n, r, s)
    res = plse.run(grid, plse.SolverConfig(p=p, master_seed=7, generation_limit=4))
    o = orc.run(grid, p=p, seed=7, generation_limit=4, tie=oracle.TIE_CANON)
    for k in ("best_f", "best_score", "stop_reason", "generations", "total_iterations", "l", "upper_bound"):
        assert getattr(res, k) == o[k], k
    assert bool(res.proven_optimal) == bool(o["proven_optimal"])
    assert np.array_equal(res.best_solution, o["best_colors"])


def test_two_device_islands_match_island_restatement(plse, orc):
    """Island model at G=2 on one GPU (sequentially, no cross-kernel waits): stream offsets,
    elite export / migrant import and the per-island phases vs tests/island_sim.py."""
    import sys
    import os
    import torch
    sys.path.insert(0, os.path.dirname(__file__))
    import island_sim as S

    n, r, s, p, seed, gens, budget, elites = 10, 0.5, 3, 12, 21, 3, 400, 3
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    pops = [plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=seed, phase1_iters=budget,
                                                       p_total=2 * p, offset=rk * p)) for rk in range(2)]
    for pop in pops:
        pop.initialize_population()
        pop.offspring = pop.members
    rb = pops[0].row_bytes
    for gen in range(1, gens + 1):
        for pop in pops:
            pop.improve(gen)
        # the exchange after the improve phase: each island's best members become extra pool candidates
        # of the other island's update (in the order distances-before / distances-after the import)
        bufs = [torch.empty((elites, rb), dtype=torch.uint8, device="cuda") for _ in pops]
        for pop, b in zip(pops, bufs):
            pop.export_elites(elites, b.data_ptr())
        torch.cuda.synchronize()
        if gen % 2:
            pops[0].import_migrants(elites, bufs[1].data_ptr())
            pops[1].import_migrants(elites, bufs[0].data_ptr())
        for pop in pops:
            pop.compute_cross_distances()
        if not gen % 2:
            pops[0].import_migrants(elites, bufs[1].data_ptr())
            pops[1].import_migrants(elites, bufs[0].data_ptr())
        for pop in pops:
            pop.update_population()
            pop.build_offspring(gen)
    want = S.simulate(orc, grid, p, 2, seed, gens, budget, elites)
    for pop, w in zip(pops, want):
        assert np.array_equal(pop.members, w)


@pytest.mark.parametrize("p", [300, 1024])
def test_tensor_core_distances_match_cuda_core(plse, orc, p, monkeypatch):
    """K3 on tcgen05 (one-hot i8 UMMA) vs the CUDA-core Hamming kernel, both exact, at a size with
    partial 128x256 tiles (p=300) and full tiles (p=1024)."""
    grid = orc.generate_instance(60, 0.5, 12345)
    g = plse.preprocess(grid)
    rng = np.random.default_rng(p)
    mem = orc.init_population(grid, p, 5)
    # mix fully coloured, partially uncoloured and repaired (legal) rows
    for i in range(0, p, 3):
        mem[i, rng.random(g.vertex_count) < 0.4] = 0
    monkeypatch.setenv("PLSE_TC", "1")
    a = plse.DevicePopulation(g, plse.SolverConfig(p=p))
    monkeypatch.setenv("PLSE_TC", "0")
    b = plse.DevicePopulation(g, plse.SolverConfig(p=p))
    for pop in (a, b):
        pop.members = mem
        pop.compute_full_distances()
    da, db = a.dist, b.dist
    assert np.array_equal(da, db)
    sample = rng.integers(0, p, size=(64, 2))
    for i, j in sample:
        assert da[i, j] == int((mem[i] != mem[j]).sum())


def test_race_mode_reaches_target_and_stops_early(plse, orc):
    grid = orc.generate_instance(30, 0.5, 12345)
    full = plse.run(grid, plse.SolverConfig(p=256, master_seed=3, generation_limit=3))
    race = plse.run(grid, plse.SolverConfig(p=256, master_seed=3, generation_limit=3,
                                           target_score=float(full.best_score), race=True))
    assert race.best_score >= full.best_score
    assert race.total_iterations <= full.total_iterations
    assert race.stop_reason in ("optimal", "target")
