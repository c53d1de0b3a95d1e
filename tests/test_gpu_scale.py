"""Parity at the headline configuration (BASELINE C3: generate_instance(60, 0.5, 12345), p = 16384, the full
100|V| = 180,000-step budget) -- the paths only this size exercises:

* improve: 4144 warp slots (28 per SM) serve 16384 individuals through the work counter, so every individual with an
  index beyond the slot count runs on a slot that already searched one or more individuals in the same launch
  (the monotone tabu clock and the cache reset); sampled individuals are compared with the oracle;
* K3: the grouped raster of k_sim_tc over 128 tile rows (ten full 12-row groups and a partial one), on the
  cross block and the upper-triangle fresh block, sampled rows against numpy;
* the pool update: 32 admission blocks of 1024 candidates, fed to the oracle's update_population with the
  device's own distance blocks: members, dist, shortfall must be equal;
* matching with 512-word exclusion rows and AUX crossover, over three generations with run-scoped exclusion;
* PLITS at p = 16384 (1184 slots, ~14 individuals per slot).

The oracle runs in a thread pool (ctypes releases the GIL) so the module stays within a few minutes."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

P, SEED = 16384, 1
SLOTS_HINT = 4144  # 148 SMs x 28 warps; the test reads the actual count below


def _sample(p, k, rng, must=()):
    idx = set(int(x) for x in must)
    idx.update(int(x) for x in np.linspace(0, p - 1, k // 2).round())
    while len(idx) < k:
        idx.add(int(rng.integers(0, p)))
    return sorted(idx)


def _hamming_rows(A, B, rows):
    return np.stack([(A[i][None, :] != B).sum(1) for i in rows]).astype(np.int64)


def test_c3_headline_generations(plse, orc):
    grid = orc.generate_instance(60, 0.5, 12345)
    g = plse.preprocess(grid)
    nv = g.vertex_count
    budget = 100 * nv
    pop = plse.DevicePopulation(g, plse.SolverConfig(p=P, master_seed=SEED))
    slots = pop.counters().slots
    assert slots < P  # slots are reused inside one launch
    hint = min(SLOTS_HINT, slots)
    pop.initialize_population()
    mem = pop.members
    assert np.array_equal(mem[:64], orc.init_population(grid, 64, SEED))
    dist = pop.dist
    pop.offspring = mem
    off = mem
    excl = np.zeros((P, P), np.uint8)
    rng = np.random.default_rng(7)
    pool = ThreadPoolExecutor(max_workers=16)
    for gen in (1, 2, 3):
        it, bf, bi = pop.improve(gen)
        imp = pop.improved
        f_imp, c_imp, iters = pop.stats(plse.IMPROVED)
        assert it == int(iters.sum()) and bf == int(f_imp.min()) and bi == int(np.argmin(f_imp))
        # (a) sampled individuals, most of them served by a slot's 2nd..4th search of the launch
        k = 64 if gen == 1 else 24
        idx = _sample(P, k, rng, must=[hint, hint + 1, 2 * hint + 3, 3 * hint + 7, P - 1])
        assert sum(i >= hint for i in idx) >= k // 2
        futs = {i: pool.submit(orc.improve, grid, off[i], orc.derive_seed(SEED, 2, gen * P + i), budget,
                               0.6, 0, oracle.TIE_CANON) for i in idx}
        for i, fu in futs.items():
            o = fu.result()
            assert iters[i] == o["iterations"], (gen, i)
            assert np.array_equal(imp[i], o["best"]), (gen, i)
        # (b) K3 blocks: sampled rows (incl. the partial last raster group, rows >= 15360) against numpy
        pop.compute_cross_distances()
        cross = pop.get_dist(plse.CROSS)
        fresh = pop.get_dist(plse.FRESH)
        if gen == 1:
            rows = _sample(P, 256, rng, must=[0, 127, 128, 1535, 1536, 15359, 15360, P - 1])
            assert np.array_equal(cross[rows], _hamming_rows(mem, imp, rows))
            assert np.array_equal(fresh[rows], _hamming_rows(imp, imp, rows))
        else:
            rows = _sample(P, 32, rng, must=[15360, P - 1])
            assert np.array_equal(cross[rows], _hamming_rows(mem, imp, rows))
            assert np.array_equal(fresh[rows], _hamming_rows(imp, imp, rows))
        # (c) the update fed the device's own blocks: 2p = 32768 candidates, 32 admission blocks
        want = orc.update(grid, mem, dist, imp, cross, fresh)
        del cross, fresh
        info = pop.update_population()
        mem = pop.members
        assert info.pool_best_f == want["pool_best_f"]
        assert info.shortfall_slots == want["shortfall_slots"]
        assert np.array_equal(mem, want["members"])
        dist = pop.dist
        assert np.array_equal(dist, want["dist"])
        # (d) matching (512-word exclusion rows, run scope) + AUX crossover
        pop.build_offspring(gen)
        off = pop.offspring
        want_off, want_part = orc.offspring(grid, mem, dist, excl, SEED, gen)
        assert np.array_equal(pop.partners(), want_part)
        assert np.array_equal(off, want_off)
    pool.shutdown()
    pop.close()


def test_c3_plits_slot_reuse(plse, orc):
    """k_plits at p = 16384: ~14 individuals per warp slot in one launch (a bounded phase-1 budget keeps
    the oracle side short; the slot reuse is independent of the budget)."""
    grid = orc.generate_instance(60, 0.5, 12345)
    g = plse.preprocess(grid)
    b1, b2 = 3000, 0
    pop = plse.DevicePopulation(g, plse.SolverConfig(p=P, master_seed=SEED, phase1_iters=b1, phase2_iters=b2,
                                                     variant=plse.MPMA))
    slots = pop.counters().slots
    assert P / slots >= 10
    pop.initialize_population()
    off = pop.members
    pop.offspring = off
    pop.improve(1)
    imp = pop.improved
    _, _, iters = pop.stats(plse.IMPROVED)
    rng = np.random.default_rng(3)
    idx = _sample(P, 48, rng, must=[slots, 5 * slots + 1, 13 * slots + 2, P - 1])
    with ThreadPoolExecutor(max_workers=16) as ex:
        futs = {i: ex.submit(orc.plits, grid, off[i], orc.derive_seed(SEED, 2, P + i), b1, b2, 0.6, 0,
                             tie=oracle.TIE_CANON) for i in idx}
        for i, fu in futs.items():
            o = fu.result()
            assert iters[i] == o["iterations"], i
            assert np.array_equal(imp[i], o["best"]), i
