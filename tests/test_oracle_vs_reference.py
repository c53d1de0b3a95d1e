"""Randomised cross-check of the C oracle against the compiled reference
(oracle/_ref).  Skipped where the reference was not built."""
import numpy as np
import pytest

import oracle


def test_instances_graphs_and_trajectories(orc, ref):
    rng = np.random.default_rng(1)
    for _ in range(12):
        n = int(rng.integers(4, 25))
        r = float(rng.uniform(0.2, 0.8))
        s = int(rng.integers(0, 2**63))
        a, b = orc.generate_instance(n, r, s), ref.generate_instance(n, r, s)
        assert np.array_equal(a, b)
        ga, gb = orc.preprocess(a), ref.preprocess(a)
        assert ga.same_as(gb)
        if ga.nv == 0:
            continue
        mem, dist = ref.init_population(a, 6, s & 0xFFFF)
        assert np.array_equal(orc.init_population(a, 6, s & 0xFFFF), mem)
        assert np.array_equal(orc.full_distances(mem), dist)
        for i in range(6):
            seed = int(rng.integers(0, 2**63))
            alpha = float(rng.choice([0.0, 0.3, 0.6, 1.0]))
            o = orc.improve(a, mem[i], seed, 50 * ga.nv, alpha=alpha, tie=oracle.TIE_REF)
            w = ref.improve(a, mem[i], seed, 50 * ga.nv, alpha=alpha)
            assert o["iterations"] == w["iterations"]
            assert np.array_equal(o["best"], w["best"])


@pytest.mark.parametrize("mode", [(0, 0, 0), (1, 1, 0), (2, 0, 0), (0, 0, 1), (0, 0, 2), (0, 1, 2)])
def test_generations(orc, ref, mode):
    x, m, e = mode
    grid = orc.generate_instance(12, 0.6, 77)
    g = orc.preprocess(grid)
    p = 12
    mem, dist = ref.init_population(grid, p, 5)
    mo, do, mr, dr = mem.copy(), dist.copy(), mem.copy(), dist.copy()
    excl = np.zeros((p, p), np.uint8)
    ex = ref.new_exclusion(p)
    off = mem.copy()
    for gen in range(1, 8):
        imp = np.stack([orc.improve(grid, off[i], orc.derive_seed(5, 2, gen * p + i), 20 * g.nv,
                                    tie=oracle.TIE_REF)["best"] for i in range(p)])
        c1, f1 = orc.cross_distances(mo, imp)
        c2, f2 = ref.cross_distances(grid, mr, imp)
        assert np.array_equal(c1, c2) and np.array_equal(f1, f2)
        u1, u2 = orc.update(grid, mo, do, imp, c1, f1), ref.update(grid, mr, dr, imp, c2, f2)
        assert np.array_equal(u1["members"], u2["members"]) and np.array_equal(u1["dist"], u2["dist"])
        assert u1["shortfall_slots"] == u2["shortfall_slots"] and u1["pool_best_f"] == u2["pool_best_f"]
        mo, do, mr, dr = u1["members"], u1["dist"], u2["members"], u2["dist"]
        if e == 1:
            excl[:] = 0
            ref.lib.ref_excl_reset(ex, p)
        o1, _ = orc.offspring(grid, mo, do, excl, 5, gen, crossover=x, matching=m, exclusion=e)
        o2 = ref.offspring(grid, mr, dr, ex, 5, gen, crossover=x, matching=m, exclusion=e)
        assert np.array_equal(o1, o2)
        off = o1


def test_full_run_ref_policy(orc, ref):
    for n, r, s, p in [(8, 0.5, 1, 8), (15, 0.6, 2, 12), (25, 0.4, 3, 8)]:
        grid = orc.generate_instance(n, r, s)
        a = orc.run(grid, p=p, seed=11, generation_limit=3, tie=oracle.TIE_REF)
        b = ref.run(grid, p=p, seed=11, generation_limit=3, workers=1)
        for k in ("best_f", "best_score", "proven_optimal", "stop_reason", "generations", "total_iterations"):
            assert a[k] == b[k], k
        assert np.array_equal(a["best_colors"], b["best_colors"])
