"""The per-step parity contract of the north star ("gamma tables, chosen moves, tabu lists ... bit-exact
per step against the CPU oracle"): the device state probe (plse_probe) materialises, before chosen steps,
the gamma table the step reads (coloring.hpp:105-116, kept incrementally by coloring.hpp:139-156 in the
oracle; derived from the kernel's occupancy masks on the device) and the live tabu entries
(search_util.hpp:54-81), and both must equal the oracle's at step 0 (post-repair), 1, 100 and 10^4 --
plus the tabu caches must agree with the dense table.  Moves are covered by the trace tests."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

STEPS = [0, 1, 2, 100, 1000, 10_000, 25_000]


@pytest.mark.parametrize("n,r,s", [(30, 0.5, 12345), (60, 0.5, 12345), (70, 0.6, 12345), (60, 0.7, 12345)])
def test_gamma_and_tabu_match_oracle_per_step(plse, orc, n, r, s):
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p, seed, budget = 8, 3, 30_000
    mem = orc.init_population(grid, p, seed)
    pop = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=seed, phase1_iters=budget))
    pop.offspring = mem
    reached = 0
    for idx in (0, 5):
        got, mism = pop.probe(idx, 1, STEPS)
        want = orc.improve_probe(grid, mem[idx], orc.derive_seed(seed, 2, p + idx), budget, STEPS,
                                 tie=oracle.TIE_CANON)
        assert mism == 0
        assert len(got) == len(want) >= 2
        for a, b in zip(got, want):
            assert a["step"] == b["step"]
            assert np.array_equal(a["gamma"], b["gamma"]), f"gamma differs before step {a['step']}"
            assert a["n_tabu"] == b["n_tabu"]
            assert np.array_equal(a["tabu"], b["tabu"]), f"tabu list differs before step {a['step']}"
        reached = max(reached, len(got))
        assert any(d["n_tabu"] > 0 for d in got)
    assert reached >= 3


@pytest.mark.parametrize("n,r,s", [(30, 0.5, 12345), (60, 0.5, 12345), (70, 0.6, 12345)])
def test_plits_gamma_and_tabu_match_oracle_per_step(plse, orc, n, r, s):
    """the same contract for the MPMA variant's PLITS (plits.hpp:96-292): illegal states, colour 0 tabu, a
    fresh tabu clock in phase 2 -- the probe points span both phases"""
    grid = orc.generate_instance(n, r, s)
    g = plse.preprocess(grid)
    p, seed, b1, b2 = 8, 3, 3000, 400
    mem = orc.init_population(grid, p, seed)
    pop = plse.DevicePopulation(g, plse.SolverConfig(p=p, master_seed=seed, phase1_iters=b1, phase2_iters=b2,
                                                     variant=plse.MPMA))
    pop.offspring = mem
    steps = [0, 1, 2, 50, 500, b1 - 1, b1, b1 + 1, b1 + 150]
    for idx in (0, 3):
        got, mism = pop.probe(idx, 1, steps)
        want = orc.improve_probe(grid, mem[idx], orc.derive_seed(seed, 2, p + idx), b1, steps,
                                 tie=oracle.TIE_CANON, plits_budget2=b2)
        assert mism == 0
        assert len(got) == len(want) >= 2
        for a, b in zip(got, want):
            assert a["step"] == b["step"]
            assert np.array_equal(a["gamma"], b["gamma"]), f"gamma differs before step {a['step']}"
            assert a["n_tabu"] == b["n_tabu"]
            assert np.array_equal(a["tabu"], b["tabu"]), f"tabu list differs before step {a['step']}"
