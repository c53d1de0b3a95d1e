"""Randomised end-to-end parity: whole run()s over random instances and configurations.

Canonical tie-break against the oracle's OR_TIE_CANON run, and the reference tie-break against
the compiled reference's run() itself, for both variants: best f, score, stop reason,
generations, total iterations and the best solution, bit for bit.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _config(rng):
    n = int(rng.integers(3, 36))
    r = float(rng.uniform(0.1, 0.9))
    s = int(rng.integers(0, 2**31))
    p = int(rng.integers(2, 33))
    cross = int(rng.integers(0, 3))
    match = int(rng.integers(0, 2))
    excl = int(rng.integers(0, 3))
    gens = int(rng.integers(1, 5))
    b1 = int(rng.choice([0, 50, 400, 2000]))
    b2 = int(rng.choice([0, 5, 60]))
    alpha = float(rng.choice([0.6, 0.3, 1.0]))
    seed = int(rng.integers(0, 2**62))
    return n, r, s, p, cross, match, excl, gens, b1, b2, alpha, seed


@pytest.mark.parametrize("case", range(24))
def test_fuzz_canonical_runs_equal_oracle(plse, orc, case):
    rng = np.random.default_rng(1000 + case)
    n, r, s, p, cross, match, excl, gens, b1, b2, alpha, seed = _config(rng)
    variant = case % 2  # 0 = MPMA (PLITS), 1 = Partial-MPMA
    grid = orc.generate_instance(n, r, s)
    if plse.preprocess(grid).vertex_count == 0:
        pytest.skip("trivial instance")
    res = plse.run(grid, plse.SolverConfig(p=p, alpha=alpha, crossover=cross, matching=match, exclusion=excl,
                                           master_seed=seed, generation_limit=gens, phase1_iters=b1, phase2_iters=b2,
                                           variant=variant, beta=20.0))
    o = orc.run(grid, p=p, alpha=alpha, crossover=cross, matching=match, exclusion=excl, seed=seed,
                generation_limit=gens, phase1_iters=b1, phase2_iters=b2, tie=oracle.TIE_CANON, variant=variant)
    for k in ("best_f", "best_score", "stop_reason", "generations", "total_iterations"):
        assert getattr(res, k) == o[k], (k, case)
    assert np.array_equal(res.best_solution, o["best_colors"])


@pytest.mark.parametrize("case", range(24))
def test_fuzz_reference_tie_runs_equal_reference(plse, ref, case):
    rng = np.random.default_rng(2000 + case)
    n, r, s, p, cross, match, excl, gens, b1, b2, alpha, seed = _config(rng)
    variant = case % 2
    grid = ref.generate_instance(n, r, s)
    if plse.preprocess(grid).vertex_count == 0:
        pytest.skip("trivial instance")
    res = plse.run(grid, plse.SolverConfig(p=p, alpha=alpha, crossover=cross, matching=match, exclusion=excl,
                                           master_seed=seed, generation_limit=gens, phase1_iters=b1, phase2_iters=b2,
                                           variant=variant, tie_mode=plse.TIE_REF))
    want = ref.run(grid, p=p, alpha=alpha, crossover=cross, matching=match, exclusion=excl, seed=seed,
                   generation_limit=gens, phase1_iters=b1, phase2_iters=b2, variant=variant, workers=3)
    for k in ("best_f", "best_score", "stop_reason", "generations", "total_iterations"):
        assert getattr(res, k) == want[k], (k, case)
    assert np.array_equal(res.best_solution, want["best_colors"])
