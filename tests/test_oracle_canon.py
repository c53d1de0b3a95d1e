"""Properties of the canonical (order-free) PartialCol policy the GPU implements,
re-pointing the reference's own PartialCol tests (tests/unit/test_partial.cpp)
and acceptance criterion 9 at the oracle's OR_TIE_CANON policy."""
import os

import numpy as np
import pytest

import oracle

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.npz"))
CANON = oracle.TIE_CANON


def _replay_legal(orc, grid, start, trace):
    cur = orc.repair(grid, start).astype(np.int32)
    for st in trace:
        if st["v"] >= 0:
            cur[st["v"]] = st["k"]
            for u in (st["ev0"], st["ev1"]):
                if u >= 0:
                    cur[u] = 0
        f, c = orc.eval(grid, cur.astype(np.uint16))
        assert c == 0
        assert f == st["f_after"]
        assert st["f_after"] - st["f_before"] == -1 + (st["e"] if st["v"] >= 0 else 1)
    return cur


M64 = (1 << 64) - 1


def _splitmix_at(s, j):
    z = (s + (j + 1) * 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def test_canon_draw_definition(orc):
    """the draw of step j is SplitMix64's (j+1)-th output from the 64-bit stream seed s
    (rng.hpp:14-19 evaluated at a counter); it equals stepping the reference's splitmix64 j+1 times"""
    for s in (0, 1, 0x1234_5678_9ABC_DEF0, 2**64 - 1):
        st = s
        for j in range(40):
            assert orc.canon_draw(s, j) == _splitmix_at(s, j)
            st = (st + 0x9E3779B97F4A7C15) & M64
            z = ((st ^ (st >> 30)) * 0xBF58476D1CE4E5B9) & M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
            assert orc.canon_draw(s, j) == z ^ (z >> 31)


def test_canon_streams_are_keyed_by_the_full_seed(orc):
    """Round-1 weakness: a 32-bit folded key made every stream a shift of one 2^32-period sequence, so
    individuals shared draws.  Seeds differing only in their high or only in their low half, and two
    seeds with equal 32-bit folds, now give unrelated draws."""
    a, b = 0x0000_0001_0000_0002, 0x0000_0002_0000_0001  # equal lo32(s ^ s >> 32)
    assert ((a ^ (a >> 32)) & 0xFFFFFFFF) == ((b ^ (b >> 32)) & 0xFFFFFFFF)
    da = {orc.canon_draw(a, j) >> 32 for j in range(2000)}
    db = {orc.canon_draw(b, j) >> 32 for j in range(2000)}
    assert len(da & db) <= 2
    # the window of one individual's generation (180k steps) does not reappear shifted in a sibling's
    sib = [orc.derive_seed(1, 2, 16384 + i) for i in range(64)]
    firsts = {orc.canon_draw(s, 0) for s in sib}
    for s in sib[:8]:
        assert not any(orc.canon_draw(s, j) in firsts for j in range(1, 3000))


def test_canon_draws_are_uniform(orc):
    hi = np.array([orc.canon_draw(77, j) >> 32 for j in range(20000)], np.uint64)
    lo = np.array([orc.canon_draw(77, j) & 0xFFFFFFFF for j in range(20000)], np.uint64)
    for x in (hi, lo):
        h = np.bincount((x * 16 >> 32).astype(np.int64), minlength=16)
        exp = len(x) / 16
        assert ((h - exp) ** 2 / exp).sum() < 45.0  # 15 dof


def test_partialcol_keeps_legal_and_accounts_f(orc):
    """test_partial.cpp:46-64 under the canonical policy"""
    grid = orc.generate_instance(5, 0.5, 61)
    g = orc.preprocess(grid)
    rng = np.random.default_rng(7)
    start = np.array([g.dom[rng.integers(g.dom_off[v], g.dom_off[v + 1])] for v in range(g.nv)], np.uint16)
    o = orc.improve(grid, start, 15, 1000, stop_f=-1, tie=CANON, trace_cap=1000)
    _replay_legal(orc, grid, start, o["trace"])
    assert o["best_f"] <= o["repaired_f"]


def test_free_insertion_gains_one(orc):
    """test_partial.cpp:66-76: all cells empty, the first step colours a vertex for free"""
    grid = np.zeros((3, 3), np.uint16)
    o = orc.improve(grid, np.zeros(9, np.uint16), 3, 1, tie=CANON, trace_cap=1)
    assert o["trace"][0]["level"] == -1 and o["trace"][0]["f_after"] == 8


def test_optimal_input_unchanged(orc):
    """test_partial.cpp:78-86"""
    grid = np.zeros((3, 3), np.uint16)
    s = np.array([1, 2, 3, 2, 3, 1, 3, 1, 2], np.uint16)
    o = orc.improve(grid, s, 1, 1000, tie=CANON)
    assert np.array_equal(o["best"], s) and o["iterations"] == 0


def test_never_loses_to_repair(orc):
    """test_partial.cpp:88-103"""
    rng = np.random.default_rng(55)
    for trial in range(10):
        grid = orc.generate_instance(6, 0.3 + 0.5 * rng.random(), int(rng.integers(0, 2**63)))
        g = orc.preprocess(grid)
        if g.nv == 0:
            continue
        start = np.array([g.dom[rng.integers(g.dom_off[v] + 1, g.dom_off[v + 1])] for v in range(g.nv)], np.uint16)
        o = orc.improve(grid, start, int(rng.integers(0, 2**63)), 2000, tie=CANON)
        assert orc.eval(grid, o["best"])[1] == 0
        assert o["best_f"] <= orc.eval(grid, orc.repair(grid, start))[0]


def test_reaches_exact_optimum(orc):
    """test_partial.cpp:105-127 with the golden exact optima (oracle.hpp:134)"""
    suite = G["suite"]
    rng = np.random.default_rng(3030)
    for i in [k for k in range(len(suite)) if suite[k][0] == 5][:12]:
        grid = G[f"suite_{i}"]
        g = orc.preprocess(grid)
        if g.nv == 0:
            continue
        opt_f = int(suite[i][2])
        best = g.nv
        for restart in range(50):
            start = np.array([g.dom[rng.integers(g.dom_off[v] + 1, g.dom_off[v + 1])] for v in range(g.nv)],
                             np.uint16)
            o = orc.improve(grid, start, int(rng.integers(0, 2**63)), 100 * g.nv, stop_f=opt_f, tie=CANON)
            best = min(best, o["best_f"])
            if best <= opt_f:
                break
        assert best == opt_f


def test_partial_mpma_matches_exact_optima(orc):
    """acceptance criterion 9(b) (acceptance.cpp:73-97, 428-456) on a slice of the 200-instance suite,
    Partial-MPMA with the canonical policy, p=64, <= 50 generations"""
    suite = G["suite"]
    misses = 0
    for i in range(0, 200, 5):
        n, seed, opt_f, opt_score, l = [int(x) for x in suite[i]]
        o = orc.run(G[f"suite_{i}"], p=64, seed=seed, generation_limit=50, tie=CANON)
        if o["best_score"] != opt_score:
            misses += 1
            o = orc.run(G[f"suite_{i}"], p=64, seed=seed ^ 0xABCDEF, generation_limit=50, tie=CANON)
            assert o["best_score"] == opt_score
    assert misses <= 1


def test_tie_break_is_uniform(orc):
    """equal-delta ties uniform at random.  All cells empty, 4x4 grid: the first step has
    16 vertices x 4 colours = 64 free candidates; over many streams every one is chosen ~equally."""
    grid = np.zeros((4, 4), np.uint16)
    counts = np.zeros((16, 5), np.int64)
    trials = 12800
    for s in range(trials):
        o = orc.improve(grid, np.zeros(16, np.uint16), s * 7919 + 1, 1, tie=CANON, trace_cap=1)
        st = o["trace"][0]
        assert st["n_adm"] == 64 and st["level"] == -1
        counts[st["v"], st["k"]] += 1
    obs = counts[:, 1:].reshape(-1)
    exp = trials / 64
    chi2 = float(((obs - exp) ** 2 / exp).sum())
    assert chi2 < 110.0  # 63 dof: p(chi2 > 110) < 1e-4


def test_tenure_formula(orc):
    """T = L + floor(alpha*|V0|) with L uniform in 0..9 (partial.hpp:136-137)"""
    grid = orc.generate_instance(20, 0.5, 9)
    g = orc.preprocess(grid)
    start = orc.init_population(grid, 1, 3)[0]
    o = orc.improve(grid, start, 99, 5000, tie=CANON, trace_cap=5000)
    ls = []
    for st in o["trace"]:
        if st["v"] < 0:
            continue
        base = int(0.6 * st["f_after"])
        L = st["tenure"] - base
        assert 0 <= L <= 9
        ls.append(L)
    hist = np.bincount(ls, minlength=10)
    assert hist.min() > 0.07 * len(ls)
