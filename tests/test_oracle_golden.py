"""The C oracle (OR_TIE_REF policy) against golden vectors recorded from the
real reference (tests/golden/make_golden.py).  Runs without /root/reference."""
import os

import numpy as np
import pytest

import oracle

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.npz"))

INST = [(5, 0.5, 61), (10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (60, 0.5, 12345), (70, 0.6, 12345),
        (50, 0.4, 12345), (4, 0.2, 7), (6, 0.8, 3)]


@pytest.mark.parametrize("n,r,s", INST)
def test_generate_instance_and_preprocess(orc, n, r, s):
    grid = orc.generate_instance(n, r, s)
    assert np.array_equal(grid, G[f"inst_{n}_{r}_{s}"])
    g = orc.preprocess(grid)
    want = np.concatenate([[g.nv, g.l], g.cell_row, g.cell_col, g.adj_off, g.adj, g.dom_off,
                           g.dom.astype(np.int32)]).astype(np.int32)
    assert np.array_equal(want, G[f"graph_{n}_{r}_{s}"])


def test_lsc_instance(orc):
    assert np.array_equal(orc.lsc_instance(20, 0.4, 7), G["lsc_20_0.4_7"])
    assert np.array_equal(orc.lsc_instance(70, 0.4, 7), G["lsc_70_0.4_7"])


@pytest.mark.parametrize("n,r,s", [(10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345)])
def test_repair_and_gamma(orc, n, r, s):
    grid = G[f"inst_{n}_{r}_{s}"]
    cols = G[f"repair_in_{n}"]
    for c, want in zip(cols, G[f"repair_out_{n}"]):
        got = orc.repair(grid, c)
        assert np.array_equal(got, want)
        assert orc.eval(grid, got)[1] == 0
        assert np.array_equal(orc.repair(grid, got), got)  # idempotent (test_partial.cpp:42)
    assert np.array_equal(orc.gamma(grid, cols[0]), G[f"gamma_{n}"])


@pytest.mark.parametrize("n,r,s", [(10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (60, 0.5, 12345)])
def test_improve_ref_policy_trajectories(orc, n, r, s):
    grid = G[f"inst_{n}_{r}_{s}"]
    mem = G[f"improve_in_{n}"]
    nv = mem.shape[1]
    for i, row in enumerate(G[f"improve_out_{n}"]):
        o = orc.improve(grid, mem[i], 1000 + i, 100 * nv if n <= 30 else 20000, tie=oracle.TIE_REF)
        assert o["iterations"] == row[0]
        assert o["best_f"] == row[1]
        assert np.array_equal(o["best"], row[2:].astype(np.uint16))


@pytest.mark.parametrize("n,r,s", [(10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (60, 0.5, 12345)])
def test_per_step_states_ref_policy(orc, n, r, s):
    """replay the reference's per-step current colouring from the oracle's REF trace"""
    grid = G[f"inst_{n}_{r}_{s}"]
    mem = G[f"improve_in_{n}"]
    states, bf = G[f"states_{n}"], G[f"states_bf_{n}"]
    o = orc.improve(grid, mem[0], 4242, len(states), tie=oracle.TIE_REF, trace_cap=len(states))
    cur = G[f"states_rep_{n}"].astype(np.int32).copy()
    assert np.array_equal(orc.repair(grid, mem[0]), G[f"states_rep_{n}"])
    for t, st in enumerate(o["trace"]):
        if st["v"] >= 0:
            cur[st["v"]] = st["k"]
            for u in (st["ev0"], st["ev1"]):
                if u >= 0:
                    cur[u] = 0
        assert np.array_equal(cur, states[t].astype(np.int32)), t
        assert st["best_f"] == bf[t]


def test_population_chain(orc):
    grid = G["inst_20_0.7_505"]
    p = 16
    mem = orc.init_population(grid, p, 55)
    assert np.array_equal(mem, G["chain_init_members"])
    dist = orc.full_distances(mem)
    assert np.array_equal(dist, G["chain_init_dist"])
    nv = mem.shape[1]
    imp = np.stack([orc.improve(grid, mem[i], orc.derive_seed(55, 2, p + i), 100 * nv, tie=oracle.TIE_REF)["best"]
                    for i in range(p)])
    assert np.array_equal(imp, G["chain_improved"])
    cr, fr = orc.cross_distances(mem, imp)
    assert np.array_equal(cr, G["chain_cross"]) and np.array_equal(fr, G["chain_fresh"])
    u = orc.update(grid, mem, dist, imp, cr, fr)
    assert np.array_equal(u["members"], G["chain_members1"]) and np.array_equal(u["dist"], G["chain_dist1"])
    assert [u["pool_best_f"]] + u["shortfall_slots"] == G["chain_info1"].tolist()
    excl = np.zeros((p, p), np.uint8)
    off, _ = orc.offspring(grid, u["members"], u["dist"], excl, 55, 1)
    assert np.array_equal(off, G["chain_offspring1"])


def test_full_runs(orc):
    for row in G["runs"]:
        n, pp, bf, bs, po, sr, gens, its = [int(x) for x in row]
        o = orc.run(G[f"run_inst_{n}"], p=pp, seed=7, generation_limit=5, tie=oracle.TIE_REF)
        assert (o["best_f"], o["best_score"], o["proven_optimal"], oracle.STOP_NAMES.index(o["stop_reason"]),
                o["generations"], o["total_iterations"]) == (bf, bs, po, sr, gens, its)
        assert np.array_equal(o["best_colors"], G[f"run_best_{n}"])
