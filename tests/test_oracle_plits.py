"""The PLITS restatement (oracle/plse_oracle.c or_plits, plits.hpp:96-292) pinned to
the reference, and its canonical tie-break pinned to its own specification.

* OR_TIE_REF == plits_run of the compiled reference, colouring and iteration count,
  on random instances, colourings, seeds and budgets (plus golden vectors);
* OR_TIE_REF per-step trace == PlitsSearch::step(&applied) driven through both phases;
* OR_TIE_CANON replayed in Python: every step takes the r-th admissible minimum-delta
  candidate in ascending (v, k) order, r = floor(hi32 * N / 2^32), tenure
  floor(lo32 * 10 / 2^32) + floor(alpha * active), tabu honoured except through
  aspiration (test_plits.cpp:60-109 restated for the canonical rule);
* the MPMA run (engine.hpp:193-197) of the oracle == the reference's run().
"""
import os

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "ref_golden.npz"))


def _random_full(gr, rng):
    return np.array([gr.dom[gr.dom_off[v] + 1 + rng.integers(0, gr.dom_off[v + 1] - gr.dom_off[v] - 1)]
                     for v in range(gr.nv)], np.uint16)


def _random_partial(gr, rng):
    return np.array([gr.dom[gr.dom_off[v] + rng.integers(0, gr.dom_off[v + 1] - gr.dom_off[v])]
                     for v in range(gr.nv)], np.uint16)


def test_plits_golden(orc):
    for key in [k for k in G.files if k.startswith("plits_in_")]:
        tag = key[len("plits_in_"):]
        grid = G[f"plits_grid_{tag}"]
        seed, i1, i2, stop, its = (int(x) for x in G[f"plits_meta_{tag}"])
        o = orc.plits(grid, G[key], seed, i1, i2, 0.6, stop, tie=oracle.TIE_REF)
        assert np.array_equal(o["best"], G[f"plits_out_{tag}"]) and o["iterations"] == its, tag


def test_plits_ref_matches_reference(orc, ref):
    rng = np.random.default_rng(96)
    for t in range(80):
        n = int(rng.integers(3, 18))
        g = ref.generate_instance(n, float(rng.uniform(0.15, 0.85)), int(rng.integers(0, 2**40)))
        gr = ref.preprocess(g)
        if gr.nv == 0:
            continue
        cols = _random_full(gr, rng) if t % 3 else _random_partial(gr, rng)
        seed = int(rng.integers(0, 2**63))
        i1 = [0, 50, int(rng.integers(1, 4000))][t % 3]
        i2 = [0, 3, int(rng.integers(1, 300))][(t // 3) % 3]
        stop = 1 if gr.l == 1 else 0
        alpha = [0.6, 0.0, 1.5][t % 3]
        a = orc.plits(g, cols, seed, i1, i2, alpha, stop, tie=oracle.TIE_REF)
        b, it = ref.plits(g, cols, seed, i1, i2, alpha, stop)
        assert np.array_equal(a["best"], b), t
        assert a["iterations"] == it, t
        f, c = orc.eval(g, a["best"])
        assert c == 0 and f == a["final_f"]


def test_plits_ref_trace_matches_reference(orc, ref):
    rng = np.random.default_rng(97)
    for t in range(12):
        n = int(rng.integers(5, 14))
        g = ref.generate_instance(n, float(rng.uniform(0.2, 0.7)), int(rng.integers(0, 2**40)))
        gr = ref.preprocess(g)
        if gr.nv == 0:
            continue
        cols = _random_full(gr, rng)
        seed = int(rng.integers(0, 2**63))
        i1, i2 = int(rng.integers(50, 1500)), int(rng.integers(5, 80))
        o = orc.plits(g, cols, seed, i1, i2, 0.6, 0, tie=oracle.TIE_REF, trace_cap=5000)
        rec, bs, out, n_steps = ref.plits_trace(g, cols, seed, i1, i2, 0.6, 0, cap=5000)
        assert n_steps == o["iterations"]
        for q, e in enumerate(o["trace"]):
            assert (e["phase"], e["v"], e["k"] if e["v"] >= 0 else 0) == tuple(rec[q, :3]), (t, q)
            if e["v"] >= 0:
                assert (e["df"], e["dc"]) == tuple(rec[q, 3:5])
            assert (e["f"], e["c"]) == tuple(rec[q, 5:7]), (t, q)
            assert e["best_scaled"] == bs[q], (t, q)
        assert np.array_equal(o["best"], out)


def _canon_replay(orc, g, cols, seed, i1, i2, alpha, stop):
    """Python restatement of the canonical PLITS rule, checked against or_plits' trace."""
    gr = orc.preprocess(g)
    nv, n = gr.nv, g.shape[0]
    o = orc.plits(g, cols, seed, i1, i2, alpha, stop, tie=oracle.TIE_CANON, trace_cap=100000)
    tr = o["trace"]
    adj = [gr.adj[gr.adj_off[v]:gr.adj_off[v + 1]] for v in range(nv)]
    dom = [gr.dom[gr.dom_off[v]:gr.dom_off[v + 1]] for v in range(nv)]
    col = np.array(cols, np.int64)
    J = 0
    for phase, (wf, wc, budget) in enumerate([(2, 1, i1 or 100 * nv), (2, 2 * nv, i2 or 2 * nv)], start=1):
        until = {}
        gam = np.zeros((nv, n + 1), np.int64)
        for v in range(nv):
            if col[v]:
                for u in adj[v]:
                    gam[u, col[v]] += 1
        f = int((col == 0).sum())
        c = int(sum(gam[v, col[v]] for v in range(nv) if col[v])) // 2
        best, bf, bc, bs = col.copy(), f, c, wf * f + wc * c
        hit = False
        for j in range(budget):
            if bc == 0 and bf <= stop:
                hit = True
                break
            cands = []
            cur_s = wf * f + wc * c
            for v in range(nv):
                cur = col[v]
                if cur and gam[v, cur] == 0:
                    continue
                for k in dom[v]:
                    if k == cur:
                        continue
                    k, cur = int(k), int(cur)
                    df = int(k == 0) - int(cur == 0)
                    dc = (gam[v, k] if k else 0) - (gam[v, cur] if cur else 0)
                    d = wf * df + wc * dc
                    if until.get((v, k), 0) > j and cur_s + d >= bs:
                        continue
                    cands.append((d, v, int(k)))
            if not cands and all(col[v] and gam[v, col[v]] == 0 for v in range(nv)):
                break  # exhausted
            e = tr[J]
            assert e["phase"] == phase and e["step"] == J
            if not cands:
                assert e["v"] == -1
            else:
                dmin = min(x[0] for x in cands)
                at = [x for x in cands if x[0] == dmin]
                x = orc.canon_draw(seed, J)
                r = ((x >> 32) * len(at)) >> 32
                _, v, k = at[r]
                assert (e["v"], e["k"], e["delta"], e["n_adm"]) == (v, k, dmin, len(at)), (phase, j)
                frm = col[v]
                for u in adj[v]:
                    if frm:
                        gam[u, frm] -= 1
                    if k:
                        gam[u, k] += 1
                col[v] = k
                f = int((col == 0).sum())
                c = int(sum(gam[q, col[q]] for q in range(nv) if col[q])) // 2
                active = int(sum(1 for q in range(nv) if col[q] == 0 or gam[q, col[q]] > 0))
                ten = (((x & 0xFFFFFFFF) * 10) >> 32) + int(alpha * active)
                assert e["tenure"] == ten and e["active"] == active
                until[(v, int(frm))] = j + 1 + ten
                if wf * f + wc * c < bs:
                    bs, best, bf, bc = wf * f + wc * c, col.copy(), f, c
            assert (e["f"], e["c"], e["best_scaled"]) == (f, c, bs)
            J += 1
        if bc == 0 and bf <= stop:
            hit = True
        col = best
        if hit:
            break
    assert J == o["iterations"]
    return o


def test_plits_canon_replay(orc):
    rng = np.random.default_rng(98)
    done = 0
    for t in range(30):
        n = int(rng.integers(4, 9))
        g = orc.generate_instance(n, float(rng.uniform(0.2, 0.7)), int(rng.integers(0, 2**40)))
        gr = orc.preprocess(g)
        if gr.nv == 0:
            continue
        cols = _random_full(gr, rng) if t % 2 else _random_partial(gr, rng)
        o = _canon_replay(orc, g, cols, int(rng.integers(0, 2**63)), int(rng.integers(20, 400)),
                          int(rng.integers(2, 40)), [0.6, 0.3][t % 2], 1 if gr.l == 1 else 0)
        f, c = orc.eval(g, o["best"])
        assert c == 0 and f == o["final_f"]
        done += 1
    assert done > 15


def test_plits_canon_reaches_exact_optima(orc):
    """test_plits.cpp:213-235 for the canonical rule: the suite's exact optima within 50 restarts."""
    suite = G["suite"]
    for i in range(0, 60, 5):
        grid = G[f"suite_{i}"]
        gr = orc.preprocess(grid)
        if gr.nv == 0:
            continue
        opt_f = int(suite[i][2])
        rng = np.random.default_rng(i)
        best = gr.nv
        for restart in range(50):
            o = orc.plits(grid, _random_full(gr, rng), int(rng.integers(0, 2**63)), 0, 0, 0.6, opt_f,
                          tie=oracle.TIE_CANON)
            best = min(best, o["final_f"])
            if best <= opt_f:
                break
        assert best == opt_f, i


def test_mpma_run_matches_reference(orc, ref):
    for n, r, s, p in [(10, 0.5, 3, 8), (20, 0.6, 9, 12), (30, 0.5, 4, 16), (14, 0.4, 21, 6)]:
        g = ref.generate_instance(n, r, s)
        a = orc.run(g, p=p, seed=s, generation_limit=4, phase1_iters=400, tie=oracle.TIE_REF, variant=0, log_cap=8)
        b = ref.run(g, p=p, seed=s, generation_limit=4, phase1_iters=400, variant=0, workers=2, log_cap=8)
        for k in ("best_f", "best_score", "stop_reason", "generations", "total_iterations"):
            assert a[k] == b[k], (n, k)
        assert np.array_equal(a["best_colors"], b["best_colors"])
        assert a["log"] == b["log"]


def test_mpma_run_golden(orc):
    if "mpma_runs" not in G.files:
        pytest.skip("golden fixture absent")
    for row in G["mpma_runs"]:
        n, p, seed, bf, its, gens = (int(x) for x in row)
        o = orc.run(G[f"mpma_inst_{n}"], p=p, seed=seed, generation_limit=4, phase1_iters=400,
                    tie=oracle.TIE_REF, variant=0)
        assert (o["best_f"], o["total_iterations"], o["generations"]) == (bf, its, gens)
        assert np.array_equal(o["best_colors"], G[f"mpma_best_{n}"])
