"""Generate tests/golden/ref_golden.npz from the REAL reference.

Runs the unmodified reference headers compiled in place (oracle/_ref, built by
oracle/Makefile from /root/reference) and records input/output vectors for the
hot path, so that the C oracle stays pinned where /root/reference does not
exist (the GPU box, the driver's CPU check).  Re-run with:

    make -C oracle && python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    R = oracle.Reference()
    out = {}
    # --- instances (instance.hpp:204) and the LSC builder (builders.hpp:46)
    inst = [(5, 0.5, 61), (10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (60, 0.5, 12345), (70, 0.6, 12345),
            (50, 0.4, 12345), (4, 0.2, 7), (6, 0.8, 3)]
    for n, r, s in inst:
        g = R.generate_instance(n, r, s)
        out[f"inst_{n}_{r}_{s}"] = g
        gr = R.preprocess(g)
        out[f"graph_{n}_{r}_{s}"] = np.concatenate([[gr.nv, gr.l], gr.cell_row, gr.cell_col, gr.adj_off, gr.adj,
                                                    gr.dom_off, gr.dom.astype(np.int32)]).astype(np.int32)
    out["lsc_20_0.4_7"] = R.lsc_instance(20, 0.4, 7)
    out["lsc_70_0.4_7"] = R.lsc_instance(70, 0.4, 7)

    # --- repair (partial.hpp:22) and gamma (coloring.hpp:105) on random colourings
    rng = np.random.default_rng(404)
    for n, r, s in [(10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345)]:
        g = out[f"inst_{n}_{r}_{s}"]
        gr = R.preprocess(g)
        cols = []
        for t in range(8):
            c = np.array([gr.dom[rng.integers(gr.dom_off[v], gr.dom_off[v + 1])] for v in range(gr.nv)], np.uint16)
            cols.append(c)
        cols = np.stack(cols)
        out[f"repair_in_{n}"] = cols
        out[f"repair_out_{n}"] = np.stack([R.repair(g, c) for c in cols])
        out[f"gamma_{n}"] = R.gamma(g, cols[0])

    # --- partial_mpma_improve trajectories (REF tie-break) and per-step states
    for n, r, s in [(10, 0.3, 606), (20, 0.7, 505), (30, 0.5, 12345), (60, 0.5, 12345)]:
        g = out[f"inst_{n}_{r}_{s}"]
        mem, _ = R.init_population(g, 4, 77)
        nv = mem.shape[1]
        res = []
        for i in range(4):
            seed = 1000 + i
            o = R.improve(g, mem[i], seed, 100 * nv if n <= 30 else 20000)
            res.append(np.concatenate([[o["iterations"], o["best_f"]], o["best"]]).astype(np.int64))
        out[f"improve_in_{n}"] = mem
        out[f"improve_out_{n}"] = np.stack(res)
        rep, states, bf = R.improve_states(g, mem[0], 4242, 300)
        out[f"states_rep_{n}"] = rep
        out[f"states_{n}"] = states
        out[f"states_bf_{n}"] = bf

    # --- one population generation chain (init -> improve -> distances -> update -> offspring)
    g = out["inst_20_0.7_505"]
    p = 16
    mem, dist = R.init_population(g, p, 55)
    out["chain_init_members"] = mem
    out["chain_init_dist"] = dist
    nv = mem.shape[1]
    imp = np.stack([R.improve(g, mem[i], oracle.Oracle().derive_seed(55, 2, p + i), 100 * nv)["best"]
                    for i in range(p)])
    out["chain_improved"] = imp
    cr, fr = R.cross_distances(g, mem, imp)
    out["chain_cross"] = cr
    out["chain_fresh"] = fr
    u = R.update(g, mem, dist, imp, cr, fr)
    out["chain_members1"] = u["members"]
    out["chain_dist1"] = u["dist"]
    out["chain_info1"] = np.array([u["pool_best_f"]] + u["shortfall_slots"], np.int32)
    ex = R.new_exclusion(p)
    out["chain_offspring1"] = R.offspring(g, u["members"], u["dist"], ex, 55, 1)

    # --- full runs (engine.hpp:114), workers=1, Partial-MPMA
    runs = []
    for n, r, s, pp in [(10, 0.5, 3, 16), (20, 0.7, 505, 16), (30, 0.5, 12345, 16)]:
        gg = R.generate_instance(n, r, s)
        out[f"run_inst_{n}"] = gg
        rr = R.run(gg, p=pp, seed=7, generation_limit=5, workers=1)
        runs.append([n, pp, rr["best_f"], rr["best_score"], rr["proven_optimal"], ["optimal", "time_limit",
                     "iteration_limit", "generation_limit", "trivial"].index(rr["stop_reason"]), rr["generations"],
                     rr["total_iterations"]])
        out[f"run_best_{n}"] = rr["best_colors"]
    out["runs"] = np.array(runs, np.int64)

    # --- acceptance c1/c9 small suite (acceptance.cpp:49-60) with exact optima (oracle.hpp:134)
    O = oracle.Oracle()
    suite = []
    for i in range(200):
        n = 4 + (i % 3)
        r = 0.3 + 0.1 * ((i // 3) % 6)
        seed = O.derive_seed(20240801, 1000, i)
        gg = R.generate_instance(n, r, seed)
        f, exact = R.solve_exact(gg)
        assert exact
        gr = R.preprocess(gg)
        suite.append([n, seed & 0xFFFFFFFFFFFF, f, n * n - gr.l - f, gr.l])
        out[f"suite_{i}"] = gg
    out["suite"] = np.array(suite, np.int64)

    # --- per-generation GenerationStats of a run (engine.hpp:214-233)
    gg = out["run_inst_20"]
    rr = R.run(gg, p=16, seed=7, generation_limit=5, workers=1, log_cap=8)
    out["run_log_20"] = np.array([[e["generation"], e["best_f"], e["shortfall"], e["iterations"]]
                                  for e in rr["log"]], np.int64)
    out["run_log_20_means"] = np.array([[e["mean_f"], e["mean_distance"]] for e in rr["log"]], np.float64)

    # --- certificates (coloring.hpp:171) and verify_certificate (verify.hpp:20)
    rng = np.random.default_rng(171)
    for n, r, s in [(10, 0.3, 606), (20, 0.7, 505)]:
        g = out[f"inst_{n}_{r}_{s}"]
        gr = R.preprocess(g)
        cols = np.zeros(gr.nv, np.uint16)
        for v in range(gr.nv):
            d = gr.dom[gr.dom_off[v]:gr.dom_off[v + 1]]
            cols[v] = d[rng.integers(0, len(d))]
        cert = R.to_grid(g, cols)
        out[f"cert_colors_{n}"] = cols
        out[f"cert_grid_{n}"] = cert
        for t, bad in enumerate([cert, g]):
            legal, score, probs = R.verify_certificate(g, bad)
            out[f"verify_{n}_{t}"] = np.frombuffer(("\n".join(probs)).encode() or b"\0", np.uint8)
            out[f"verify_{n}_{t}_ls"] = np.array([legal, score], np.int64)
        alt = cert.copy()
        alt[np.nonzero(g)[0][0], np.nonzero(g)[1][0]] = 0
        legal, score, probs = R.verify_certificate(g, alt)
        out[f"verify_{n}_alt"] = np.frombuffer(("\n".join(probs)).encode(), np.uint8)
        out[f"verify_{n}_alt_ls"] = np.array([legal, score], np.int64)

    # --- result_to_json(...).dump(2) (report.hpp:85, plse.cpp:154)
    if R.has_result_json():
        res = dict(best_f=3, best_score=80, proven_optimal=0, l=2, upper_bound=83, vertex_count=50, generations=5,
                   total_iterations=12345, elapsed_seconds=1.25)
        out["json_a"] = np.frombuffer(R.result_json("instance.txt", 12, res, "generation_limit", 16, 0.6, 10.0, 20.0,
                                                    0, 0, 0, 0, 0, 0, 31337, 2, 0.0, 0, 5).encode(), np.uint8)
        out["json_b"] = np.frombuffer(R.result_json("QC-60-50-0.txt", 60, res, "time_limit", 12288, 0.35, 12.5,
                                                    25.0, 1000, 7, 1, 1, 1, 2, 2**64 - 1, 144, 1e-3, 10**12, 0,
                                                    True).encode(), np.uint8)

    # --- PLITS (plits.hpp:276) and the MPMA run (engine.hpp:193-197)
    rng = np.random.default_rng(276)
    for tag, (n, r, s) in enumerate([(8, 0.4, 17), (12, 0.5, 606), (20, 0.6, 505), (9, 0.3, 3)]):
        g = R.generate_instance(n, r, s)
        gr = R.preprocess(g)
        cols = np.array([gr.dom[gr.dom_off[v] + 1 + rng.integers(0, gr.dom_off[v + 1] - gr.dom_off[v] - 1)]
                         for v in range(gr.nv)], np.uint16)
        seed = int(rng.integers(0, 2**62))
        i1, i2 = [(0, 0), (300, 10), (2000, 0), (50, 5)][tag]
        stop = 1 if gr.l == 1 else 0
        res, its = R.plits(g, cols, seed, i1, i2, 0.6, stop)
        out[f"plits_grid_{tag}"] = g
        out[f"plits_in_{tag}"] = cols
        out[f"plits_out_{tag}"] = res
        out[f"plits_meta_{tag}"] = np.array([seed, i1, i2, stop, its], np.int64)
    mruns = []
    for n, r, s, pp in [(10, 0.5, 3, 8), (20, 0.6, 9, 12)]:
        g = R.generate_instance(n, r, s)
        rr = R.run(g, p=pp, seed=s, generation_limit=4, phase1_iters=400, variant=0, workers=1)
        out[f"mpma_inst_{n}"] = g
        out[f"mpma_best_{n}"] = rr["best_colors"]
        mruns.append([n, pp, s, rr["best_f"], rr["total_iterations"], rr["generations"]])
    out["mpma_runs"] = np.array(mruns, np.int64)
    path = os.path.join(HERE, "ref_golden.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
