"""§8(f) rank 2 on the CPU: the result API around the device solver.

* ``report.result_to_json`` + ``report.dumps`` == report.hpp:85 ``result_to_json(...).dump(2)``
  byte for byte (golden text and the compiled reference);
* ``to_grid`` == coloring.hpp:171 and ``verify_certificate`` == verify.hpp:20 (same problems,
  same order, same wording);
* ``derive_seed`` == rng.hpp:81 and the ``generate`` subcommand writes the files plse.cpp:111
  writes;
* the oracle's per-generation statistics (mean f, mean distance) == the reference's
  GenerationStats, so the GPU test of the same numbers is pinned.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "ref_golden.npz"))


def _text(key):
    return bytes(G[key]).decode().rstrip("\0")


def test_derive_seed_matches_oracle(plse, orc):
    for m, t, i in [(0, 0, 0), (88, 4, 0), (88, 4, 7), (2**64 - 1, 2, 10**12), (12345, 1, 3)]:
        assert plse.derive_seed(m, t, i) == orc.derive_seed(m, t, i)


def _result(plse, **kw):
    base = dict(best_f=3, best_score=80, proven_optimal=False, stop_reason="generation_limit", l=2,
                upper_bound=83, vertex_count=50, generations=5, total_iterations=12345, elapsed_seconds=1.25,
                time_to_best_seconds=0.0, best_solution=None)
    base.update(kw)
    return plse.RunResult(**base)


def test_result_json_golden(plse):
    from paper_2103_10453_b200 import report as R
    a = R.result_to_json("instance.txt", 12, _result(plse),
                         plse.SolverConfig(p=16, master_seed=31337, workers=2, generation_limit=5, variant=plse.MPMA))
    assert R.dumps(a) == _text("json_a")
    cfg = plse.SolverConfig(p=12288, alpha=0.35, gamma=12.5, beta=25.0, phase1_iters=1000, phase2_iters=7,
                            variant=plse.PARTIAL, crossover=plse.UX, matching=plse.RANDOM, exclusion=plse.OFF,
                            master_seed=2**64 - 1, workers=144, time_limit=1e-3, iteration_limit=10**12)
    b = R.result_to_json("QC-60-50-0.txt", 60, _result(plse, stop_reason="time_limit"), cfg, include_timing=True)
    assert R.dumps(b) == _text("json_b")
    assert list(b) == ["instance", "n", "vertices", "l", "upper_bound", "best_score", "f", "proven_optimal",
                       "stop_reason", "generations", "total_iterations", "elapsed_seconds", "config"]


@pytest.mark.parametrize("case", range(8))
def test_result_json_matches_reference_bytes(plse, ref, case):
    from paper_2103_10453_b200 import report as R
    if not ref.has_result_json():
        pytest.skip("nlohmann/json not found when oracle/_ref was built")
    rng = np.random.default_rng(case)
    alpha = [0.6, 0.1, 1 / 3, 2.5e20, 1e-7, 0.0, 1e15, 100000.0][case]
    tl = [0.0, 1e-7, 123456789.125, 1e300, 0.1 + 0.2, 7.0, 1234567890123456.0, 0.00001][case]
    seed = int(rng.integers(0, 2**63)) * (1 + case % 2)
    timing = case % 2 == 1
    fields = dict(best_f=int(rng.integers(0, 99)), best_score=int(rng.integers(0, 9999)), proven_optimal=case % 3 == 0,
                  l=int(rng.integers(0, 5)), upper_bound=int(rng.integers(0, 9999)), vertex_count=int(rng.integers(0, 5000)),
                  generations=int(rng.integers(0, 10**6)), total_iterations=int(rng.integers(0, 2**62)),
                  elapsed_seconds=float(rng.random() * 100))
    stop = ["optimal", "time_limit", "iteration_limit", "generation_limit", "trivial", "optimal", "time_limit",
            "optimal"][case]
    cfg = plse.SolverConfig(p=int(rng.integers(2, 20000)), alpha=alpha, gamma=10.0 + case, beta=20.0 + 0.5 * case,
                            phase1_iters=case * 1000, phase2_iters=case, variant=case % 2,
                            crossover=case % 3, matching=case % 2, exclusion=(case + 1) % 3, master_seed=seed,
                            workers=1 + case, time_limit=tl, iteration_limit=case * 10**9,
                            generation_limit=case * 7)
    ours = R.dumps(R.result_to_json(f"inst-{case}.txt", 5 + case, _result(plse, stop_reason=stop, **fields), cfg,
                                    timing))
    theirs = ref.result_json(f"inst-{case}.txt", 5 + case, dict(fields, proven_optimal=int(fields["proven_optimal"])),
                             stop, cfg.p, cfg.alpha, cfg.gamma, cfg.beta, cfg.phase1_iters, cfg.phase2_iters,
                             cfg.variant, cfg.crossover, cfg.matching, cfg.exclusion, cfg.master_seed, cfg.workers,
                             cfg.time_limit, cfg.iteration_limit, cfg.generation_limit, timing)
    assert ours == theirs


def test_to_grid_golden(plse):
    for n, r, s in [(10, 0.3, 606), (20, 0.7, 505)]:
        g = G[f"inst_{n}_{r}_{s}"]
        graph = plse.preprocess(g)
        assert np.array_equal(plse.to_grid(g, graph, G[f"cert_colors_{n}"]), G[f"cert_grid_{n}"])


def test_to_grid_rejects_colours_outside_the_domain(plse):
    g = G["inst_10_0.3_606"]
    graph = plse.preprocess(g)
    cols = np.zeros(graph.vertex_count, np.uint16)
    v = 0
    dom = set(graph.dom[graph.dom_offsets[v]:graph.dom_offsets[v + 1]].tolist())
    cols[v] = next(k for k in range(1, 11) if k not in dom)
    with pytest.raises(ValueError, match="domain"):
        plse.to_grid(g, graph, cols)
    with pytest.raises(ValueError):
        plse.to_grid(g, graph, cols[:-1])


def test_verify_certificate_golden(plse):
    for n, r, s in [(10, 0.3, 606), (20, 0.7, 505)]:
        g = G[f"inst_{n}_{r}_{s}"]
        cases = [(G[f"cert_grid_{n}"], f"verify_{n}_0"), (g, f"verify_{n}_1")]
        alt = G[f"cert_grid_{n}"].copy()
        rr, cc = np.nonzero(g)
        alt[rr[0], cc[0]] = 0
        cases.append((alt, f"verify_{n}_alt"))
        for cert, key in cases:
            rep = plse.verify_certificate(g, cert)
            legal, score = G[key + "_ls"]
            text = _text(key)
            assert rep.legal == bool(legal) and rep.score == score
            assert rep.problems == (text.split("\n") if text else [])


def test_verify_certificate_matches_reference(plse, ref):
    rng = np.random.default_rng(20)
    for t in range(60):
        n = int(rng.integers(2, 14))
        g = ref.generate_instance(n, float(rng.uniform(0.1, 0.9)), int(rng.integers(0, 2**40)))
        cert = g.copy()
        empty = np.argwhere(g == 0)
        for (a, b) in empty[rng.random(len(empty)) < 0.7]:
            cert[a, b] = rng.integers(1, n + 1)
        if t % 4 == 1:  # alter pre-filled cells
            filled = np.argwhere(g != 0)
            for (a, b) in filled[rng.random(len(filled)) < 0.2]:
                cert[a, b] = rng.integers(0, n + 1)
        if t % 10 == 9:  # order mismatch
            cert = np.zeros((n + 1, n + 1), np.uint16)
        rep = plse.verify_certificate(g, cert)
        legal, score, probs = ref.verify_certificate(g, cert)
        assert (rep.legal, rep.score, rep.problems) == (legal, score, probs)


def test_to_grid_matches_reference(plse, ref):
    rng = np.random.default_rng(21)
    for _ in range(20):
        n = int(rng.integers(2, 16))
        g = ref.generate_instance(n, float(rng.uniform(0.1, 0.9)), int(rng.integers(0, 2**40)))
        graph = plse.preprocess(g)
        cols = np.zeros(graph.vertex_count, np.uint16)
        for v in range(graph.vertex_count):
            d = graph.dom[graph.dom_offsets[v]:graph.dom_offsets[v + 1]]
            cols[v] = 0 if rng.random() < 0.2 else d[rng.integers(0, len(d))]
        assert np.array_equal(plse.to_grid(g, graph, cols), ref.to_grid(g, cols))


def _cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2103_10453_b200", *args], capture_output=True, text=True,
                          cwd=cwd or ROOT, timeout=600)


def test_cli_generate_matches_reference_streams(plse, orc, tmp_path):
    out = _cli("generate", "-n", "12", "-r", "0.6", "-c", "3", "-o", str(tmp_path), "--seed", "88")
    assert out.returncode == 0, out.stderr
    assert out.stderr.strip() == "seed 88"
    lines = out.stdout.strip().split("\n")
    for i in range(3):
        path = tmp_path / f"QC-12-60-{i}.txt"
        g = orc.generate_instance(12, 0.6, orc.derive_seed(88, 4, i))
        assert path.read_text() == plse.serialize_instance(g)
        assert lines[i] == f"{path} ({int((g != 0).sum())} filled)"


def test_cli_verify(plse, tmp_path):
    g = G["inst_20_0.7_505"]
    (tmp_path / "i.txt").write_text(plse.serialize_instance(g))
    alt = g.copy()
    rr, cc = np.nonzero(g)
    alt[rr[0], cc[0]] = 0
    alt[rr[1], cc[1]] = 0
    (tmp_path / "bad.txt").write_text(plse.serialize_instance(alt))
    (tmp_path / "dup.txt").write_text(plse.serialize_instance(G["cert_grid_20"]))
    out = _cli("verify", str(tmp_path / "i.txt"), str(tmp_path / "i.txt"))
    graph = plse.preprocess(g)
    ub = 400 - 2 if graph.l == 1 else 400 - graph.l
    assert out.returncode == 0
    assert out.stdout == f"legal, score {int((g != 0).sum())}\nupper bound {ub} (l = {graph.l})\n"
    out = _cli("verify", str(tmp_path / "i.txt"), str(tmp_path / "bad.txt"))
    assert out.returncode == 1
    probs = [f"pre-filled cell ({rr[t]},{cc[t]}) altered: expected {g[rr[t], cc[t]]}, got 0" for t in range(2)]
    assert out.stdout == "illegal certificate:\n" + "".join(f"  {p}\n" for p in probs)
    # a certificate that breaks the Latin condition already fails to parse (instance.hpp:145-166)
    out = _cli("verify", str(tmp_path / "i.txt"), str(tmp_path / "dup.txt"))
    assert out.returncode == 1 and out.stderr.startswith("error: line ") and "duplicate symbol" in out.stderr
    out = _cli("verify", str(tmp_path / "missing.txt"), str(tmp_path / "i.txt"))
    assert out.returncode == 1 and out.stderr.startswith("error: cannot open instance file")


def test_cli_rejects_bad_flags(tmp_path):
    (tmp_path / "i.txt").write_text("2\n0 0\n0 0\n")
    for flags, msg in [(["--variant", "x"], "unknown variant: x"), (["--crossover", "y"], "unknown crossover mode: y"),
                       (["--pop", "1"], "population size must be at least 2"),
                       (["--gamma", "30"], "beta must exceed gamma")]:
        out = _cli("solve", str(tmp_path / "i.txt"), "--seed", "1", *flags)
        assert out.returncode == 1 and out.stderr.strip() == f"error: {msg}", out.stderr


def test_generation_stats_golden(orc):
    """The oracle's GenerationStats (mean f / mean distance) vs the reference's, REF tie mode."""
    gg = G["run_inst_20"]
    o = orc.run(gg, p=16, seed=7, generation_limit=5, tie=oracle.TIE_REF, log_cap=8)
    got = np.array([[e["generation"], e["best_f"], e["shortfall"], e["iterations"]] for e in o["log"]], np.int64)
    assert np.array_equal(got, G["run_log_20"])
    means = np.array([[e["mean_f"], e["mean_distance"]] for e in o["log"]])
    assert np.array_equal(means, G["run_log_20_means"])


def test_generation_stats_match_reference(orc, ref):
    for n, r, s, p in [(10, 0.5, 3, 8), (20, 0.6, 9, 12)]:
        gg = ref.generate_instance(n, r, s)
        a = orc.run(gg, p=p, seed=s, generation_limit=4, phase1_iters=300, tie=oracle.TIE_REF, log_cap=8)
        b = ref.run(gg, p=p, seed=s, generation_limit=4, phase1_iters=300, log_cap=8)
        assert a["log"] == b["log"]


def _bench_rows_from_ref_json(js):
    from paper_2103_10453_b200 import suite as S
    import json as J
    d = J.loads(js)
    return [S.BenchRow(instance=r["instance"], n=r["n"], r_percent=r["r"], id=r["id"], repeat=r["repeat"],
                       seed=r["seed"], p=r["p"], crossover=r["crossover"], matching=r["matching"],
                       variant=r["variant"], score=r["score"], f=r["f"], upper_bound=r["upper_bound"],
                       proven_optimal=r["proven_optimal"], generations=r["generations"], iterations=r["iterations"],
                       elapsed_seconds=r["elapsed_seconds"]) for r in d["rows"]]


def test_bench_report_format_matches_reference(plse, ref, tmp_path):
    """bench.hpp: rows CSV, aggregates CSV and report JSON of the same rows, byte for byte; the
    kBench seed derivation and the QC-name parsing (bench.hpp:64-81, 228-233)."""
    import io
    from paper_2103_10453_b200 import report as R
    from paper_2103_10453_b200 import suite as S
    if not hasattr(ref.lib, "ref_bench"):
        pytest.skip("nlohmann/json not found when oracle/_ref was built")
    out = _cli("generate", "-n", "6", "-r", "0.45", "-c", "2", "-o", str(tmp_path), "--seed", "5")
    assert out.returncode == 0
    (tmp_path / "odd-name.txt").write_text(plse.serialize_instance(G["inst_6_0.8_3"]))
    (tmp_path / "QC-7-10-zz.txt").write_text(plse.serialize_instance(G["inst_6_0.8_3"]))  # n mismatch -> fallback
    rows_csv, agg_csv, js = ref.bench(str(tmp_path), 2, 77, 8, 2, phase1=200, crossovers="aux,ux",
                                      matchings="nearest", pops="8,6")
    rows = _bench_rows_from_ref_json(js)
    assert len(rows) == 4 * 2 * 2 * 2
    rep = S.BenchReport(rows=rows)
    S.compute_aggregates(rep)
    a, b = io.StringIO(), io.StringIO()
    S.write_rows_csv(rep, a)
    S.write_aggregates_csv(rep, b)
    assert a.getvalue() == rows_csv
    assert b.getvalue() == agg_csv
    assert R.dumps(S.report_to_json(rep)) == js
    tasks = S.suite_tasks(str(tmp_path))
    assert [t.stem for t in tasks] == sorted({r.instance for r in rows})
    k = 0
    for t in tasks:
        grid = plse.parse_instance(open(t.path).read())
        for sidx in range(4):
            for rep_i in range(2):
                row = rows[k]
                assert row.instance == t.stem and row.repeat == rep_i
                assert row.seed == plse.derive_seed(77, 5, (t.instance_index * 4 + sidx) * 2 + rep_i)
                assert (row.n, row.r_percent, row.id) == S.parse_instance_name(t.stem, grid)
                k += 1
