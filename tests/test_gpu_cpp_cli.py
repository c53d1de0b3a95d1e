"""The C++ front-end (tools/plse_b200.cpp over include/plse_b200.hpp; `python -m paper_2103_10453_b200` is a
thin wrapper over it) on the GPU: with the reference tie-break its `solve` output is the reference CLI's byte
for byte; its `bench` rows equal the Python bench-report library's (suite.run_bench over run()); `solve --log`
streams GenerationStats."""
import csv
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2103_10453_b200", "plse_b200")


def _run(*args):
    return subprocess.run([str(a) for a in args], capture_output=True, text=True, timeout=900, cwd=ROOT)


def test_cpp_solve_ref_ties_equals_reference(plse, orc, ref, tmp_path):
    if not ref.has_result_json():
        pytest.skip("nlohmann/json not found when oracle/_ref was built")
    grid = orc.generate_instance(12, 0.6, 88)
    inst = tmp_path / "instance.txt"
    inst.write_text(plse.serialize_instance(grid))
    out = _run(CLI, "solve", inst, "--seed", 31337, "--pop", 16, "--gen-limit", 5, "--workers", 2, "--variant",
               "partial", "--tie", "ref", "--cert", tmp_path / "c.txt")
    assert out.returncode in (0, 2), out.stderr
    r = ref.run(grid, p=16, seed=31337, generation_limit=5, workers=2)
    want = ref.result_json("instance.txt", 12, r, r["stop_reason"], 16, 0.6, 10.0, 20.0, 0, 0, 1, 0, 0, 0, 31337, 2,
                           0.0, 0, 5)
    assert out.stdout == want + "\n"
    cert = plse.parse_instance((tmp_path / "c.txt").read_text())
    assert np.array_equal(cert, ref.to_grid(grid, r["best_colors"]))
    assert out.stderr.startswith(f"score {r['best_score']}/{r['upper_bound']}")


def test_cpp_solve_log_and_mpma(plse, orc, tmp_path):
    grid = orc.generate_instance(20, 0.6, 9)
    inst = tmp_path / "i.txt"
    inst.write_text(plse.serialize_instance(grid))
    out = _run(CLI, "solve", inst, "--seed", 9, "--pop", 12, "--gen-limit", 3, "--phase1-iters", 400, "--log")
    assert out.returncode in (0, 2), out.stderr
    o = orc.run(grid, p=12, seed=9, generation_limit=3, phase1_iters=400, tie=oracle.TIE_CANON, variant=0,
                log_cap=8)
    logs = [l for l in out.stderr.split("\n") if l.startswith("gen ")]
    assert len(logs) == len(o["log"])
    for line, e in zip(logs, o["log"]):
        t = line.split()
        assert (int(t[1]), int(t[3]), int(t[9])) == (e["generation"], e["best_f"], e["iterations"])


def test_cpp_bench_equals_python_bench(plse, tmp_path):
    suite = tmp_path / "suite"
    assert _run(CLI, "generate", "-n", 8, "-r", 0.5, "-c", 2, "-o", suite, "--seed", 9).returncode == 0
    flags = ["--repeats", "2", "--pop", "8", "--gen-limit", "3", "--phase1-iters", "300", "--variant", "partial",
             "--seed", "4", "--sweep-crossover", "aux", "ux"]
    a = _run(CLI, "bench", suite, *flags, "--csv", tmp_path / "a.csv", "--json", tmp_path / "a.json")
    assert a.returncode == 0, a.stderr
    # the same sweep through the Python library: plse.cpp:199-250's loop over suite.run_bench
    import dataclasses
    import io
    from paper_2103_10453_b200 import report as R
    from paper_2103_10453_b200 import suite as S
    base = plse.SolverConfig(p=8, generation_limit=3, phase1_iters=300, variant=plse.PARTIAL, master_seed=4)
    sweep = [dataclasses.replace(base, crossover=R.parse_crossover(c)) for c in ("aux", "ux")]
    rep = S.run_bench(S.suite_tasks(str(suite)), sweep, 2, 4, 1, io.StringIO())
    with open(tmp_path / "b.csv", "w") as fh:
        S.write_rows_csv(rep, fh)
    ra, rb = (list(csv.DictReader(open(tmp_path / f"{x}.csv"))) for x in "ab")
    assert len(ra) == len(rb) == 8
    for x, y in zip(ra, rb):
        assert {k: v for k, v in x.items() if k != "elapsed_seconds"} == \
               {k: v for k, v in y.items() if k != "elapsed_seconds"}


def test_cpp_solve_default_variant_ref_ties_equals_reference(plse, orc, ref, tmp_path):
    """The reference CLI's defaults (variant mpma, p = 1024 scaled down here) with --tie ref: same JSON."""
    if not ref.has_result_json():
        pytest.skip("nlohmann/json not found when oracle/_ref was built")
    grid = orc.generate_instance(12, 0.6, 88)
    inst = tmp_path / "instance.txt"
    inst.write_text(plse.serialize_instance(grid))
    out = _run(CLI, "solve", inst, "--seed", 31337, "--pop", 16, "--gen-limit", 5, "--workers", 2, "--tie", "ref")
    assert out.returncode in (0, 2), out.stderr
    r = ref.run(grid, p=16, seed=31337, generation_limit=5, workers=2, variant=0)
    want = ref.result_json("instance.txt", 12, r, r["stop_reason"], 16, 0.6, 10.0, 20.0, 0, 0, 0, 0, 0, 0, 31337, 2,
                           0.0, 0, 5)
    assert out.stdout == want + "\n"
