"""The C++ host API (include/plse_b200.hpp) and the C++ CLI (tools/plse_b200.cpp) on the CPU:
same answers as the Python front-end, the oracle and the compiled reference.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "ref_golden.npz"))
CLI = os.path.join(ROOT, "paper_2103_10453_b200", "plse_b200")


@pytest.fixture(scope="module")
def probe(tmp_path_factory, plse):
    out = str(tmp_path_factory.mktemp("cpp") / "probe")
    lib_dir = os.path.dirname(plse.lib_path())
    cmd = ["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "host_api_probe.cpp"), "-o", out, "-L" + lib_dir, "-lplse_b200",
           "-Wl,-rpath," + lib_dir]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def _run(*args):
    return subprocess.run([str(a) for a in args], capture_output=True, text=True, timeout=300)


def test_cpp_instance_and_seeds(probe, plse, orc):
    r = _run(probe, "instance", 8, 0.45, 77)
    lines = r.stdout.split("\n")
    g = plse.generate_instance(8, 0.45, 77)
    assert "\n".join(lines[:9]) + "\n" == plse.serialize_instance(g)
    assert lines[9] == "roundtrip ok"
    assert int(lines[10]) == orc.derive_seed(88, 4, 3)
    gr = plse.preprocess(g)
    ub = 64 - 2 if gr.l == 1 else 64 - gr.l
    assert lines[11] == f"{gr.vertex_count} {gr.l} {ub}"


def test_cpp_exact_matches_reference(probe, plse, ref, tmp_path):
    for i in range(0, 200, 13):
        grid = G[f"suite_{i}"]
        path = tmp_path / f"s{i}.txt"
        path.write_text(plse.serialize_instance(grid))
        for budget in (50_000_000, 50):
            out = _run(probe, "exact", path, budget).stdout.split("\n")
            f, ex, nodes = (int(x) for x in out[0].split())
            cert = np.array([int(x) for x in out[1].split()], np.uint16)
            want = ref.solve_exact_full(grid, budget)
            assert (f, bool(ex), nodes) == want[:3] and np.array_equal(cert, want[3]), (i, budget)
            legal, score, nprob = (int(x) for x in out[2].split())
            assert legal == 1 and nprob == 0 and score == grid.size - plse.preprocess(grid).l - f


def test_cpp_verify_problems_match_python(probe, plse, tmp_path):
    g = G["inst_20_0.7_505"]
    alt = g.copy()
    rr, cc = np.nonzero(g)
    alt[rr[0], cc[0]] = 0
    alt[rr[3], cc[3]] = 0
    (tmp_path / "i.txt").write_text(plse.serialize_instance(g))
    (tmp_path / "c.txt").write_text(plse.serialize_instance(alt))
    out = _run(probe, "verify", tmp_path / "i.txt", tmp_path / "c.txt").stdout.rstrip("\n").split("\n")
    rep = plse.verify_certificate(g, alt)
    assert out[0] == f"{int(rep.legal)} {rep.score}" and out[1:] == rep.problems


@pytest.mark.parametrize("case", range(6))
def test_cpp_result_json_matches_python_and_reference(probe, plse, ref, case):
    from paper_2103_10453_b200 import report as R
    opt = case % 2
    stop = ["optimal", "time_limit", "generation_limit", "iteration_limit", "trivial", "target"][case]
    elapsed = [1.25, 0.1 + 0.2, 1e-7, 123456.5, 100000.0, 1e15][case]
    p, alpha = [16, 12288, 2, 1024, 99, 7][case], [0.6, 1 / 3, 1e15, 0.0, 2.5e20, 100000.0][case]
    cross = ["aux", "ux", "none", "aux", "ux", "none"][case]
    seed = [31337, 2**64 - 1, 0, 12345, 7, 2**63][case]
    tl = [0.001, 0.0, 1e300, 7.0, 1234567890123456.0, 0.00001][case]
    variant = ["partial", "mpma"][case % 2]
    timing = case % 3 == 0
    cpp = _run(probe, "json", opt, stop, repr(elapsed), p, repr(alpha), cross, seed, repr(tl), variant,
               int(timing)).stdout
    res = plse.RunResult(best_f=3, best_score=80, proven_optimal=bool(opt), stop_reason=stop, l=2, upper_bound=83,
                         vertex_count=50, generations=5, total_iterations=12345, elapsed_seconds=elapsed,
                         time_to_best_seconds=0.0, best_solution=None)
    cfg = plse.SolverConfig(p=p, alpha=alpha, crossover=R.parse_crossover(cross), master_seed=seed, time_limit=tl,
                            variant=R.parse_variant(variant), workers=2)
    py = R.dumps(R.result_to_json("instance.txt", 12, res, cfg, timing)) + "\n"
    assert cpp == py
    if ref.has_result_json():
        want = ref.result_json("instance.txt", 12, dict(best_f=3, best_score=80, proven_optimal=opt, l=2,
                                                        upper_bound=83, vertex_count=50, generations=5,
                                                        total_iterations=12345, elapsed_seconds=elapsed),
                               stop, p, alpha, 10.0, 20.0, 0, 0, R.parse_variant(variant), R.parse_crossover(cross),
                               0, 0, seed, 2, tl, 0, 0, timing)
        assert cpp == want + "\n"


def test_cpp_error_types(probe):
    out = _run(probe, "errors").stdout.split("\n")
    assert out[0] == "runtime_error: line 2: duplicate symbol 1 in row 0"
    assert out[1] == "invalid_argument: population size must be at least 2"
    assert out[2] in ("CudaError",)  # no sm_100 device in this container: fails loudly, no CPU fallback


def test_cpp_cli_generate_and_verify_match_python(plse, tmp_path):
    a, b = tmp_path / "a", tmp_path / "b"
    r1 = _run(CLI, "generate", "-n", 10, "-r", 0.55, "-c", 3, "-o", a, "--seed", 4242)
    r2 = subprocess.run([sys.executable, "-m", "paper_2103_10453_b200", "generate", "-n", "10", "-r", "0.55", "-c",
                         "3", "-o", str(b), "--seed", "4242"], capture_output=True, text=True, cwd=ROOT)
    assert r1.returncode == r2.returncode == 0
    assert r1.stdout.replace(str(a), "X") == r2.stdout.replace(str(b), "X") and r1.stderr == r2.stderr
    for i in range(3):
        assert (a / f"QC-10-55-{i}.txt").read_text() == (b / f"QC-10-55-{i}.txt").read_text()
    inst = a / "QC-10-55-0.txt"
    for extra in ([], ["--exact"]):
        v1 = _run(CLI, "verify", inst, inst, *extra)
        v2 = subprocess.run([sys.executable, "-m", "paper_2103_10453_b200", "verify", str(inst), str(inst), *extra],
                            capture_output=True, text=True, cwd=ROOT)
        assert (v1.returncode, v1.stdout) == (v2.returncode, v2.stdout)
    bad = _run(CLI, "solve", tmp_path / "missing.txt")
    assert bad.returncode == 1 and bad.stderr.startswith("error: cannot open instance file")
    assert _run(CLI, "nonsense").returncode == 106
