"""§8(f) rank 4: the exact optimum (oracle.hpp:24-179) and the verifier (verify.hpp).

* the oracle's C restatement (or_solve_exact / or_enumerate_exact) == the compiled
  reference: optimum, exactness flag, node count and certificate, including node-budget
  exhaustion;
* the product's host branch and bound (plse_solve_exact, used by ``verify --exact``) ==
  the same, node for node, with the recursion replaced by an explicit stack;
* branch and bound == full enumeration on tiny graphs (test_oracle.cpp's cross-check);
* the acceptance c1/c9 suite's exact optima (golden, from the reference).
"""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "ref_golden.npz"))


def test_exact_suite_golden(plse, orc):
    suite = G["suite"]
    for i in range(0, 200, 3):
        grid = G[f"suite_{i}"]
        f, ex, nodes, cert = orc.solve_exact(grid)
        assert ex and f == suite[i][2], i
        r = plse.solve_exact(grid)
        assert (r.optimum_f, r.exact, r.nodes) == (f, ex, nodes) and np.array_equal(r.certificate, cert), i
        fo, co = orc.eval(grid, cert)
        assert co == 0 and fo == f


def test_exact_matches_reference(plse, orc, ref):
    rng = np.random.default_rng(134)
    for t in range(60):
        n = int(rng.integers(3, 8))
        grid = ref.generate_instance(n, float(rng.uniform(0.15, 0.8)), int(rng.integers(0, 2**40)))
        budget = [50_000_000, 7, 100, 1][t % 4]
        want = ref.solve_exact_full(grid, budget)
        got = orc.solve_exact(grid, budget)
        assert got[:3] == want[:3] and np.array_equal(got[3], want[3]), t
        r = plse.solve_exact(grid, budget)
        assert (r.optimum_f, r.exact, r.nodes) == want[:3] and np.array_equal(r.certificate, want[3]), t


def test_branch_and_bound_equals_enumeration(orc, ref):
    rng = np.random.default_rng(141)
    done = 0
    for t in range(40):
        n = int(rng.integers(3, 6))
        grid = orc.generate_instance(n, float(rng.uniform(0.45, 0.85)), int(rng.integers(0, 2**40)))
        if orc.preprocess(grid).nv > 12:
            continue
        e = orc.solve_exact(grid, enumerate=True)
        b = orc.solve_exact(grid)
        assert e[0] == b[0]
        re = ref.solve_exact_full(grid, enumerate=True)
        assert e[:3] == re[:3] and np.array_equal(e[3], re[3])
        done += 1
    assert done > 10


def test_cli_verify_exact(plse, tmp_path):
    import subprocess
    import sys
    grid = G["suite_7"]
    (tmp_path / "i.txt").write_text(plse.serialize_instance(grid))
    r = plse.solve_exact(grid)
    g = plse.preprocess(grid)
    (tmp_path / "c.txt").write_text(plse.serialize_instance(plse.to_grid(grid, g, r.certificate)))
    out = subprocess.run([sys.executable, "-m", "paper_2103_10453_b200", "verify", str(tmp_path / "i.txt"),
                          str(tmp_path / "c.txt"), "--exact"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    n = grid.shape[0]
    score = n * n - g.l - r.optimum_f
    ub = n * n - 2 if g.l == 1 else n * n - g.l
    assert out.returncode == 0, out.stderr
    assert out.stdout == (f"legal, score {score}\nupper bound {ub} (l = {g.l})\n"
                          f"exact optimum {score}, gap 0\n")
