"""``python -m paper_2103_10453_b200`` -- the solver front-end of tools/plse.cpp on the device path.

Subcommands and flags follow plse.cpp:245-311 (``generate``, ``solve``,
``verify``, ``bench``); output files, stdout/stderr lines and exit codes follow
cmd_generate (plse.cpp:111-130), cmd_solve (132-174), cmd_verify (175-198)
and cmd_bench (199-250, the suite harness in ``suite.py``).  ``solve`` runs :func:`paper_2103_10453_b200.run` on one B200;
its JSON is report.hpp's ``result_to_json`` printed as ``dump(2)``, so two
runs with the same seed and flags write byte-identical JSON and certificates
(acceptance.cpp criterion 8).
"""
from __future__ import annotations

import argparse
import math
import os
import secrets
import sys
from typing import List, Optional

from . import (SolverConfig, derive_seed, generate_instance, parse_instance, preprocess, run, serialize_instance,
               to_grid, verify_certificate)
from . import report as R

_KINSTANCE_GEN = 4  # rng.hpp:76 stream_tag::kInstanceGen


def _g(x: float) -> str:
    """``std::ostream << double`` with the default precision (6 significant digits, %g)."""
    return f"{x:g}"


def _add_solver_flags(ap: argparse.ArgumentParser) -> None:
    """plse.cpp:47-67 add_solver_flags"""
    ap.add_argument("-p", "--pop", type=int, default=1024, help="population size (default 1024)")
    ap.add_argument("--alpha", type=float, default=0.6, help="tabu tenure slope (default 0.6)")
    ap.add_argument("--gamma", type=float, default=10.0, help="population spacing divisor (default 10)")
    ap.add_argument("--beta", type=float, default=20.0, help="AUX crossover divisor (default 20)")
    ap.add_argument("--phase1-iters", type=int, default=0, help="phase-1 tabu iterations (0 = 100*|V|)")
    ap.add_argument("--phase2-iters", type=int, default=0, help="phase-2 tabu iterations (0 = 2*|V|)")
    ap.add_argument("--variant", default="mpma", help="mpma|partial (partial suits r >= 0.8)")
    ap.add_argument("--crossover", default="aux", help="aux|ux|none")
    ap.add_argument("--matching", default="nearest", help="nearest|random")
    ap.add_argument("--exclusion", default="run", help="tested-pair exclusion: run|generation|off")
    ap.add_argument("--time-limit", type=float, default=0.0, help="wall-clock limit in seconds (0 = none)")
    ap.add_argument("--iter-limit", type=int, default=0, help="total tabu-iteration budget (0 = none)")
    ap.add_argument("--gen-limit", type=int, default=0, help="generation cap (0 = none)")
    ap.add_argument("--seed", type=int, default=None, help="master RNG seed (omitted: drawn from OS entropy)")
    ap.add_argument("--workers", type=int, default=0, help="worker threads (default: hardware, or PLSE_WORKERS)")
    ap.add_argument("--paper-params", action="store_true",
                    help="use the published defaults (p=12288, alpha=0.6, gamma=10, beta=20)")
    ap.add_argument("--device", type=int, default=0, help="CUDA device (device path only)")
    ap.add_argument("--tie", default="canon", choices=["canon", "ref"],
                    help="device path: canonical tie-break (throughput) or the reference's reservoir draws "
                         "(bit-exact with the reference)")


def _resolve_seed(args) -> int:
    """plse.cpp:69-75"""
    if args.seed is None:
        args.seed = secrets.randbits(64)
    return args.seed & ((1 << 64) - 1)


def _resolve_workers(args) -> int:
    """plse.cpp:77-84 (default_workers: parallel.hpp:13-16)"""
    if args.workers > 0:
        return args.workers
    env = os.environ.get("PLSE_WORKERS")
    if env:
        try:
            count = int(env)
        except ValueError:
            count = 0
        if count > 0:
            return count
    return os.cpu_count() or 1


def make_config(args) -> SolverConfig:
    """plse.cpp:86-106 make_config (+ SolverConfig::validate, engine.hpp:38-46)"""
    cfg = SolverConfig(
        p=12288 if args.paper_params else args.pop, alpha=args.alpha, gamma=args.gamma, beta=args.beta,
        phase1_iters=args.phase1_iters, phase2_iters=args.phase2_iters, variant=R.parse_variant(args.variant),
        crossover=R.parse_crossover(args.crossover), matching=R.parse_matching(args.matching),
        exclusion=R.parse_exclusion(args.exclusion), time_limit=args.time_limit,
        iteration_limit=args.iter_limit, generation_limit=args.gen_limit, master_seed=_resolve_seed(args),
        workers=_resolve_workers(args), device=args.device, tie_mode=1 if args.tie == "ref" else 0)
    validate_config(cfg)
    return cfg


def validate_config(cfg: SolverConfig) -> None:
    """engine.hpp:38-46 SolverConfig::validate"""
    from . import AUX
    if cfg.p < 2:
        raise ValueError("population size must be at least 2")
    if not cfg.gamma > 1.0:
        raise ValueError("gamma must exceed 1")
    if cfg.crossover == AUX and not cfg.beta > cfg.gamma:
        raise ValueError("beta must exceed gamma")
    if not cfg.alpha >= 0.0:
        raise ValueError("alpha must be non-negative")
    if cfg.phase1_iters < 0 or cfg.phase2_iters < 0:
        raise ValueError("phase budgets must be positive")
    if cfg.workers < 1:
        raise ValueError("workers must be at least 1")


def load_instance(path: str):
    """instance.hpp:186-192"""
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        raise RuntimeError("cannot open instance file: " + path) from None
    return parse_instance(text)


def save_instance(grid, path: str) -> None:
    """instance.hpp:194-198"""
    try:
        with open(path, "w") as fh:
            fh.write(serialize_instance(grid))
    except OSError:
        raise RuntimeError("cannot write file: " + path) from None


def cmd_generate(args) -> int:
    """plse.cpp:111-130"""
    master = _resolve_seed(args)
    os.makedirs(args.out_dir, exist_ok=True)
    r_tag = int(math.floor(100.0 * args.ratio + 0.5))  # std::lround (r > 0)
    for i in range(args.count):
        grid = generate_instance(args.order, args.ratio, derive_seed(master, _KINSTANCE_GEN, i))
        path = os.path.join(args.out_dir, f"QC-{args.order}-{r_tag}-{i}.txt")
        save_instance(grid, path)
        print(f"{path} ({int((grid != 0).sum())} filled)")
    print(f"seed {master}", file=sys.stderr)
    return 0


def cmd_solve(args) -> int:
    """plse.cpp:132-174"""
    grid = load_instance(args.instance)
    cfg = make_config(args)
    graph = preprocess(grid)
    mem = 3.0 * cfg.p * cfg.p * 4 + 3.0 * cfg.p * graph.vertex_count * 2  # plse.cpp:101-108 warn_memory
    if mem > 2e9:
        print(f"warning: p={cfg.p} needs about {int(mem / 1e6)} MB for distance blocks; consider a smaller --pop",
              file=sys.stderr)

    on_gen = None
    if args.log:
        def on_gen(st):
            line = (f"gen {st.generation} best_f {st.best_f} mean_f {_g(st.mean_f)} mean_dist "
                    f"{_g(st.mean_distance)} iters {st.iterations} elapsed {_g(st.elapsed_seconds)}")
            if st.shortfall > 0:
                line += f" shortfall {st.shortfall}"
            print(line, file=sys.stderr)

    result = run(grid, cfg, on_gen)
    text = R.dumps(R.result_to_json(os.path.basename(args.instance), grid.shape[0], result, cfg, args.timing)) + "\n"
    if not args.json:
        sys.stdout.write(text)
    else:
        with open(args.json, "w") as fh:
            fh.write(text)
    if args.cert:
        save_instance(to_grid(grid, graph, result.best_solution), args.cert)
    print(f"score {result.best_score}/{result.upper_bound}{' (optimal)' if result.proven_optimal else ''} in "
          f"{_g(result.elapsed_seconds)}s, {result.total_iterations} iterations, seed {cfg.master_seed}",
          file=sys.stderr)
    return 0 if result.proven_optimal else 2


def cmd_verify(args) -> int:
    """plse.cpp:175-198"""
    from . import solve_exact
    inst = load_instance(args.instance)
    cert = load_instance(args.certificate)
    rep = verify_certificate(inst, cert)
    if not rep.legal:
        print("illegal certificate:")
        for prob in rep.problems:
            print("  " + prob)
        return 1
    print(f"legal, score {rep.score}")
    g = preprocess(inst)
    n = inst.shape[0]
    ub = n * n - 2 if g.l == 1 else n * n - g.l  # lsgraph.hpp:220-225 compute_bounds
    print(f"upper bound {ub} (l = {g.l})")
    if args.exact:
        ex = solve_exact(inst, args.node_budget)
        optimum = n * n - g.l - ex.optimum_f
        print(f"exact optimum {optimum}{'' if ex.exact else ' (budget exhausted)'}, gap {optimum - rep.score}")
    return 0


def cmd_bench(args) -> int:
    """plse.cpp:199-250"""
    import dataclasses
    from . import suite as S
    tasks = S.suite_tasks(args.suite)
    if not tasks:
        print(f"error: no .txt instances under {args.suite}", file=sys.stderr)
        return 1
    base = make_config(args)
    cross = args.sweep_crossover or [args.crossover]
    match = args.sweep_matching or [args.matching]
    pops = args.sweep_pop or [base.p]
    sweep = []
    for cname in cross:
        for mname in match:
            for p in pops:
                cfg = dataclasses.replace(base, crossover=R.parse_crossover(cname), matching=R.parse_matching(mname),
                                          p=int(p))
                validate_config(cfg)
                sweep.append(cfg)
    rep = S.run_bench(tasks, sweep, args.repeats, base.master_seed, args.jobs, sys.stderr)
    import io
    if args.csv:
        with open(args.csv, "w") as fh:
            S.write_rows_csv(rep, fh)
        print(f"rows -> {args.csv}", file=sys.stderr)
    else:
        S.write_rows_csv(rep, sys.stdout)
    if args.json:
        with open(args.json, "w") as fh:
            fh.write(R.dumps(S.report_to_json(rep)) + "\n")
        print(f"report -> {args.json}", file=sys.stderr)
    agg = io.StringIO()
    S.write_aggregates_csv(rep, agg)
    sys.stderr.write(agg.getvalue())
    return 0


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2103_10453_b200",
                                 description="partial Latin square extension solver")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("generate", help="generate random instances")
    g.add_argument("-n", "--order", type=int, required=True, help="grid order")
    g.add_argument("-r", "--ratio", type=float, required=True, help="fill ratio in (0,1)")
    g.add_argument("-c", "--count", type=int, default=1, help="number of instances")
    g.add_argument("-o", "--out-dir", default=".", help="output directory")
    g.add_argument("--seed", type=int, default=None, help="master seed")
    s = sub.add_parser("solve", help="solve one instance")
    s.add_argument("instance", help="instance file")
    s.add_argument("--json", default="", help="write the run result JSON here (default: stdout)")
    s.add_argument("--cert", default="", help="write the completed-grid certificate here")
    s.add_argument("--log", action="store_true", help="per-generation log on stderr")
    s.add_argument("--timing", action="store_true", help="include wall-clock time in the JSON output")
    _add_solver_flags(s)
    v = sub.add_parser("verify", help="validate a certificate against its instance")
    v.add_argument("instance", help="instance file")
    v.add_argument("certificate", help="certificate file")
    v.add_argument("--exact", action="store_true", help="also compute the exact optimum (small instances)")
    v.add_argument("--node-budget", type=int, default=50_000_000, help="search-node cap for --exact")
    b = sub.add_parser("bench", help="solve a directory of instances")
    b.add_argument("suite", help="directory of instance files")
    b.add_argument("--repeats", type=int, default=5, help="independent runs per instance (default 5)")
    b.add_argument("--csv", default="", help="write per-run rows CSV here (default: stdout)")
    b.add_argument("--json", default="", help="write the full report JSON here")
    b.add_argument("--sweep-crossover", nargs="+", default=[], help="ablation: crossover modes to sweep")
    b.add_argument("--sweep-matching", nargs="+", default=[], help="ablation: matching strategies to sweep")
    b.add_argument("--sweep-pop", nargs="+", type=int, default=[], help="ablation: population sizes to sweep")
    b.add_argument("--jobs", type=int, default=1, help="instances solved concurrently (default 1)")
    _add_solver_flags(b)
    args = ap.parse_args(argv)
    try:
        if args.cmd == "generate":
            return cmd_generate(args)
        if args.cmd == "solve":
            return cmd_solve(args)
        if args.cmd == "bench":
            return cmd_bench(args)
        return cmd_verify(args)
    except Exception as e:  # noqa: BLE001 -- plse.cpp:312-315
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
