"""Benchmark-suite harness over the device solver (bench.hpp:19-252, plse.cpp:199-250).

``run_bench`` solves every instance file of a suite ``repeats`` times for every
configuration of a sweep and returns a :class:`BenchReport` whose per-run rows
and per-class aggregates print exactly as the reference's ``write_rows_csv``,
``write_aggregates_csv`` and ``report_to_json(...).dump(2)``.  Run seeds derive
from (master seed, instance index, sweep index, repeat) through stream tag
kBench (rng.hpp:77), so a report does not depend on ``jobs``.  With ``jobs`` >
1 the runs are spread over the visible devices (one host thread per job).
"""
from __future__ import annotations

import dataclasses
import json
import math
import os
import threading
from typing import IO, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import SolverConfig, derive_seed, run
from . import report as R

_KBENCH = 5  # rng.hpp:77 stream_tag::kBench

__all__ = ["BenchRow", "BenchAggregate", "BenchReport", "BenchTask", "parse_instance_name", "compute_aggregates",
           "write_rows_csv", "write_aggregates_csv", "report_to_json", "run_bench", "suite_tasks"]


def _g(x: float) -> str:
    """``std::ostream << double`` (default precision: %g, 6 significant digits)."""
    return f"{x:g}"


@dataclasses.dataclass
class BenchRow:
    """bench.hpp:21-39"""
    instance: str = ""
    n: int = 0
    r_percent: int = 0
    id: str = ""
    repeat: int = 0
    seed: int = 0
    p: int = 0
    crossover: str = ""
    matching: str = ""
    variant: str = ""
    score: int = 0
    f: int = 0
    upper_bound: int = 0
    proven_optimal: bool = False
    generations: int = 0
    iterations: int = 0
    elapsed_seconds: float = 0.0


@dataclasses.dataclass
class BenchAggregate:
    """bench.hpp:41-55"""
    n: int = 0
    r_percent: int = 0
    crossover: str = ""
    matching: str = ""
    variant: str = ""
    p: int = 0
    instances: int = 0
    runs: int = 0
    f_best_mean: float = 0.0
    f_avg_mean: float = 0.0
    optimal_rate: float = 0.0
    time_mean: float = 0.0


@dataclasses.dataclass
class BenchReport:
    """bench.hpp:57-60"""
    rows: List[BenchRow] = dataclasses.field(default_factory=list)
    aggregates: List[BenchAggregate] = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class BenchTask:
    """bench.hpp:187-191"""
    path: str
    stem: str
    instance_index: int = 0


def _cpp_round(x: float) -> int:
    """std::lround: halves away from zero."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def _istream_int(s: str, i: int):
    """``istream >> int`` from position i: skip whitespace, optional sign, digits (None on failure)."""
    while i < len(s) and s[i] in " \t\n\v\f\r":
        i += 1
    j = i
    if j < len(s) and s[j] in "+-":
        j += 1
    k = j
    while k < len(s) and s[k].isdigit():
        k += 1
    if k == j:
        return None, i
    return int(s[i:k]), k


def _istream_char(s: str, i: int):
    """``istream >> char``: skip whitespace, take one character."""
    while i < len(s) and s[i] in " \t\n\v\f\r":
        i += 1
    if i >= len(s):
        return None, i
    return s[i], i + 1


def parse_instance_name(stem: str, grid: np.ndarray) -> Tuple[int, int, str]:
    """bench.hpp:64-81: QC-<n>-<100r>-<id>, else the grid's order and measured fill ratio."""
    n = int(grid.shape[0])
    r_percent = _cpp_round(100.0 * float((grid != 0).sum()) / (n * n))
    ident = stem
    if stem.startswith("QC-"):
        t = stem[3:]
        pn, i = _istream_int(t, 0)
        d1, i = _istream_char(t, i) if pn is not None else (None, i)
        pr, i = _istream_int(t, i) if d1 is not None else (None, i)
        d2, i = _istream_char(t, i) if pr is not None else (None, i)
        pid = t[i:].split("\n", 1)[0] if d2 is not None else ""
        if pn is not None and d1 == "-" and pr is not None and d2 == "-" and pid and pn == n:
            r_percent = pr
            ident = pid
    return n, r_percent, ident


def compute_aggregates(report: BenchReport) -> None:
    """bench.hpp:83-118: classes (n, r, crossover, matching, variant, p); f_best per instance."""
    classes: Dict[tuple, Dict[str, List[BenchRow]]] = {}
    for row in report.rows:
        key = (row.n, row.r_percent, row.crossover, row.matching, row.variant, row.p)
        classes.setdefault(key, {}).setdefault(row.instance, []).append(row)
    report.aggregates = []
    for key in sorted(classes):
        instances = classes[key]
        agg = BenchAggregate(*key)
        agg.instances = len(instances)
        best_sum = score_sum = time_sum = 0.0
        optimal = runs = 0
        for name in sorted(instances):
            best = 0
            for row in instances[name]:
                best = max(best, row.score)
                score_sum += row.score
                time_sum += row.elapsed_seconds
                optimal += int(row.proven_optimal)
                runs += 1
            best_sum += best
        agg.runs = runs
        agg.f_best_mean = best_sum / agg.instances
        agg.f_avg_mean = score_sum / runs
        agg.optimal_rate = optimal / runs
        agg.time_mean = time_sum / runs
        report.aggregates.append(agg)


def write_rows_csv(report: BenchReport, out: IO[str]) -> None:
    """bench.hpp:120-132"""
    out.write("instance,n,r,id,repeat,seed,p,crossover,matching,variant,score,f,upper_bound,"
              "proven_optimal,generations,iterations,elapsed_seconds\n")
    for r in report.rows:
        out.write(f"{r.instance},{r.n},{r.r_percent},{r.id},{r.repeat},{r.seed},{r.p},{r.crossover},{r.matching},"
                  f"{r.variant},{r.score},{r.f},{r.upper_bound},{1 if r.proven_optimal else 0},{r.generations},"
                  f"{r.iterations},{_g(r.elapsed_seconds)}\n")


def write_aggregates_csv(report: BenchReport, out: IO[str]) -> None:
    """bench.hpp:134-143"""
    out.write("n,r,crossover,matching,variant,p,instances,runs,f_best_mean,f_avg_mean,optimal_rate,time_mean\n")
    for a in report.aggregates:
        out.write(f"{a.n},{a.r_percent},{a.crossover},{a.matching},{a.variant},{a.p},{a.instances},{a.runs},"
                  f"{_g(a.f_best_mean)},{_g(a.f_avg_mean)},{_g(a.optimal_rate)},{_g(a.time_mean)}\n")


def report_to_json(report: BenchReport) -> dict:
    """bench.hpp:145-185 (key order preserved); print with report.dumps."""
    rows = [{"instance": r.instance, "n": r.n, "r": r.r_percent, "id": r.id, "repeat": r.repeat, "seed": r.seed,
             "p": r.p, "crossover": r.crossover, "matching": r.matching, "variant": r.variant, "score": r.score,
             "f": r.f, "upper_bound": r.upper_bound, "proven_optimal": bool(r.proven_optimal),
             "generations": r.generations, "iterations": r.iterations,
             "elapsed_seconds": float(r.elapsed_seconds)} for r in report.rows]
    aggs = [{"n": a.n, "r": a.r_percent, "crossover": a.crossover, "matching": a.matching, "variant": a.variant,
             "p": a.p, "instances": a.instances, "runs": a.runs, "f_best_mean": float(a.f_best_mean),
             "f_avg_mean": float(a.f_avg_mean), "optimal_rate": float(a.optimal_rate),
             "time_mean": float(a.time_mean)} for a in report.aggregates]
    return {"rows": rows, "aggregates": aggs}


def load_instance(path: str):
    """instance.hpp:186-192"""
    from . import parse_instance
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        raise RuntimeError("cannot open instance file: " + path) from None
    return parse_instance(text)


def suite_tasks(suite_dir: str) -> List[BenchTask]:
    """plse.cpp:203-211: the suite's *.txt files in sorted path order."""
    files = sorted(os.path.join(suite_dir, f) for f in os.listdir(suite_dir)
                   if f.endswith(".txt") and os.path.isfile(os.path.join(suite_dir, f)))
    return [BenchTask(p, os.path.splitext(os.path.basename(p))[0], i) for i, p in enumerate(files)]


def run_bench(tasks: Sequence[BenchTask], sweep: Sequence[SolverConfig], repeats: int, master_seed: int,
              jobs: int = 1, progress: Optional[IO[str]] = None, devices: Optional[Sequence[int]] = None,
              load=None) -> BenchReport:
    """bench.hpp:196-250"""
    if not tasks:
        raise ValueError("empty benchmark suite")
    if not sweep:
        raise ValueError("empty configuration sweep")
    if load is None:
        load = load_instance
    specs = [(t, s, rep) for t in tasks for s in range(len(sweep)) for rep in range(repeats)]
    rows: List[Optional[BenchRow]] = [None] * len(specs)
    if devices is None:
        try:
            import torch
            devices = list(range(max(torch.cuda.device_count(), 1)))
        except Exception:  # noqa: BLE001 -- torch is optional here
            devices = [0]
    lock = threading.Lock()
    errors: List[BaseException] = []

    def one(k: int, device: int) -> None:
        task, s, rep = specs[k]
        grid = load(task.path)
        cfg = dataclasses.replace(sweep[s], device=device)
        cfg.master_seed = derive_seed(master_seed, _KBENCH,
                                      ((task.instance_index * len(sweep) + s) * repeats + rep) & ((1 << 64) - 1))
        res = run(grid, cfg)
        row = BenchRow(instance=task.stem, repeat=rep, seed=cfg.master_seed, p=cfg.p,
                       crossover=R.crossover_name(cfg.crossover), matching=R.matching_name(cfg.matching),
                       variant=R.variant_name(cfg.variant), score=res.best_score, f=res.best_f,
                       upper_bound=res.upper_bound, proven_optimal=res.proven_optimal,
                       generations=res.generations, iterations=res.total_iterations,
                       elapsed_seconds=res.elapsed_seconds)
        row.n, row.r_percent, row.id = parse_instance_name(task.stem, grid)
        rows[k] = row
        if progress is not None:
            with lock:
                progress.write(f"{row.instance} repeat {row.repeat} score {row.score}/{row.upper_bound}"
                               f"{' optimal' if row.proven_optimal else ''}\n")

    jobs = max(1, int(jobs))
    if jobs == 1:
        for k in range(len(specs)):
            one(k, devices[0])
    else:
        nxt = [0]

        def worker(w: int) -> None:
            while True:
                with lock:
                    k = nxt[0]
                    nxt[0] += 1
                if k >= len(specs) or errors:
                    return
                try:
                    one(k, devices[w % len(devices)])
                except BaseException as e:  # noqa: BLE001 -- re-raised after the join
                    errors.append(e)
                    return

        threads = [threading.Thread(target=worker, args=(w,)) for w in range(jobs)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
    report = BenchReport(rows=[r for r in rows if r is not None])
    compute_aggregates(report)
    return report
