"""Machine-readable run results (report.hpp:14-103) for the device solver.

``result_to_json`` builds the same ordered object as the reference's
``result_to_json`` and ``dumps`` prints it the way ``tools/plse.cpp:154``
does (``nlohmann::ordered_json::dump(2)``): two-space indent, ``": "`` key
separator, shortest round-trip doubles, UTF-8 strings unescaped, non-finite
doubles as ``null``.  Wall-clock time is opt-in so the default output is
byte-identical across reruns with the same seed and flags.
"""
from __future__ import annotations

import json
import math
from typing import Any, Dict

from . import (AUX, GENERATION, MPMA, NEAREST, NONE, OFF, PARTIAL, RANDOM, RUN, UX, RunResult,
               SolverConfig)

__all__ = ["variant_name", "parse_variant", "crossover_name", "parse_crossover", "matching_name",
           "parse_matching", "exclusion_name", "parse_exclusion", "config_to_json", "result_to_json", "dumps"]


def variant_name(v: int) -> str:
    """report.hpp:14"""
    return "mpma" if v == MPMA else "partial"


def parse_variant(s: str) -> int:
    """report.hpp:18"""
    if s == "mpma":
        return MPMA
    if s == "partial":
        return PARTIAL
    raise ValueError("unknown variant: " + s)


def crossover_name(m: int) -> str:
    """report.hpp:24"""
    return {AUX: "aux", UX: "ux"}.get(m, "none")


def parse_crossover(s: str) -> int:
    """report.hpp:32"""
    try:
        return {"aux": AUX, "ux": UX, "none": NONE}[s]
    except KeyError:
        raise ValueError("unknown crossover mode: " + s) from None


def matching_name(m: int) -> str:
    """report.hpp:39"""
    return "nearest" if m == NEAREST else "random"


def parse_matching(s: str) -> int:
    """report.hpp:43"""
    try:
        return {"nearest": NEAREST, "random": RANDOM}[s]
    except KeyError:
        raise ValueError("unknown matching strategy: " + s) from None


def exclusion_name(e: int) -> str:
    """report.hpp:49"""
    return {RUN: "run", GENERATION: "generation"}.get(e, "off")


def parse_exclusion(s: str) -> int:
    """report.hpp:57"""
    try:
        return {"run": RUN, "generation": GENERATION, "off": OFF}[s]
    except KeyError:
        raise ValueError("unknown exclusion scope: " + s) from None


def _num(x: float) -> Any:
    # nlohmann writes NaN / inf as null; finite doubles keep a decimal point (0 -> 0.0)
    x = float(x)
    return x if math.isfinite(x) else None


def config_to_json(config: SolverConfig) -> Dict[str, Any]:
    """report.hpp:63-81 (key order preserved)"""
    return {
        "p": int(config.p),
        "alpha": _num(config.alpha),
        "gamma": _num(config.gamma),
        "beta": _num(config.beta),
        "phase1_iters": int(config.phase1_iters),
        "phase2_iters": int(config.phase2_iters),
        "variant": variant_name(config.variant),
        "crossover": crossover_name(config.crossover),
        "matching": matching_name(config.matching),
        "exclusion": exclusion_name(config.exclusion),
        "seed": int(config.master_seed) & ((1 << 64) - 1),
        "workers": int(config.workers),
        "time_limit": _num(config.time_limit),
        "iteration_limit": int(config.iteration_limit),
        "generation_limit": int(config.generation_limit),
    }


def result_to_json(instance_name: str, order: int, result: RunResult, config: SolverConfig,
                   include_timing: bool = False) -> Dict[str, Any]:
    """report.hpp:85-103 (key order preserved)"""
    j: Dict[str, Any] = {
        "instance": instance_name,
        "n": int(order),
        "vertices": int(result.vertex_count),
        "l": int(result.l),
        "upper_bound": int(result.upper_bound),
        "best_score": int(result.best_score),
        "f": int(result.best_f),
        "proven_optimal": bool(result.proven_optimal),
        "stop_reason": result.stop_reason,
        "generations": int(result.generations),
        "total_iterations": int(result.total_iterations),
    }
    if include_timing:
        j["elapsed_seconds"] = _num(result.elapsed_seconds)
    j["config"] = config_to_json(config)
    return j


def _nl_float(x: float) -> str:
    """nlohmann::detail::dtoa_impl::format_buffer over the shortest round-trip digits: fixed notation
    while the decimal point lies in (-4, 15] digits of the first digit, else d.ddde+XX."""
    if x != x or x in (float("inf"), float("-inf")):
        return "null"
    if x == 0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    r = repr(abs(x))
    if "e" in r:
        m, e = r.split("e")
        e10 = int(e)
    else:
        m, e10 = r, None
    if "." in m:
        ip, fp = m.split(".")
    else:
        ip, fp = m, ""
    if e10 is None:
        # fixed repr: value = ip.fp
        digits = (ip + fp).lstrip("0")
        lead = len(ip.lstrip("0")) if ip.strip("0") else -(len(fp) - len(fp.lstrip("0")))
        n = lead  # decimal point position relative to the first significant digit
    else:
        digits = (ip + fp).lstrip("0")
        n = e10 + 1
    digits = digits.rstrip("0") or "0"
    k = len(digits)
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    m2 = digits[0] + ("." + digits[1:] if k > 1 else "")
    ex = n - 1
    return f"{sign}{m2}e{'-' if ex < 0 else '+'}{abs(ex):02d}"


def _dump(v: Any, depth: int) -> str:
    if isinstance(v, dict):
        if not v:
            return "{}"
        pad, end = "  " * (depth + 1), "  " * depth
        return "{\n" + ",\n".join(f"{pad}{json.dumps(k, ensure_ascii=False)}: {_dump(x, depth + 1)}"
                                   for k, x in v.items()) + f"\n{end}}}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        pad, end = "  " * (depth + 1), "  " * depth
        return "[\n" + ",\n".join(f"{pad}{_dump(x, depth + 1)}" for x in v) + f"\n{end}]"
    if isinstance(v, bool) or v is None:
        return "true" if v is True else "false" if v is False else "null"
    if isinstance(v, float):
        return _nl_float(v)
    if isinstance(v, int):
        return str(v)
    return json.dumps(v, ensure_ascii=False)


def dumps(j: Dict[str, Any]) -> str:
    """nlohmann ``dump(2)``: the text plse.cpp:154 writes (without the trailing newline)."""
    return _dump(j, 0)
