"""B200-native Partial-MPMA (arXiv 2103.10453) behind the reference's operator API.

Python mirror of the reference's host interface for the hot path
(/root/reference/proj/include/plse), bound through the C ABI in
``include/plse_b200.h`` (ctypes; no torch types cross the boundary):

================================  =======================================
this module                       reference
================================  =======================================
``generate_instance``             instance.hpp:204  generate_instance
``parse_instance``                instance.hpp:107  parse_instance
``serialize_instance``            instance.hpp:172  serialize_instance
``preprocess``                    lsgraph.hpp:115   preprocess(build_graph)
``DevicePopulation``              Population + the five run() phases:
  ``.initialize_population()``    engine.hpp:88     initialize_population
  ``.improve(gen)``               engine.hpp:184    parallel partial_mpma_improve
  ``.compute_cross_distances()``  population.hpp:41 compute_cross_distances
  ``.update_population()``        population.hpp:103 update_population
  ``.build_offspring(gen)``       crossover.hpp:54  build_offspring
``run``                           engine.hpp:114    run (variant=partial)
``to_grid``                       coloring.hpp:171  to_grid (certificate)
``verify_certificate``            verify.hpp:20     verify_certificate
``solve_exact``                   oracle.hpp:134    solve_exact (host branch and bound)
``report.result_to_json``         report.hpp:85     result_to_json
``python -m paper_2103_10453_b200``  tools/plse.cpp  generate / solve / verify
================================  =======================================

Errors map like the reference's exceptions: ``std::invalid_argument`` ->
``ValueError``, ``std::runtime_error`` -> ``RuntimeError``; device failures
raise ``PlseCudaError``; requests outside the device envelope raise
``NotImplementedError``.  There is no CPU fallback: importing this package on
a machine without the built library raises ``ImportError``, and creating a
device context without an sm_100 GPU raises ``PlseCudaError``.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Callable, List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PLSE_LIB") or os.path.join(HERE, "libplse_b200.so")  # PLSE_LIB: A/B experiments

__all__ = [
    "generate_instance", "lsc_instance", "parse_instance", "serialize_instance", "preprocess", "ReducedGraph",
    "SolverConfig", "RunResult", "GenerationStats", "run", "DevicePopulation", "UpdateInfo", "PlseCudaError",
    "lib_path", "TIE_CANON", "TIE_REF", "derive_seed", "to_grid", "verify_certificate", "VerifyReport", "solve_exact", "ExactResult", "AUX", "UX", "NONE", "NEAREST", "RANDOM", "RUN", "GENERATION", "OFF",
]

AUX, UX, NONE = 0, 1, 2
NEAREST, RANDOM = 0, 1
RUN, GENERATION, OFF = 0, 1, 2
MPMA, PARTIAL = 0, 1
MEMBERS, OFFSPRING, IMPROVED = 0, 1, 2
TIE_CANON, TIE_REF = 0, 1
DIST, CROSS, FRESH = 0, 1, 2
STOP_NAMES = ["optimal", "time_limit", "iteration_limit", "generation_limit", "trivial", "target"]


class PlseCudaError(RuntimeError):
    """A CUDA / device failure (PLSE_ERR_CUDA)."""


# ----------------------------------------------------------------- ctypes
class _Graph(C.Structure):
    _fields_ = [("order", C.c_int32), ("vertex_count", C.c_int32), ("l", C.c_int32),
                ("cell_row", C.POINTER(C.c_int32)), ("cell_col", C.POINTER(C.c_int32)),
                ("dom_offsets", C.POINTER(C.c_int32)), ("dom", C.POINTER(C.c_uint16)),
                ("n_prefilled", C.c_int32), ("prefilled", C.POINTER(C.c_int32))]


class _Params(C.Structure):
    _fields_ = [("p", C.c_int32), ("alpha", C.c_double), ("gamma", C.c_double), ("beta", C.c_double),
                ("phase1_iters", C.c_int64), ("crossover", C.c_int32), ("matching", C.c_int32),
                ("exclusion", C.c_int32), ("tie_mode", C.c_int32), ("master_seed", C.c_uint64),
                ("p_total", C.c_int64), ("offset", C.c_int64), ("variant", C.c_int32), ("phase2_iters", C.c_int64)]


class Step(C.Structure):
    """plse_step: one PartialCol step of the parity probe (partial.hpp:92-143)."""
    _fields_ = [("step", C.c_int64), ("v", C.c_int32), ("k", C.c_int32), ("e", C.c_int32),
                ("ev0", C.c_int32), ("ev1", C.c_int32), ("f_before", C.c_int32), ("f_after", C.c_int32),
                ("best_f", C.c_int32), ("tenure", C.c_int32), ("n_adm", C.c_int32), ("level", C.c_int32)]


class Counters(C.Structure):
    _fields_ = [("improve_ms", C.c_double), ("alg_bytes", C.c_double), ("moves", C.c_int64),
                ("grid", C.c_int32), ("threads", C.c_int32), ("warps_per_sm", C.c_int32), ("slots", C.c_int32),
                ("smem_bytes", C.c_int64), ("kernel_launches", C.c_int64), ("distances_ms", C.c_double),
                ("update_ms", C.c_double), ("offspring_ms", C.c_double), ("k3_ops", C.c_double),
                ("k3_tensor_cores", C.c_int32)]


class _RunResult(C.Structure):
    _fields_ = [("best_f", C.c_int32), ("best_score", C.c_int32), ("proven_optimal", C.c_int32),
                ("stop_reason", C.c_int32), ("l", C.c_int32), ("upper_bound", C.c_int32),
                ("vertex_count", C.c_int32), ("generations", C.c_int64), ("total_iterations", C.c_int64),
                ("elapsed_seconds", C.c_double), ("time_to_best_seconds", C.c_double)]


class _SolverConfig(C.Structure):
    _fields_ = [("params", _Params), ("variant", C.c_int32), ("time_limit", C.c_double),
                ("iteration_limit", C.c_int64), ("generation_limit", C.c_int64), ("device", C.c_int32),
                ("disable_optimal_stop", C.c_int32), ("target_score", C.c_double), ("race", C.c_int32)]


class GenerationStats(C.Structure):
    """plse_generation_stats (GenerationStats, engine.hpp:49-57)"""
    _fields_ = [("generation", C.c_int64), ("best_f", C.c_int32), ("mean_f", C.c_double),
                ("mean_distance", C.c_double), ("iterations", C.c_int64), ("elapsed_seconds", C.c_double),
                ("shortfall", C.c_int32)]

    def __repr__(self):
        return "GenerationStats(" + ", ".join(f"{k}={getattr(self, k)!r}" for k, _ in self._fields_) + ")"


_GEN_CB = C.CFUNCTYPE(None, C.POINTER(GenerationStats), C.c_void_p)


def lib_path() -> str:
    return LIB_PATH


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2103_10453_b200.build` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
    i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
    i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
    vp, ctx = C.c_void_p, C.c_void_p
    sig = {
        "plse_abi_version": ([], C.c_int),
        "plse_last_error": ([vp], C.c_char_p),
        "plse_generate_instance": ([C.c_int32, C.c_double, C.c_uint64, u16p], C.c_int),
        "plse_parse_instance": ([C.c_char_p, C.POINTER(C.c_int32), vp, C.c_int32], C.c_int),
        "plse_preprocess": ([C.c_int32, u16p, C.POINTER(vp)], C.c_int),
        "plse_graph_free": ([vp], None),
        "plse_graph_view": ([vp, C.POINTER(_Graph)], C.c_int),
        "plse_to_grid": ([vp, u16p, u16p], C.c_int),
        "plse_solve_exact": ([vp, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                              u16p], C.c_int),
        "plse_verify_certificate": ([C.c_int32, u16p, C.c_int32, u16p, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32), vp, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
        "plse_create": ([C.POINTER(_Graph), C.POINTER(_Params), C.c_int32, C.POINTER(vp)], C.c_int),
        "plse_destroy": ([ctx], None),
        "plse_set_colors": ([ctx, C.c_int32, u16p, C.c_int64], C.c_int),
        "plse_get_colors": ([ctx, C.c_int32, u16p], C.c_int),
        "plse_get_row": ([ctx, C.c_int32, C.c_int32, u16p], C.c_int),
        "plse_get_dist": ([ctx, C.c_int32, i32p], C.c_int),
        "plse_set_dist": ([ctx, C.c_int32, i32p], C.c_int),
        "plse_get_stats": ([ctx, C.c_int32, vp, vp, vp], C.c_int),
        "plse_get_partners": ([ctx, i32p], C.c_int),
        "plse_get_counters": ([ctx, C.POINTER(Counters)], C.c_int),
        "plse_timer_start": ([ctx], C.c_int),
        "plse_timer_stop": ([ctx, C.POINTER(C.c_double)], C.c_int),
        "plse_device_colors": ([ctx, C.c_int32, C.POINTER(vp), C.POINTER(C.c_int64)], C.c_int),
        "plse_init_population": ([ctx], C.c_int),
        "plse_full_distances": ([ctx], C.c_int),
        "plse_improve": ([ctx, C.c_uint64, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
                         C.c_int),
        "plse_distances": ([ctx], C.c_int),
        "plse_update": ([ctx, vp, vp, vp], C.c_int),
        "plse_reset_exclusion": ([ctx], C.c_int),
        "plse_offspring": ([ctx, C.c_uint64], C.c_int),
        "plse_trace": ([ctx, C.c_int32, C.c_uint64, C.c_int64, vp, C.POINTER(C.c_int64)], C.c_int),
        "plse_export_elites": ([ctx, C.c_int32, vp, vp], C.c_int),
        "plse_import_migrants": ([ctx, C.c_int32, vp], C.c_int),
        "plse_stream": ([ctx, C.POINTER(vp)], C.c_int),
        "plse_probe": ([ctx, C.c_int32, C.c_uint64, C.c_int32, vp, vp, C.c_int32, vp, vp, C.POINTER(C.c_int32),
                        C.POINTER(C.c_int32)], C.c_int),
        "plse_solve": ([C.c_int32, u16p, C.POINTER(_SolverConfig), C.POINTER(_RunResult), u16p, _GEN_CB, vp],
                       C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.plse_abi_version() != 2:
        raise ImportError("libplse_b200.so ABI mismatch")
    return L


_lib = _load()


def _check(rc: int, ctx=None) -> None:
    if rc == 0:
        return
    msg = (_lib.plse_last_error(ctx) or b"").decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise PlseCudaError(msg)
    if rc == 3:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


# --------------------------------------------------------------- instances
def generate_instance(n: int, r: float, seed: int) -> np.ndarray:
    """instance.hpp:204 -- random partial Latin square (n x n uint16 grid)."""
    g = np.zeros(n * n, np.uint16)
    _check(_lib.plse_generate_instance(n, r, seed & (2**64 - 1), g))
    return g.reshape(n, n)


class _Xoshiro:
    """xoshiro256++ seeded by splitmix64 (rng.hpp:21-58) -- host-side, for instance builders only."""
    M = (1 << 64) - 1

    def __init__(self, seed: int):
        sm = seed & self.M
        self.s = []
        for _ in range(4):
            sm = (sm + 0x9E3779B97F4A7C15) & self.M
            z = sm
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
            self.s.append(z ^ (z >> 31))

    def next(self) -> int:
        s, M = self.s, self.M
        rotl = lambda x, k: ((x << k) | (x >> (64 - k))) & M
        result = (rotl((s[0] + s[3]) & M, 23) + s[0]) & M
        t = (s[1] << 17) & M
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = rotl(s[3], 45)
        return result

    def below(self, bound: int) -> int:
        threshold = ((1 << 64) - bound) % bound
        while True:
            x = self.next()
            if x >= threshold:
                return x % bound


def lsc_instance(n: int, r: float, seed: int) -> np.ndarray:
    """Latin-square-completion instance (config C5's stand-in for qwhdec.order70): a permuted cyclic
    square with cells deleted, so a full completion exists -- builders::lsc_instance
    (tests/support/builders.hpp:30-58)."""
    rng = _Xoshiro(seed)

    def perm(m):
        a = list(range(m))
        for i in range(m - 1, 0, -1):
            j = rng.below(i + 1)
            a[i], a[j] = a[j], a[i]
        return a

    rows, cols, syms = perm(n), perm(n), perm(n)
    grid = np.array([[syms[(rows[a] + cols[b]) % n] + 1 for b in range(n)] for a in range(n)], np.uint16)
    rng = _Xoshiro(seed ^ 0x5DEECE66D)
    keep = int(r * n * n)
    cells = perm(n * n)
    flat = grid.reshape(-1)
    for c in cells[keep:]:
        flat[c] = 0
    return grid


def parse_instance(text: str) -> np.ndarray:
    """instance.hpp:107 -- 'n' then n rows of n symbols (0 = empty)."""
    n = C.c_int32()
    _check(_lib.plse_parse_instance(text.encode(), C.byref(n), None, 0))
    g = np.zeros(n.value * n.value, np.uint16)
    _check(_lib.plse_parse_instance(text.encode(), C.byref(n), g.ctypes.data_as(C.c_void_p), g.size))
    return g.reshape(n.value, n.value)


def serialize_instance(grid: np.ndarray) -> str:
    """instance.hpp:172"""
    n = grid.shape[0]
    return f"{n}\n" + "".join(" ".join(str(int(x)) for x in row) + "\n" for row in grid)


_M64 = (1 << 64) - 1


def _splitmix64(state: int):
    state = (state + 0x9E3779B97F4A7C15) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return state, z ^ (z >> 31)


def derive_seed(master: int, tag: int, index: int) -> int:
    """rng.hpp:81-88 -- the (master, purpose tag, index) stream seed."""
    s, h = _splitmix64(master & _M64)
    s, h = _splitmix64(h ^ ((tag * 0xD1B54A32D192ED03) & _M64))
    s, h = _splitmix64(h ^ ((index * 0x8CB92BA72F3D8DD7) & _M64))
    return h


@dataclasses.dataclass
class VerifyReport:
    """verify.hpp:11-15"""
    legal: bool
    score: int
    problems: List[str]


def verify_certificate(instance: np.ndarray, certificate: np.ndarray) -> VerifyReport:
    """verify.hpp:20-73 -- order, pre-filled cells, Latin condition; score = filled cells."""
    a = np.ascontiguousarray(instance, np.uint16)
    b = np.ascontiguousarray(certificate, np.uint16)
    legal, score, length = C.c_int32(), C.c_int32(), C.c_int64()
    _check(_lib.plse_verify_certificate(a.shape[0], a.reshape(-1), b.shape[0], b.reshape(-1), C.byref(legal),
                                        C.byref(score), None, 0, C.byref(length)))
    buf = C.create_string_buffer(length.value + 1)
    _check(_lib.plse_verify_certificate(a.shape[0], a.reshape(-1), b.shape[0], b.reshape(-1), C.byref(legal),
                                        C.byref(score), C.cast(buf, C.c_void_p), len(buf), C.byref(length)))
    text = buf.value.decode()
    return VerifyReport(bool(legal.value), int(score.value), text.split("\n") if text else [])


@dataclasses.dataclass
class ReducedGraph:
    """lsgraph.hpp:67 (cells row-major, CSR domains starting with 0, prefilled triples)."""
    order: int
    vertex_count: int
    l: int
    cell_row: np.ndarray
    cell_col: np.ndarray
    dom_offsets: np.ndarray
    dom: np.ndarray
    prefilled: np.ndarray  # (k, 3): row, col, symbol

    def _struct(self) -> _Graph:
        self._keep = [np.ascontiguousarray(a, dt) for a, dt in (
            (self.cell_row, np.int32), (self.cell_col, np.int32), (self.dom_offsets, np.int32),
            (self.dom, np.uint16), (self.prefilled.reshape(-1), np.int32))]
        cr, cc, do, dm, pf = self._keep
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        return _Graph(self.order, self.vertex_count, self.l, P(cr, C.c_int32), P(cc, C.c_int32),
                      P(do, C.c_int32), P(dm, C.c_uint16), len(pf) // 3, P(pf, C.c_int32))


def preprocess(grid: np.ndarray) -> ReducedGraph:
    """lsgraph.hpp:115 -- Alg. 1 reduction of an instance grid."""
    grid = np.ascontiguousarray(grid, np.uint16)
    n = grid.shape[0]
    h = C.c_void_p()
    _check(_lib.plse_preprocess(n, grid.reshape(-1), C.byref(h)))
    try:
        v = _Graph()
        _check(_lib.plse_graph_view(h, C.byref(v)))
        nv = v.vertex_count
        arr = lambda ptr, cnt: np.ctypeslib.as_array(ptr, shape=(cnt,)).copy() if cnt else np.zeros(0, ptr._type_)
        dom_off = arr(v.dom_offsets, nv + 1)
        return ReducedGraph(v.order, nv, v.l, arr(v.cell_row, nv), arr(v.cell_col, nv), dom_off,
                            arr(v.dom, int(dom_off[-1])), arr(v.prefilled, 3 * v.n_prefilled).reshape(-1, 3))
    finally:
        _lib.plse_graph_free(h)


@dataclasses.dataclass
class ExactResult:
    """oracle.hpp:11-16"""
    optimum_f: int
    certificate: np.ndarray
    exact: bool
    nodes: int


def solve_exact(instance: np.ndarray, node_budget: int = 50_000_000) -> ExactResult:
    """oracle.hpp:134 solve_exact on the instance's reduced graph (host C++, branch and bound)."""
    inst = np.ascontiguousarray(instance, np.uint16)
    h = C.c_void_p()
    _check(_lib.plse_preprocess(inst.shape[0], inst.reshape(-1), C.byref(h)))
    try:
        view = _Graph()
        _check(_lib.plse_graph_view(h, C.byref(view)))
        cert = np.zeros(max(view.vertex_count, 1), np.uint16)
        f, ex, nodes = C.c_int32(), C.c_int32(), C.c_int64()
        _check(_lib.plse_solve_exact(h, node_budget, C.byref(f), C.byref(ex), C.byref(nodes), cert))
    finally:
        _lib.plse_graph_free(h)
    return ExactResult(int(f.value), cert[:view.vertex_count].copy(), bool(ex.value), int(nodes.value))


def to_grid(instance: np.ndarray, graph: "ReducedGraph", solution: np.ndarray) -> np.ndarray:
    """coloring.hpp:171-183 -- the certificate: pre-filled symbols plus the solution's coloured cells."""
    inst = np.ascontiguousarray(instance, np.uint16)
    colors = np.ascontiguousarray(solution, np.uint16).reshape(-1)
    if colors.size != graph.vertex_count:
        raise ValueError("solution size differs from the graph's vertex count")
    h = C.c_void_p()
    _check(_lib.plse_preprocess(inst.shape[0], inst.reshape(-1), C.byref(h)))
    try:
        out = np.zeros(inst.size, np.uint16)
        _check(_lib.plse_to_grid(h, colors, out))
    finally:
        _lib.plse_graph_free(h)
    return out.reshape(inst.shape)


# ------------------------------------------------------------------ config
@dataclasses.dataclass
class SolverConfig:
    """engine.hpp:26-47 (+ RunLimits engine.hpp:20-24)."""
    p: int = 12288
    alpha: float = 0.6
    phase1_iters: int = 0
    phase2_iters: int = 0  # MPMA (PLITS) phase-2 budget, 0 -> 2|V|
    gamma: float = 10.0
    beta: float = 20.0
    crossover: int = AUX
    matching: int = NEAREST
    exclusion: int = RUN
    master_seed: int = 0
    time_limit: float = 0.0
    iteration_limit: int = 0
    generation_limit: int = 0
    variant: int = PARTIAL
    device: int = 0
    p_total: int = 0
    offset: int = 0
    disable_optimal_stop: bool = False
    target_score: float = 0.0
    race: bool = False  # with target_score: device-global early exit (time-to-target, not parity mode)
    workers: int = 1  # reported in the result JSON (report.hpp:76); the device path uses one host thread
    tie_mode: int = 0  # TIE_CANON (throughput) or TIE_REF (the reference's reservoir draws, bit-exact)

    def _params(self) -> _Params:
        return _Params(self.p, self.alpha, self.gamma, self.beta, self.phase1_iters, self.crossover, self.matching,
                       self.exclusion, self.tie_mode, self.master_seed & (2**64 - 1), self.p_total, self.offset, self.variant,
                       self.phase2_iters)


@dataclasses.dataclass
class RunResult:
    """engine.hpp:59-71"""
    best_f: int
    best_score: int
    proven_optimal: bool
    stop_reason: str
    l: int
    upper_bound: int
    vertex_count: int
    generations: int
    total_iterations: int
    elapsed_seconds: float
    time_to_best_seconds: float
    best_solution: np.ndarray


def run(grid: np.ndarray, config: SolverConfig,
        on_generation: Optional[Callable[["GenerationStats"], None]] = None) -> RunResult:
    """engine.hpp:114 -- the whole Partial-MPMA run on one B200."""
    grid = np.ascontiguousarray(grid, np.uint16)
    n = grid.shape[0]
    cfg = _SolverConfig(config._params(), config.variant, config.time_limit, config.iteration_limit,
                        config.generation_limit, config.device, int(config.disable_optimal_stop),
                        config.target_score, int(config.race))
    res = _RunResult()
    best = np.zeros(n * n + 1, np.uint16)
    errors: List[BaseException] = []

    def cb(stats_ptr, _user):
        if on_generation is None:
            return
        try:
            on_generation(GenerationStats.from_buffer_copy(stats_ptr.contents))
        except BaseException as e:  # noqa: BLE001 -- re-raised after the C call returns
            errors.append(e)

    cfun = _GEN_CB(cb) if on_generation is not None else _GEN_CB()  # NULL: no per-generation stats work
    _check(_lib.plse_solve(n, grid.reshape(-1), C.byref(cfg), C.byref(res), best, cfun, None))
    if errors:
        raise errors[0]
    return RunResult(res.best_f, res.best_score, bool(res.proven_optimal), STOP_NAMES[res.stop_reason], res.l,
                     res.upper_bound, res.vertex_count, res.generations, res.total_iterations,
                     res.elapsed_seconds, res.time_to_best_seconds, best[:res.vertex_count].copy())


@dataclasses.dataclass
class UpdateInfo:
    """population.hpp:90-95"""
    pool_best_f: int
    shortfall_slots: List[int]


class DevicePopulation:
    """A device-resident population (one B200) with the reference's five phases.

    Buffers: ``members`` (Population::members), ``offspring`` (input of the
    improve phase), ``improved`` (its output); distance matrices ``dist``
    (members x members), ``cross`` (members x improved), ``fresh`` (improved x
    improved).  Colours cross the boundary as uint16 (Color), distances as int32.
    """

    def __init__(self, graph: ReducedGraph, config: SolverConfig):
        self.graph = graph
        self.config = config
        self.p = config.p
        self.nv = graph.vertex_count
        self._ctx = C.c_void_p()
        gs = graph._struct()
        prm = config._params()
        _check(_lib.plse_create(C.byref(gs), C.byref(prm), config.device, C.byref(self._ctx)))

    def close(self) -> None:
        if self._ctx:
            _lib.plse_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- buffers
    def _set(self, which, colors):
        a = np.ascontiguousarray(colors, np.uint16).reshape(-1)
        _check(_lib.plse_set_colors(self._ctx, which, a, a.size), self._ctx)

    def _get(self, which):
        return self.read_colors(which)

    def read_colors(self, which, out=None) -> np.ndarray:
        """Copy one of the device colourings (MEMBERS / OFFSPRING / IMPROVED) into `out` -- a C-contiguous
        uint16 [p, |V|] array the caller keeps, e.g. over pinned memory, so repeated reads allocate nothing
        and run at the full copy rate -- or into a new array."""
        if out is None:
            out = np.empty((self.p, self.nv), np.uint16)
        if out.dtype != np.uint16 or out.shape != (self.p, self.nv) or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous uint16 array of shape ({self.p}, {self.nv})")
        _check(_lib.plse_get_colors(self._ctx, which, out.reshape(-1)), self._ctx)
        return out

    def read_row(self, which, index: int) -> np.ndarray:
        """One individual's colouring (uint16 [|V|]) without copying the whole population."""
        out = np.empty(self.nv, np.uint16)
        _check(_lib.plse_get_row(self._ctx, which, int(index), out), self._ctx)
        return out

    def write_colors(self, which, colors) -> None:
        """Upload a colouring (uint16 [p, |V|]; checked against the vertex domains on the device)."""
        self._set(which, colors)

    members = property(lambda s: s._get(MEMBERS), lambda s, v: s._set(MEMBERS, v))
    offspring = property(lambda s: s._get(OFFSPRING), lambda s, v: s._set(OFFSPRING, v))
    improved = property(lambda s: s._get(IMPROVED), lambda s, v: s._set(IMPROVED, v))

    def get_dist(self, which=DIST) -> np.ndarray:
        a = np.zeros(self.p * self.p, np.int32)
        _check(_lib.plse_get_dist(self._ctx, which, a), self._ctx)
        return a.reshape(self.p, self.p)

    def set_dist(self, d: np.ndarray, which=DIST) -> None:
        a = np.ascontiguousarray(d, np.int32).reshape(-1)
        _check(_lib.plse_set_dist(self._ctx, which, a), self._ctx)

    dist = property(lambda s: s.get_dist(DIST), lambda s, v: s.set_dist(v, DIST))

    def stats(self, which=MEMBERS):
        f = np.zeros(self.p, np.int32)
        c = np.zeros(self.p, np.int32)
        it = np.zeros(self.p, np.int64)
        _check(_lib.plse_get_stats(self._ctx, which, f.ctypes.data_as(C.c_void_p), c.ctypes.data_as(C.c_void_p),
                                   it.ctypes.data_as(C.c_void_p)), self._ctx)
        return f, c, it

    def partners(self) -> np.ndarray:
        a = np.zeros(self.p, np.int32)
        _check(_lib.plse_get_partners(self._ctx, a), self._ctx)
        return a

    def counters(self) -> Counters:
        c = Counters()
        _check(_lib.plse_get_counters(self._ctx, C.byref(c)), self._ctx)
        return c

    def timer_start(self) -> None:
        """Record a CUDA event on this population's stream."""
        _check(_lib.plse_timer_start(self._ctx), self._ctx)

    def timer_stop(self) -> float:
        """Record a second event, synchronise, return the device-side elapsed ms."""
        ms = C.c_double()
        _check(_lib.plse_timer_stop(self._ctx, C.byref(ms)), self._ctx)
        return ms.value

    def device_colors(self, which=MEMBERS):
        """(device pointer, row stride) of a u8 population buffer."""
        ptr, stride = C.c_void_p(), C.c_int64()
        _check(_lib.plse_device_colors(self._ctx, which, C.byref(ptr), C.byref(stride)), self._ctx)
        return ptr.value, stride.value

    # -- phases
    def initialize_population(self) -> None:
        _check(_lib.plse_init_population(self._ctx), self._ctx)

    def compute_full_distances(self) -> None:
        _check(_lib.plse_full_distances(self._ctx), self._ctx)

    def improve(self, generation: int):
        """Improve every offspring -> improved; returns (iterations, best_f, best_idx)."""
        it, bf, bi = C.c_int64(), C.c_int32(), C.c_int32()
        _check(_lib.plse_improve(self._ctx, generation, C.byref(it), C.byref(bf), C.byref(bi)), self._ctx)
        return it.value, bf.value, bi.value

    def compute_cross_distances(self) -> None:
        _check(_lib.plse_distances(self._ctx), self._ctx)

    def update_population(self, info: bool = True) -> Optional[UpdateInfo]:
        """population.hpp:103-183 on the device.  With info=False nothing is read back (no host
        synchronisation); the UpdateInfo is returned only when asked for."""
        if not info:
            _check(_lib.plse_update(self._ctx, None, None, None), self._ctx)
            return None
        pbf, nsf = C.c_int32(), C.c_int32()
        slots = np.zeros(self.p, np.int32)
        _check(_lib.plse_update(self._ctx, C.byref(pbf), C.byref(nsf), slots.ctypes.data_as(C.c_void_p)), self._ctx)
        return UpdateInfo(pbf.value, slots[:nsf.value].tolist())

    def reset_exclusion(self) -> None:
        _check(_lib.plse_reset_exclusion(self._ctx), self._ctx)

    def build_offspring(self, generation: int) -> None:
        _check(_lib.plse_offspring(self._ctx, generation), self._ctx)

    def trace(self, idx: int, generation: int, max_steps: int):
        """Per-step parity probe: runs OFFSPRING[idx] through improve (clobbers IMPROVED[idx])."""
        buf = (Step * max(max_steps, 1))()
        n = C.c_int64()
        _check(_lib.plse_trace(self._ctx, idx, generation, max_steps, C.cast(buf, C.c_void_p), C.byref(n)),
               self._ctx)
        m = min(n.value, max_steps)
        return [{k: getattr(buf[i], k) for k, _ in Step._fields_} for i in range(m)], n.value

    def probe(self, idx: int, generation: int, steps, tabu_cap: int = 4096):
        """Per-step state probe (canonical PartialCol or PLITS): runs OFFSPRING[idx] through improve and returns,
        for every listed step the search reaches, the gamma table (|V| x (order+1), coloring.hpp:105-116)
        and the live tabu entries (v, k, until) on the reference's iteration clock (search_util.hpp:54-81);
        plus the number of vertices whose tabu cache disagreed with the dense table."""
        steps = np.ascontiguousarray(steps, np.int64)
        n = len(steps)
        w = self.graph.order + 1
        gam = np.zeros((max(n, 1), self.nv, w), np.int32)
        tabu = np.zeros((max(n, 1), max(tabu_cap, 1), 3), np.int32)
        nt = np.zeros(max(n, 1), np.int32)
        dumped, mism = C.c_int32(), C.c_int32()
        _check(_lib.plse_probe(self._ctx, idx, generation, n, steps.ctypes.data_as(C.c_void_p),
                               gam.ctypes.data_as(C.c_void_p), tabu_cap, tabu.ctypes.data_as(C.c_void_p),
                               nt.ctypes.data_as(C.c_void_p), C.byref(dumped), C.byref(mism)), self._ctx)
        out = [dict(step=int(steps[q]), gamma=gam[q], tabu=tabu[q, :min(nt[q], tabu_cap)].copy(), n_tabu=int(nt[q]))
               for q in range(dumped.value)]
        return out, mism.value

    def export_elites(self, n_elite: int, dev_ptr: int, with_f: bool = False):
        """The n_elite best members ((illegal, f, slot) order) as u8 rows into dev_ptr, written on this
        population's stream (see `stream`); with_f also returns their f (synchronises)."""
        f = np.zeros(max(n_elite, 1), np.int32)
        _check(_lib.plse_export_elites(self._ctx, n_elite, C.c_void_p(dev_ptr),
                                       f.ctypes.data_as(C.c_void_p) if with_f else None), self._ctx)
        return f[:n_elite] if with_f else None

    def import_migrants(self, n_in: int, dev_ptr: int) -> None:
        """Stage n_in u8 rows (device pointer, read on this population's stream) as extra candidates of
        the next update_population; call between improve() and update_population()."""
        _check(_lib.plse_import_migrants(self._ctx, n_in, C.c_void_p(dev_ptr)), self._ctx)

    @property
    def stream(self) -> int:
        """The cudaStream_t (as an int) every phase of this population runs on."""
        s = C.c_void_p()
        _check(_lib.plse_stream(self._ctx, C.byref(s)), self._ctx)
        return s.value or 0

    @property
    def row_bytes(self) -> int:
        """bytes per exported/imported u8 colour row (|V| rounded up to 16)."""
        return (self.nv + 15) // 16 * 16
