"""ctypes front-end for the CPU checker.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, ``__graft_entry__.smoke()``
and bench.py's ``cpu_baseline`` / ``--impl reference`` legs -- never by the
product package.  Two libraries:

* ``liboracle.so``      -- the plain-C restatement (plse_oracle.c), always built.
* ``_ref/libplse_ref.so`` -- the unmodified reference headers compiled in place
  (ref_shim.cpp); present wherever ``/root/reference`` was available at build
  time (it travels to the GPU box as a built artefact).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB_GENERIC = os.path.join(HERE, "_ref", "libplse_ref.so")
REF_LIB_SPR = os.path.join(HERE, "_ref", "libplse_ref_spr.so")


def _host_is_spr() -> bool:
    """the host CPU runs -march=sapphirerapids code (avx512_fp16 + amx_tile + avx512_bf16)"""
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((l for l in f if l.startswith("flags")), "").split()
        return all(x in flags for x in ("avx512_fp16", "amx_tile", "avx512_bf16", "avx512vl"))
    except OSError:
        return False


# the reference compiled for this host's ISA when available (-march=native), else generic
REF_LIB = REF_LIB_SPR if os.path.exists(REF_LIB_SPR) and _host_is_spr() else REF_LIB_GENERIC
REF_FLAGS = ("-O3 -march=sapphirerapids -std=c++20" if REF_LIB == REF_LIB_SPR else "-O3 -march=x86-64-v3 -std=c++20")

TIE_CANON, TIE_REF = 0, 1
X_AUX, X_UX, X_NONE = 0, 1, 2
M_NEAREST, M_RANDOM = 0, 1
E_RUN, E_GENERATION, E_OFF = 0, 1, 2
STOP_NAMES = ["optimal", "time_limit", "iteration_limit", "generation_limit", "trivial"]

u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class OrStep(C.Structure):
    _fields_ = [("step", C.c_int64), ("v", C.c_int32), ("k", C.c_int32), ("e", C.c_int32),
                ("ev0", C.c_int32), ("ev1", C.c_int32), ("f_before", C.c_int32),
                ("f_after", C.c_int32), ("best_f", C.c_int32), ("tenure", C.c_int32),
                ("n_adm", C.c_int32), ("level", C.c_int32)]


class OrImproveStats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("repaired_f", C.c_int32), ("best_f", C.c_int32),
                ("alg_bytes", C.c_double)]


class OrProbe(C.Structure):
    _fields_ = [("n", C.c_int), ("steps", C.c_void_p), ("gamma", C.c_void_p), ("tabu", C.c_void_p),
                ("n_tabu", C.c_void_p), ("dumped", C.c_void_p), ("cap", C.c_int)]


class OrConfig(C.Structure):
    _fields_ = [("p", C.c_int32), ("alpha", C.c_double), ("gamma", C.c_double), ("beta", C.c_double),
                ("phase1_iters", C.c_int64), ("crossover", C.c_int32), ("matching", C.c_int32),
                ("exclusion", C.c_int32), ("master_seed", C.c_uint64), ("iteration_limit", C.c_int64),
                ("generation_limit", C.c_int64), ("tie_mode", C.c_int32),
                ("disable_optimal_stop", C.c_int32), ("variant", C.c_int32), ("phase2_iters", C.c_int64)]


class OrResult(C.Structure):
    _fields_ = [("best_f", C.c_int32), ("best_score", C.c_int32), ("proven_optimal", C.c_int32),
                ("stop_reason", C.c_int32), ("l", C.c_int32), ("upper_bound", C.c_int32),
                ("vertex_count", C.c_int32), ("generations", C.c_int64),
                ("total_iterations", C.c_int64)]


class OrGenLog(C.Structure):
    _fields_ = [("generation", C.c_int64), ("best_f", C.c_int32), ("shortfall", C.c_int32),
                ("iterations", C.c_int64), ("mean_f", C.c_double), ("mean_distance", C.c_double)]


class OrPlitsStep(C.Structure):
    _fields_ = [("step", C.c_int64), ("phase", C.c_int32), ("v", C.c_int32), ("k", C.c_int32),
                ("from_", C.c_int32), ("df", C.c_int32), ("dc", C.c_int32), ("delta", C.c_int64),
                ("cur_scaled", C.c_int64), ("best_scaled", C.c_int64), ("n_adm", C.c_int32),
                ("tenure", C.c_int32), ("active", C.c_int32), ("f", C.c_int32), ("c", C.c_int32)]


class OrPlitsStats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("phase1_iterations", C.c_int64), ("hit_target", C.c_int32),
                ("repaired", C.c_int32), ("final_f", C.c_int32), ("alg_bytes", C.c_double)]


class OrExact(C.Structure):
    _fields_ = [("optimum_f", C.c_int32), ("exact", C.c_int32), ("nodes", C.c_int64)]


class RefRunResult(C.Structure):
    _fields_ = [("best_f", C.c_int32), ("best_score", C.c_int32), ("proven_optimal", C.c_int32),
                ("stop_reason", C.c_int32), ("l", C.c_int32), ("upper_bound", C.c_int32),
                ("vertex_count", C.c_int32), ("generations", C.c_int64),
                ("total_iterations", C.c_int64), ("elapsed_seconds", C.c_double),
                ("first_best_seconds", C.c_double)]


class Graph:
    """A reduced graph (lsgraph.hpp:67) as numpy CSR arrays."""

    def __init__(self, n, nv, l, cell_row, cell_col, adj_off, adj, dom_off, dom):
        self.n, self.nv, self.l = n, nv, l
        self.cell_row, self.cell_col = cell_row, cell_col
        self.adj_off, self.adj, self.dom_off, self.dom = adj_off, adj, dom_off, dom

    def same_as(self, o: "Graph") -> bool:
        return (self.n == o.n and self.nv == o.nv and self.l == o.l
                and all(np.array_equal(getattr(self, a), getattr(o, a))
                        for a in ("cell_row", "cell_col", "adj_off", "adj", "dom_off", "dom")))


def _export(lib, prefix, h, n):
    nv = getattr(lib, prefix + "graph_nv")(h)
    l = getattr(lib, prefix + "graph_l")(h)
    na = getattr(lib, prefix + "graph_adj_len")(h)
    nd = getattr(lib, prefix + "graph_dom_len")(h)
    cr = np.zeros(max(nv, 1), np.int32)
    cc = np.zeros(max(nv, 1), np.int32)
    ao = np.zeros(nv + 1, np.int32)
    ad = np.zeros(max(na, 1), np.int32)
    do = np.zeros(nv + 1, np.int32)
    dm = np.zeros(max(nd, 1), np.uint16)
    getattr(lib, prefix + "graph_export")(h, cr, cc, ao, ad, do, dm)
    return Graph(n, nv, l, cr[:nv], cc[:nv], ao, ad[:na], do, dm[:nd])


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: str = LIB):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.or_derive_seed.restype = C.c_uint64
        L.or_derive_seed.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_canon_draw.restype = C.c_uint64
        L.or_canon_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.or_generate_instance.argtypes = [C.c_int, C.c_double, C.c_uint64, u16p]
        L.or_lsc_instance.argtypes = [C.c_int, C.c_double, C.c_uint64, u16p]
        L.or_lsc_instance.restype = None
        L.or_preprocess.restype = C.c_void_p
        L.or_preprocess.argtypes = [C.c_int, u16p]
        L.or_graph_free.argtypes = [C.c_void_p]
        for f in ("or_graph_nv", "or_graph_l", "or_graph_adj_len", "or_graph_dom_len", "or_graph_order"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.or_graph_export.argtypes = [C.c_void_p, i32p, i32p, i32p, i32p, i32p, u16p]
        L.or_eval.argtypes = [C.c_void_p, u16p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.or_gamma_build.argtypes = [C.c_void_p, u16p, i32p]
        L.or_repair.argtypes = [C.c_void_p, u16p]
        L.or_solve_exact.argtypes = [C.c_void_p, C.c_int64, C.POINTER(OrExact), u16p]
        L.or_enumerate_exact.argtypes = [C.c_void_p, C.POINTER(OrExact), u16p]
        L.or_plits.argtypes = [C.c_void_p, u16p, u16p, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_int,
                               C.c_int, C.POINTER(OrPlitsStats), C.c_void_p, C.c_int64]
        L.or_plits_probe.argtypes = [C.c_void_p, u16p, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                     C.c_int, C.c_void_p]
        L.or_improve_probe.argtypes = [C.c_void_p, u16p, C.c_uint64, C.c_int64, C.c_double, C.c_int, C.c_int,
                                       C.c_void_p]
        L.or_improve.argtypes = [C.c_void_p, u16p, u16p, C.c_uint64, C.c_int64, C.c_double, C.c_int,
                                 C.c_int, C.POINTER(OrImproveStats), C.c_void_p, C.c_int64]
        L.or_cross_distances.argtypes = [C.c_int, C.c_int, u16p, u16p, i32p, i32p]
        L.or_full_distances.argtypes = [C.c_int, C.c_int, u16p, i32p]
        L.or_update.argtypes = [C.c_void_p, C.c_int, C.c_double, u16p, i32p, u16p, i32p, i32p,
                                C.POINTER(C.c_int32), i32p, C.POINTER(C.c_int32), i32p]
        L.or_update_ex.argtypes = [C.c_void_p, C.c_int, C.c_double, u16p, i32p, u16p, i32p, i32p, C.c_int,
                                   C.c_void_p, C.POINTER(C.c_int32), i32p, C.POINTER(C.c_int32), i32p]
        L.or_offspring.argtypes = [C.c_void_p, C.c_int, u16p, i32p, C.c_int, C.c_double, C.c_int, C.c_int,
                                   u8p, C.c_uint64, C.c_uint64, u16p, i32p]
        L.or_init_population.argtypes = [C.c_void_p, C.c_int, C.c_uint64, u16p]
        L.or_init_population_ex.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, u16p]
        L.or_offspring_ex.argtypes = [C.c_void_p, C.c_int, u16p, i32p, C.c_int, C.c_double, C.c_int, C.c_int,
                                      u8p, C.c_uint64, C.c_uint64, u16p, i32p]
        L.or_run.argtypes = [C.c_int, u16p, C.POINTER(OrConfig), C.POINTER(OrResult), u16p,
                             C.c_void_p, C.c_int64]
        self._handles = {}

    # -- rng / instances
    def derive_seed(self, master, tag, index):
        return self.lib.or_derive_seed(master, tag, index)

    def canon_draw(self, s, j):
        return self.lib.or_canon_draw(s, j)

    def generate_instance(self, n, r, seed):
        g = np.zeros(n * n, np.uint16)
        if self.lib.or_generate_instance(n, r, seed, g) != 0:
            raise RuntimeError("instance generation failed")
        return g.reshape(n, n)

    def lsc_instance(self, n, r, seed):
        g = np.zeros(n * n, np.uint16)
        self.lib.or_lsc_instance(n, r, seed, g)
        return g.reshape(n, n)

    # -- graph
    def _h(self, grid):
        grid = np.ascontiguousarray(grid, np.uint16)
        key = (grid.shape[0], grid.tobytes())
        h = self._handles.get(key)
        if h is None:
            h = self.lib.or_preprocess(grid.shape[0], grid.reshape(-1))
            self._handles[key] = h
        return h

    def preprocess(self, grid) -> Graph:
        return _export(self.lib, "or_", self._h(grid), int(np.asarray(grid).shape[0]))

    def eval(self, grid, colors):
        f, c = C.c_int(), C.c_int()
        self.lib.or_eval(self._h(grid), np.ascontiguousarray(colors, np.uint16), C.byref(f), C.byref(c))
        return f.value, c.value

    def gamma(self, grid, colors):
        g = self.preprocess(grid)
        out = np.zeros(g.nv * (g.n + 1), np.int32)
        self.lib.or_gamma_build(self._h(grid), np.ascontiguousarray(colors, np.uint16), out)
        return out.reshape(g.nv, g.n + 1)

    def repair(self, grid, colors):
        c = np.array(colors, np.uint16)
        self.lib.or_repair(self._h(grid), c)
        return c

    def improve(self, grid, colors, stream_seed, budget, alpha=0.6, stop_f=0, tie=TIE_CANON,
                trace_cap=0):
        nv = len(colors)
        out = np.zeros(nv, np.uint16)
        st = OrImproveStats()
        tr = (OrStep * trace_cap)() if trace_cap else None
        self.lib.or_improve(self._h(grid), np.ascontiguousarray(colors, np.uint16), out, stream_seed,
                            budget, alpha, stop_f, tie, C.byref(st),
                            C.cast(tr, C.c_void_p) if tr is not None else None, trace_cap)
        res = dict(best=out, iterations=st.iterations, repaired_f=st.repaired_f, best_f=st.best_f,
                   alg_bytes=st.alg_bytes)
        if tr is not None:
            m = min(trace_cap, st.iterations)
            res["trace"] = [{k: getattr(tr[i], k) for k, _ in OrStep._fields_} for i in range(m)]
        return res

    def improve_probe(self, grid, colors, stream_seed, budget, steps, tabu_cap=4096, alpha=0.6, stop_f=0,
                      tie=TIE_CANON, plits_budget2=None):
        """the gamma table and the live tabu entries (v, k, until) before each listed step of or_improve
        (or of or_plits when plits_budget2 is given: steps counted over both phases, until on the phase clock)"""
        h = self._h(grid)
        nv, w = len(colors), self.lib.or_graph_order(h) + 1
        steps = np.ascontiguousarray(steps, np.int64)
        n = len(steps)
        gam = np.zeros((max(n, 1), nv, w), np.int32)
        tabu = np.zeros((max(n, 1), max(tabu_cap, 1), 3), np.int32)
        nt = np.zeros(max(n, 1), np.int32)
        dumped = np.zeros(1, np.int32)
        pr = OrProbe(n, steps.ctypes.data, gam.ctypes.data, tabu.ctypes.data, nt.ctypes.data, dumped.ctypes.data,
                     tabu_cap)
        if plits_budget2 is None:
            self.lib.or_improve_probe(h, np.ascontiguousarray(colors, np.uint16), stream_seed, budget, alpha, stop_f,
                                      tie, C.byref(pr))
        else:
            self.lib.or_plits_probe(h, np.ascontiguousarray(colors, np.uint16), stream_seed, budget, plits_budget2,
                                    alpha, stop_f, tie, C.byref(pr))
        return [dict(step=int(steps[q]), gamma=gam[q], tabu=tabu[q, :min(nt[q], tabu_cap)].copy(),
                     n_tabu=int(nt[q])) for q in range(int(dumped[0]))]

    def solve_exact(self, grid, node_budget=50_000_000, enumerate=False):
        """oracle.hpp:134 solve_exact / 141 enumerate_exact -> (f, exact, nodes, certificate)"""
        h = self._h(grid)
        nv = self.lib.or_graph_nv(h)
        cert = np.zeros(max(nv, 1), np.uint16)
        r = OrExact()
        if enumerate:
            self.lib.or_enumerate_exact(h, C.byref(r), cert)
        else:
            self.lib.or_solve_exact(h, node_budget, C.byref(r), cert)
        return r.optimum_f, bool(r.exact), r.nodes, cert[:nv]

    def plits(self, grid, colors, stream_seed, iters1=0, iters2=0, alpha=0.6, stop_f=0, tie=TIE_CANON,
              trace_cap=0):
        """plits.hpp:276 plits_run"""
        nv = len(colors)
        out = np.zeros(max(nv, 1), np.uint16)
        st = OrPlitsStats()
        tr = (OrPlitsStep * trace_cap)() if trace_cap else None
        self.lib.or_plits(self._h(grid), np.ascontiguousarray(colors, np.uint16), out, stream_seed, iters1, iters2,
                          alpha, stop_f, tie, C.byref(st), C.cast(tr, C.c_void_p) if tr is not None else None,
                          trace_cap)
        res = {k: getattr(st, k) for k, _ in OrPlitsStats._fields_}
        res["best"] = out[:nv]
        if tr is not None:
            m = min(trace_cap, st.iterations)
            res["trace"] = [{k: getattr(tr[i], k) for k, _ in OrPlitsStep._fields_} for i in range(m)]
        return res

    # -- population phases
    def cross_distances(self, members, improved):
        p, nv = members.shape
        cr = np.zeros(p * p, np.int32)
        fr = np.zeros(p * p, np.int32)
        self.lib.or_cross_distances(nv, p, np.ascontiguousarray(members, np.uint16).reshape(-1),
                                    np.ascontiguousarray(improved, np.uint16).reshape(-1), cr, fr)
        return cr.reshape(p, p), fr.reshape(p, p)

    def full_distances(self, members):
        p, nv = members.shape
        d = np.zeros(p * p, np.int32)
        self.lib.or_full_distances(nv, p, np.ascontiguousarray(members, np.uint16).reshape(-1), d)
        return d.reshape(p, p)

    def update(self, grid, members, dist, improved, cross, fresh, gamma=10.0, migrants=None):
        """population.hpp:103-183; `migrants` (k x |V|) join the pool as ids 2p..2p+k-1 (island exchange)"""
        p, nv = members.shape
        m = np.array(members, np.uint16).reshape(-1)
        d = np.array(dist, np.int32).reshape(-1)
        pbf, nsf = C.c_int32(), C.c_int32()
        sfs = np.zeros(p, np.int32)
        sel = np.zeros(p, np.int32)
        mig = np.ascontiguousarray(migrants if migrants is not None else np.zeros((0, nv)), np.uint16)
        self.lib.or_update_ex(self._h(grid), p, gamma, m, d, np.ascontiguousarray(improved, np.uint16).reshape(-1),
                              np.ascontiguousarray(cross, np.int32).reshape(-1),
                              np.ascontiguousarray(fresh, np.int32).reshape(-1), mig.shape[0],
                              mig.ctypes.data_as(C.c_void_p), C.byref(pbf), sfs, C.byref(nsf), sel)
        return dict(members=m.reshape(p, nv), dist=d.reshape(p, p), pool_best_f=pbf.value,
                    shortfall_slots=sfs[:nsf.value].tolist(), selected=sel)

    def offspring(self, grid, members, dist, excl, master_seed, generation, crossover=X_AUX, beta=20.0,
                  matching=M_NEAREST, exclusion=E_RUN):
        p, nv = members.shape
        out = np.zeros(p * nv, np.uint16)
        part = np.zeros(p, np.int32)
        self.lib.or_offspring(self._h(grid), p, np.ascontiguousarray(members, np.uint16).reshape(-1),
                              np.ascontiguousarray(dist, np.int32).reshape(-1), crossover, beta, matching,
                              exclusion, excl.reshape(-1), master_seed, generation, out, part)
        return out.reshape(p, nv), part

    def init_population(self, grid, p, master_seed, offset=0):
        g = self.preprocess(grid)
        out = np.zeros(p * g.nv, np.uint16)
        self.lib.or_init_population_ex(self._h(grid), p, master_seed, offset, out)
        return out.reshape(p, g.nv)

    def offspring_ex(self, grid, members, dist, excl, master_seed, stream_base, crossover=X_AUX, beta=20.0,
                     matching=M_NEAREST, exclusion=E_RUN):
        p, nv = members.shape
        out = np.zeros(p * nv, np.uint16)
        part = np.zeros(p, np.int32)
        self.lib.or_offspring_ex(self._h(grid), p, np.ascontiguousarray(members, np.uint16).reshape(-1),
                                 np.ascontiguousarray(dist, np.int32).reshape(-1), crossover, beta, matching,
                                 exclusion, excl.reshape(-1), master_seed, stream_base, out, part)
        return out.reshape(p, nv), part

    def run(self, grid, p=64, alpha=0.6, gamma=10.0, beta=20.0, phase1_iters=0, crossover=X_AUX,
            matching=M_NEAREST, exclusion=E_RUN, seed=0, iteration_limit=0, generation_limit=0,
            tie=TIE_CANON, disable_optimal_stop=False, log_cap=0, variant=1, phase2_iters=0):
        grid = np.ascontiguousarray(grid, np.uint16)
        n = grid.shape[0]
        cfg = OrConfig(p, alpha, gamma, beta, phase1_iters, crossover, matching, exclusion, seed,
                       iteration_limit, generation_limit, tie, int(disable_optimal_stop), variant, phase2_iters)
        res = OrResult()
        best = np.zeros(n * n + 1, np.uint16)
        log = (OrGenLog * log_cap)() if log_cap else None
        self.lib.or_run(n, grid.reshape(-1), C.byref(cfg), C.byref(res), best,
                        C.cast(log, C.c_void_p) if log is not None else None, log_cap)
        out = {k: getattr(res, k) for k, _ in OrResult._fields_}
        out["stop_reason"] = STOP_NAMES[res.stop_reason]
        out["best_colors"] = best[:res.vertex_count]
        if log is not None:
            out["log"] = [{k: getattr(log[i], k) for k, _ in OrGenLog._fields_}
                          for i in range(min(log_cap, res.generations))]
        return out


class Reference:
    """The unmodified reference (oracle/_ref/libplse_ref.so)."""

    @staticmethod
    def available(path: str = REF_LIB) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_LIB):
        L = self.lib = C.CDLL(path)
        L.ref_generate_instance.argtypes = [C.c_int, C.c_double, C.c_uint64, u16p]
        L.ref_lsc_instance.argtypes = [C.c_int, C.c_double, C.c_uint64, u16p]
        L.ref_lsc_instance.restype = None
        L.ref_preprocess.restype = C.c_void_p
        L.ref_preprocess.argtypes = [C.c_int, u16p]
        for f in ("ref_graph_nv", "ref_graph_l", "ref_graph_adj_len", "ref_graph_dom_len"):
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_graph_export.argtypes = [C.c_void_p, i32p, i32p, i32p, i32p, i32p, u16p]
        L.ref_eval.argtypes = [C.c_void_p, u16p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_gamma_build.argtypes = [C.c_void_p, u16p, i32p]
        L.ref_repair.argtypes = [C.c_void_p, u16p]
        L.ref_improve.restype = C.c_int64
        L.ref_improve.argtypes = [C.c_void_p, u16p, u16p, C.c_uint64, C.c_int64, C.c_double, C.c_int,
                                  C.POINTER(C.c_int)]
        L.ref_improve_states.restype = C.c_int64
        L.ref_improve_states.argtypes = [C.c_void_p, u16p, C.c_uint64, C.c_int64, C.c_double, u16p, u16p, i32p]
        L.ref_cross_distances.argtypes = [C.c_void_p, C.c_int, u16p, u16p, i32p, i32p]
        L.ref_update.argtypes = [C.c_void_p, C.c_int, C.c_double, u16p, i32p, u16p, i32p, i32p,
                                 C.POINTER(C.c_int32), i32p, C.POINTER(C.c_int32)]
        L.ref_excl_new.restype = C.c_void_p
        L.ref_excl_new.argtypes = [C.c_int]
        L.ref_excl_free.argtypes = [C.c_void_p]
        L.ref_excl_reset.argtypes = [C.c_void_p, C.c_int]
        L.ref_offspring.argtypes = [C.c_void_p, C.c_int, u16p, i32p, C.c_int, C.c_double, C.c_int, C.c_int,
                                    C.c_void_p, C.c_uint64, C.c_uint64, u16p]
        L.ref_init_population.argtypes = [C.c_void_p, C.c_int, C.c_uint64, u16p, C.c_void_p]
        L.ref_solve_exact.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        L.ref_solve_exact_full.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.POINTER(C.c_int),
                                           C.POINTER(C.c_int64), u16p]
        L.ref_run.argtypes = [C.c_int, u16p, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64,
                              C.c_int,
                              C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_int64, C.c_int64,
                              C.POINTER(RefRunResult), u16p]
        L.ref_improve_phase.restype = C.c_int64
        L.ref_improve_phase.argtypes = [C.c_void_p, C.c_int, u16p, C.c_void_p, C.c_uint64, C.c_uint64,
                                        C.c_int64, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.ref_default_workers.restype = C.c_int
        L.ref_plits_phase.restype = C.c_int64
        L.ref_plits_phase.argtypes = [C.c_void_p, C.c_int, u16p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int64,
                                      C.c_int64, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.ref_plits.restype = C.c_int64
        L.ref_plits.argtypes = [C.c_void_p, u16p, u16p, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_int]
        L.ref_plits_trace.restype = C.c_int64
        L.ref_plits_trace.argtypes = [C.c_void_p, u16p, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                      i32p, np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"), C.c_int64, u16p]
        L.ref_set_log.argtypes = [C.c_void_p, C.c_int64]
        L.ref_log_count.restype = C.c_int64
        L.ref_verify_certificate.argtypes = [C.c_int, u16p, C.c_int, u16p, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ref_to_grid.argtypes = [C.c_int, u16p, u16p, u16p]
        if hasattr(L, "ref_bench"):
            L.ref_bench.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_int, C.c_int64, C.c_int64, C.c_int,
                                    C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                    C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        if hasattr(L, "ref_result_json"):
            L.ref_result_json.argtypes = [C.c_char_p, C.c_int, C.POINTER(RefRunResult), C.c_char_p, C.c_int,
                                          C.c_double, C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int,
                                          C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_int64,
                                          C.c_int64, C.c_int, C.c_char_p, C.c_int]
        self._handles = {}

    def generate_instance(self, n, r, seed):
        g = np.zeros(n * n, np.uint16)
        if self.lib.ref_generate_instance(n, r, seed, g) != 0:
            raise RuntimeError("instance generation failed")
        return g.reshape(n, n)

    def lsc_instance(self, n, r, seed):
        g = np.zeros(n * n, np.uint16)
        self.lib.ref_lsc_instance(n, r, seed, g)
        return g.reshape(n, n)

    def _h(self, grid):
        grid = np.ascontiguousarray(grid, np.uint16)
        key = (grid.shape[0], grid.tobytes())
        h = self._handles.get(key)
        if h is None:
            h = self.lib.ref_preprocess(grid.shape[0], grid.reshape(-1))
            self._handles[key] = h
        return h

    def preprocess(self, grid) -> Graph:
        return _export(self.lib, "ref_", self._h(grid), int(np.asarray(grid).shape[0]))

    def eval(self, grid, colors):
        f, c = C.c_int(), C.c_int()
        self.lib.ref_eval(self._h(grid), np.ascontiguousarray(colors, np.uint16), C.byref(f), C.byref(c))
        return f.value, c.value

    def gamma(self, grid, colors):
        g = self.preprocess(grid)
        out = np.zeros(g.nv * (g.n + 1), np.int32)
        self.lib.ref_gamma_build(self._h(grid), np.ascontiguousarray(colors, np.uint16), out)
        return out.reshape(g.nv, g.n + 1)

    def repair(self, grid, colors):
        c = np.array(colors, np.uint16)
        self.lib.ref_repair(self._h(grid), c)
        return c

    def improve(self, grid, colors, stream_seed, budget, alpha=0.6, stop_f=0):
        out = np.zeros(len(colors), np.uint16)
        bf = C.c_int()
        it = self.lib.ref_improve(self._h(grid), np.ascontiguousarray(colors, np.uint16), out, stream_seed,
                                  budget, alpha, stop_f, C.byref(bf))
        return dict(best=out, iterations=it, best_f=bf.value)

    def improve_states(self, grid, colors, stream_seed, steps, alpha=0.6):
        nv = len(colors)
        rep = np.zeros(nv, np.uint16)
        states = np.zeros(steps * nv, np.uint16)
        bf = np.zeros(steps, np.int32)
        t = self.lib.ref_improve_states(self._h(grid), np.ascontiguousarray(colors, np.uint16), stream_seed,
                                        steps, alpha, rep, states, bf)
        return rep, states.reshape(steps, nv)[:t], bf[:t]

    def cross_distances(self, grid, members, improved):
        p = members.shape[0]
        cr = np.zeros(p * p, np.int32)
        fr = np.zeros(p * p, np.int32)
        self.lib.ref_cross_distances(self._h(grid), p, np.ascontiguousarray(members, np.uint16).reshape(-1),
                                     np.ascontiguousarray(improved, np.uint16).reshape(-1), cr, fr)
        return cr.reshape(p, p), fr.reshape(p, p)

    def update(self, grid, members, dist, improved, cross, fresh, gamma=10.0):
        p, nv = members.shape
        m = np.array(members, np.uint16).reshape(-1)
        d = np.array(dist, np.int32).reshape(-1)
        pbf, nsf = C.c_int32(), C.c_int32()
        sfs = np.zeros(p, np.int32)
        self.lib.ref_update(self._h(grid), p, gamma, m, d, np.ascontiguousarray(improved, np.uint16).reshape(-1),
                            np.ascontiguousarray(cross, np.int32).reshape(-1),
                            np.ascontiguousarray(fresh, np.int32).reshape(-1), C.byref(pbf), sfs, C.byref(nsf))
        return dict(members=m.reshape(p, nv), dist=d.reshape(p, p), pool_best_f=pbf.value,
                    shortfall_slots=sfs[:nsf.value].tolist())

    def new_exclusion(self, p):
        return self.lib.ref_excl_new(p)

    def offspring(self, grid, members, dist, excl_handle, master_seed, generation, crossover=X_AUX,
                  beta=20.0, matching=M_NEAREST, exclusion=E_RUN):
        p, nv = members.shape
        out = np.zeros(p * nv, np.uint16)
        self.lib.ref_offspring(self._h(grid), p, np.ascontiguousarray(members, np.uint16).reshape(-1),
                               np.ascontiguousarray(dist, np.int32).reshape(-1), crossover, beta, matching,
                               exclusion, excl_handle, master_seed, generation, out)
        return out.reshape(p, nv)

    def init_population(self, grid, p, master_seed):
        g = self.preprocess(grid)
        out = np.zeros(p * g.nv, np.uint16)
        d = np.zeros(p * p, np.int32)
        self.lib.ref_init_population(self._h(grid), p, master_seed, out, d.ctypes.data_as(C.c_void_p))
        return out.reshape(p, g.nv), d.reshape(p, p)

    def solve_exact(self, grid):
        ex = C.c_int()
        f = self.lib.ref_solve_exact(self._h(grid), C.byref(ex))
        return f, bool(ex.value)

    def solve_exact_full(self, grid, node_budget=50_000_000, enumerate=False):
        """-> (f, exact, nodes, certificate)"""
        h = self._h(grid)
        nv = self.lib.ref_graph_nv(h)
        cert = np.zeros(max(nv, 1), np.uint16)
        ex, nodes = C.c_int(), C.c_int64()
        f = self.lib.ref_solve_exact_full(h, node_budget, int(enumerate), C.byref(ex), C.byref(nodes), cert)
        return f, bool(ex.value), nodes.value, cert[:nv]

    def run(self, grid, p=64, alpha=0.6, gamma=10.0, beta=20.0, phase1_iters=0, variant=1, crossover=X_AUX,
            phase2_iters=0,
            matching=M_NEAREST, exclusion=E_RUN, seed=0, workers=1, time_limit=0.0, iteration_limit=0,
            generation_limit=0, log_cap=0):
        grid = np.ascontiguousarray(grid, np.uint16)
        n = grid.shape[0]
        res = RefRunResult()
        best = np.zeros(n * n + 1, np.uint16)
        log = (OrGenLog * log_cap)() if log_cap else None  # same layout as ref_gen_log
        self.lib.ref_set_log(C.cast(log, C.c_void_p) if log is not None else None, log_cap)
        try:
            self.lib.ref_run(n, grid.reshape(-1), p, alpha, gamma, beta, phase1_iters, phase2_iters, variant, crossover,
                             matching, exclusion, seed, workers, time_limit, iteration_limit, generation_limit,
                             C.byref(res), best)
            n_log = self.lib.ref_log_count()
        finally:
            self.lib.ref_set_log(None, 0)
        out = {k: getattr(res, k) for k, _ in RefRunResult._fields_}
        out["stop_reason"] = STOP_NAMES[res.stop_reason]
        out["best_colors"] = best[:res.vertex_count]
        if log is not None:
            out["log"] = [{k: getattr(log[i], k) for k, _ in OrGenLog._fields_} for i in range(n_log)]
        return out

    def improve_phase(self, grid, offspring, master_seed, generation, budget, alpha=0.6, stop_f=0, workers=0):
        p = offspring.shape[0]
        secs = C.c_double()
        it = self.lib.ref_improve_phase(self._h(grid), p, np.ascontiguousarray(offspring, np.uint16).reshape(-1),
                                        None, master_seed, generation, budget, alpha, stop_f, workers,
                                        C.byref(secs))
        return it, secs.value

    def plits_phase(self, grid, offspring, master_seed, generation, iters1=0, iters2=0, alpha=0.6, stop_f=0,
                    workers=0):
        """engine.hpp:184-199 with variant MPMA -> (iterations, seconds)"""
        p = offspring.shape[0]
        secs = C.c_double()
        it = self.lib.ref_plits_phase(self._h(grid), p, np.ascontiguousarray(offspring, np.uint16).reshape(-1),
                                      None, master_seed, generation, iters1, iters2, alpha, stop_f, workers,
                                      C.byref(secs))
        return it, secs.value

    def default_workers(self):
        return self.lib.ref_default_workers()

    def plits(self, grid, colors, stream_seed, iters1=0, iters2=0, alpha=0.6, stop_f=0):
        """plits.hpp:276 plits_run -> (coloring, iterations)"""
        nv = len(colors)
        out = np.zeros(max(nv, 1), np.uint16)
        it = self.lib.ref_plits(self._h(grid), np.ascontiguousarray(colors, np.uint16), out, stream_seed, iters1,
                                iters2, alpha, stop_f)
        return out[:nv], it

    def plits_trace(self, grid, colors, stream_seed, iters1=0, iters2=0, alpha=0.6, stop_f=0, cap=100000):
        """per-step (phase, v, to, df, dc, f, c), best_scaled, final coloring"""
        nv = len(colors)
        rec = np.zeros(7 * cap, np.int32)
        bs = np.zeros(cap, np.int64)
        out = np.zeros(max(nv, 1), np.uint16)
        n = self.lib.ref_plits_trace(self._h(grid), np.ascontiguousarray(colors, np.uint16), stream_seed, iters1,
                                     iters2, alpha, stop_f, rec, bs, cap, out)
        m = min(n, cap)
        return rec[:7 * m].reshape(m, 7), bs[:m], out[:nv], n

    def verify_certificate(self, instance, certificate):
        """verify.hpp:20 -> (legal, score, problems)"""
        a = np.ascontiguousarray(instance, np.uint16)
        b = np.ascontiguousarray(certificate, np.uint16)
        score = C.c_int()
        buf = C.create_string_buffer(1 << 20)
        legal = self.lib.ref_verify_certificate(a.shape[0], a.reshape(-1), b.shape[0], b.reshape(-1),
                                                C.byref(score), buf, len(buf))
        text = buf.value.decode()
        return bool(legal), score.value, (text.split("\n") if text else [])

    def to_grid(self, instance, colors):
        """coloring.hpp:171"""
        a = np.ascontiguousarray(instance, np.uint16)
        out = np.zeros_like(a)
        self.lib.ref_to_grid(a.shape[0], a.reshape(-1), np.ascontiguousarray(colors, np.uint16), out.reshape(-1))
        return out

    def bench(self, suite_dir, repeats, master_seed, p, gen_limit, phase1=0, variant=1, crossovers="aux",
              matchings="nearest", pops="", jobs=1, workers=1):
        """bench.hpp run_bench + write_rows_csv / write_aggregates_csv / report_to_json(...).dump(2)"""
        bufs = [C.create_string_buffer(1 << 20) for _ in range(3)]
        self.lib.ref_bench(suite_dir.encode(), repeats, master_seed, p, gen_limit, phase1, variant, crossovers.encode(),
                           matchings.encode(), pops.encode(), jobs, workers, C.cast(bufs[0], C.c_void_p),
                           len(bufs[0]), C.cast(bufs[1], C.c_void_p), len(bufs[1]), C.cast(bufs[2], C.c_void_p),
                           len(bufs[2]))
        return tuple(b.value.decode() for b in bufs)

    def has_result_json(self):
        return hasattr(self.lib, "ref_result_json")

    def result_json(self, name, order, result, stop_reason, p, alpha, gamma, beta, phase1, phase2, variant,
                    crossover, matching, exclusion, seed, workers, time_limit, iteration_limit, generation_limit,
                    timing=False):
        """report.hpp:85 result_to_json(...).dump(2) for the given result fields (a dict with
        RefRunResult's keys)."""
        res = RefRunResult()
        for k, _ in RefRunResult._fields_:
            if k in result and k != "stop_reason":
                setattr(res, k, result[k])
        buf = C.create_string_buffer(1 << 16)
        self.lib.ref_result_json(name.encode(), order, C.byref(res), stop_reason.encode(), p, alpha, gamma, beta,
                                 phase1, phase2, variant, crossover, matching, exclusion, seed, workers, time_limit,
                                 iteration_limit, generation_limit, int(timing), buf, len(buf))
        return buf.value.decode()
