#!/usr/bin/env python
"""bench.py -- Partial-MPMA on B200: tabu moves/s (BASELINE.json metric).

Workload (BASELINE.json configs[2], the config the metric is quoted on; it
fits one GPU): PLSE n=60, 50% preassigned (generate_instance(60, 0.5, 12345),
|V| = 1800), population 16384 per GPU, PartialCol budget 100|V| per
individual, AUX crossover + nearest-neighbour matching (engine.hpp defaults).

A STEP is one Partial-MPMA generation on the device-resident population:
improve (fused gamma/repair/PartialCol kernel over all 16384 individuals) ->
cross/fresh distance blocks -> pool update -> matching + crossover.  Moves are
counted exactly as the reference counts SearchStats.iterations
(partial.hpp:161-167).  value = moves of all ranks / max-over-ranks device time
(CUDA events on the library's stream).  Inputs live in HBM; every step's
working set (1.5 GB of distance blocks, GBs of tabu scratch) is far larger
than the 126 MB L2, so no explicit flush is needed.

N > 1 (torchrun): island model -- the population of 16384 is
sharded into N islands of 16384/N individuals (strong scaling, BASELINE C3:
"population 16384 sharded over 2/4/8 B200"; --weak keeps 16384 per GPU), stream
index space gen*p_total + rank*p + i, and every 2 generations the ranks
all-gather 32 elites each over NCCL (on the population's CUDA stream) and stage
the other ranks' elites as extra candidates of their next pool update.

--impl reference: the reference's own CPU improve phase (oracle/_ref =
/root/reference compiled in place; parallel_for over all host threads,
partial_mpma_improve, engine.hpp:184-206), each step a bounded sample of the
same C3 workload.

--variant mpma: the same generation with the MPMA variant's improve operator
(PLITS, plits.hpp:276-292; the GPU kernel k_plits), budgets 100|V| + 2|V|; the
CPU legs then time the reference's plits_run phase.  Not the headline (the
north star names the PartialCol path); reported for the §8(f) PLITS row.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tabu moves/s (whole box) at pop 16384; time-to-reference-best on PLSE n=60"
UNIT = "moves/s"


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pop", type=int, default=16384, help="total population (sharded over the GPUs)")
    ap.add_argument("--weak", action="store_true", help="--pop individuals per GPU instead of in total")
    ap.add_argument("--n", type=int, default=60)
    ap.add_argument("--r", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=12345)
    ap.add_argument("--lsc", action="store_true", help="LSC instance builders::lsc_instance(n, r, seed) (config C5)")
    ap.add_argument("--master-seed", type=int, default=1)
    ap.add_argument("--budget", type=int, default=0, help="PartialCol iterations per individual (0 = 100|V|)")
    ap.add_argument("--variant", default="partial", choices=["partial", "mpma"],
                    help="improve operator: PartialCol (headline) or PLITS (MPMA)")
    ap.add_argument("--budget2", type=int, default=0, help="PLITS phase-2 iterations (0 = 2|V|)")
    ap.add_argument("--tie", default="canon", choices=["canon", "ref"],
                    help="PartialCol tie-break: canonical (throughput) or the reference's draws (bit-exact)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--migrate-every", type=int, default=2)
    ap.add_argument("--elites", type=int, default=32)
    ap.add_argument("--cpu-per-thread", type=int, default=72, help="individuals per host thread in the CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttb", action="store_true")
    ap.add_argument("--ttb-ref-pop", type=int, default=1024)
    ap.add_argument("--ttb-hard", action="store_true",
                    help="also chase the reference's best on n=60 r=0.7 and C4 live (~15 min; tools/ttb_hard.py)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def kernel_src_hash(kernel: str) -> str:
    """sha256 (16 hex) of the sources the named improve kernel is compiled from: an ncu capture counts
    for a bench line only if it was taken of the same kernel source."""
    import hashlib
    csrc = os.path.join(ROOT, "paper_2103_10453_b200", "csrc")
    files = {"k_improve": ["improve.cu", "improve_common.cuh", "common.cuh", "device_api.h"],
             "k_plits": ["plits.cu", "plits_common.cuh", "improve_common.cuh", "common.cuh", "device_api.h"]}[kernel]
    h = hashlib.sha256()
    for name in files:
        with open(os.path.join(csrc, name), "rb") as f:
            h.update(name.encode() + b"\0" + f.read())
    return h.hexdigest()[:16]


def ncu_profile(kernel: str, config_key: str):
    """The committed ncu --set full summary of this kernel (profiles/<kernel>_ncu_summary.json) if it was
    captured from the same kernel source and config; else None (the line then says why)."""
    path = os.path.join(ROOT, "profiles", f"{kernel}_ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
    except (OSError, ValueError):
        return None, "no committed ncu summary"
    if d.get("src_hash") != kernel_src_hash(kernel):
        return None, f"{os.path.relpath(path, ROOT)} was captured from another kernel source"
    if d.get("config_key") != config_key:
        return None, f"{os.path.relpath(path, ROOT)} was captured at another config"
    return d, os.path.relpath(path, ROOT)


def lsc_grid(a):
    """C5: the order-n LSC stand-in builders::lsc_instance (tests/support/builders.hpp:46-58), restated with
    the library's xoshiro (same stream as the reference builder)."""
    from paper_2103_10453_b200 import lsc_instance
    return lsc_instance(a.n, a.r, a.seed)


def i8_peak():
    """dense i8 tensor peak for the K3 roofline: B200_PROFILING.md's dense fp8/i8 rate (4.5 POPS; the driver's
    MEASURED_PEAKS.json has no 8-bit entry).  The best library rate measured on a B200 of this pool
    (profiles/i8_peak.json: cuBLASLt int8 GEMM via torch._int_mm, tools/probes/i8_peak.py) is reported beside
    it: it sits below this repo's own k_sim_tc, so it cannot serve as the ceiling."""
    measured = None
    try:
        with open(os.path.join(ROOT, "profiles", "i8_peak.json")) as f:
            d = json.load(f)
        measured = {"cublaslt_i8_tops_burst": float(d["i8_tops_burst"]),
                    "cublaslt_i8_tops_sustained": float(d["i8_tops_sustained"]), "source": "profiles/i8_peak.json"}
    except (OSError, KeyError, ValueError):
        pass
    return 4500.0, "B200_PROFILING.md dense fp8/i8 tensor rate (4.5 POPS)", measured


def k3_roofline(ph, tensor_cores):
    """similarity GEMM (one-hot i8 tcgen05): algorithmic ops (2*K_pad per pair: p^2 cross pairs + p(p-1)/2
    fresh pairs) over the distance phase's time, which includes the one-hot expansion of both operands."""
    if ph["distances"] <= 0 or ph["k3_ops"] <= 0:
        return None
    peak, src, measured = i8_peak()
    achieved = ph["k3_ops"] / (ph["distances"] / 1e3) / 1e12
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS", "frac": achieved / peak,
            "kernel": "k_onehot + k_sim_tc" if tensor_cores else "k_hamming (CUDA cores)", "peak_source": src,
            "measured_library_rate": measured,
            "includes": "one-hot expansion (members, improved once) + cross GEMM + fresh upper-triangle GEMM"}


def population_rooflines(ph, p, nvpad, steps, peak):
    """HBM-bound population phases ('K0, K1, K4 ... report them, but they are small'): the
    algorithmic bytes each phase must move per generation over its measured time.
    K4a update: gather of the next p x p u16 distance matrix (read + write) and of the next member rows;
    K4b+c offspring: k_match scans its p x p u16 distance rows and exclusion bits, k_crossover reads two
    parent rows and writes one child row per individual."""
    out = {}
    for name, ms, by in (
            ("k4a_update (k_pool_*)", ph["update"] / steps, 4.0 * p * p + 2.0 * p * nvpad),
            ("k4bc_offspring (k_match + k_crossover)", ph["offspring"] / steps,
             2.0 * p * p + p * p / 8.0 + 3.0 * p * nvpad)):
        if ms > 0:
            gbs = by / (ms / 1e3) / 1e9
            out[name] = {"bound": "hbm", "alg_bytes": by, "ms": ms, "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak}
    return out


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_sample(a, ref, grid, gen_seed_offset=0):
    """The reference's improve phase over a bounded slice of the C3 generation-1 population."""
    threads = cpu_threads()
    s = max(threads * a.cpu_per_thread, 1)
    members, _ = ref.init_population(grid, s, a.master_seed)
    nv = members.shape[1]
    budget = a.budget if a.budget > 0 else 100 * nv
    return members, budget, threads, s


def run_reference(a):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    import oracle
    if not oracle.Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libplse_ref.so not built (needs "
                                                              "/root/reference at build time)"}))
        return 0
    ref = oracle.Reference()
    grid = ref.generate_instance(a.n, a.r, a.seed)
    members, budget, threads, s = reference_sample(a, ref, grid)
    mpma = a.variant == "mpma"
    moves = 0
    secs = 0.0
    for step in range(a.warmup + a.steps):
        if mpma:
            it, t = ref.plits_phase(grid, members, a.master_seed, step + 1, a.budget, a.budget2, workers=threads)
        else:
            it, t = ref.improve_phase(grid, members, a.master_seed, step + 1, budget, workers=threads)
        if step >= a.warmup:
            moves += it
            secs += t
    v = moves / secs
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1000 * secs / a.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic (generate_instance(60,0.5,12345), random initial population)",
        "config": {"workload": f"PLSE n={a.n} r={a.r} seed={a.seed}: reference improve phase "
                               + (f"(plits_run, parallel_for) on {s} individuals, budgets 100|V| + 2|V|" if mpma else
                                  f"(partial_mpma_improve, parallel_for) on {s} individuals x {budget} iterations"),
                   "pop_sample": s, "budget": budget, "variant": a.variant},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{s} generation-1 individuals of the C3 population, budget 100|V|, per step",
                         "build": oracle.REF_FLAGS, "lib": os.path.relpath(oracle.REF_LIB, ROOT)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "variant": a.variant,
    }
    print(json.dumps(line))
    return 0


def run_ours(a):
    world, rank, local = dist_env()
    import torch
    # functional check of the multi-rank path on a 1-GPU box (not a measurement): PLSE_BENCH_DIST=gloo
    # moves the elite exchange through host memory, PLSE_BENCH_ONE_GPU=1 puts every rank on device 0
    backend = os.environ.get("PLSE_BENCH_DIST", "nccl")
    one_gpu = os.environ.get("PLSE_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    coll = "cuda" if backend == "nccl" else "cpu"
    import paper_2103_10453_b200 as P
    from paper_2103_10453_b200.islands import DeviceIsland

    grid = lsc_grid(a) if a.lsc else P.generate_instance(a.n, a.r, a.seed)
    graph = P.preprocess(grid)
    nv = graph.vertex_count
    budget = a.budget if a.budget > 0 else 100 * nv
    mpma = a.variant == "mpma"
    if a.weak:
        p_rank = a.pop
    else:
        if a.pop % world:
            raise SystemExit(f"--pop {a.pop} does not split over {world} GPUs")
        p_rank = a.pop // world
    p_total = p_rank * world
    cfg = P.SolverConfig(p=p_rank, master_seed=a.master_seed, phase1_iters=a.budget, device=local,
                         p_total=p_total, offset=p_rank * rank, variant=P.MPMA if mpma else P.PARTIAL,
                         phase2_iters=a.budget2, tie_mode=P.TIE_REF if a.tie == "ref" else P.TIE_CANON)
    pop = P.DevicePopulation(graph, cfg)
    pop.initialize_population()
    pop.offspring = pop.members  # generation-0 offspring are the initial individuals (engine.hpp:163)
    gen = 0
    isl = DeviceIsland(pop, a.elites, rank, world) if world > 1 else None

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    phase = {"improve": 0.0, "distances": 0.0, "update": 0.0, "offspring": 0.0, "k3_ops": 0.0}
    state = {"pending": False}  # the previous generation's population phases are not yet accounted

    def add_phases(c):
        phase["distances"] += c.distances_ms
        phase["update"] += c.update_ms
        phase["offspring"] += c.offspring_ms
        phase["k3_ops"] += c.k3_ops

    def generation():
        """one Partial-MPMA generation; the only host synchronisation is the improve phase's summary
        (iterations, best f).  The population phases' timers of the PREVIOUS generation are read there."""
        nonlocal gen
        gen += 1
        it, bf, bi = pop.improve(gen)
        ctr = pop.counters()
        if state["pending"]:
            add_phases(ctr)
        phase["improve"] += ctr.improve_ms
        if isl is not None and gen % a.migrate_every == 0:
            isl.migrate()
        pop.compute_cross_distances()
        pop.update_population(info=False)
        pop.build_offspring(gen)
        state["pending"] = True
        return it, bf, ctr.improve_ms, ctr.alg_bytes

    # gen-1 improve rate (for the CPU-baseline comparison, same generation as the reference sample)
    gen1 = None
    for w in range(a.warmup):
        it, bf, ims, _ = generation()
        if w == 0:
            gen1 = {"moves": it, "improve_ms": ims, "moves_per_s": it / (ims / 1e3)}

    launches0 = pop.counters().kernel_launches
    for k in phase:
        phase[k] = 0.0
    state["pending"] = False  # the last warm-up generation's phases stay out of the timed totals
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    pop.timer_start()
    moves = 0
    imp_ms = 0.0
    alg_bytes = 0.0
    best = None
    for _ in range(a.steps):
        it, bf, ims, ab = generation()
        moves += it
        imp_ms += ims
        alg_bytes += ab
        best = bf if best is None else min(best, bf)
    ms = pop.timer_stop()
    barrier()
    clk = clocks.stop()
    last = pop.counters()
    add_phases(last)
    launches = last.kernel_launches - launches0
    timed_phase = dict(phase)

    # e2e through the public API with host buffers: H2D offspring, generation, D2H next offspring + stats.
    # The host rows live in pinned memory allocated once, as a serving loop would keep them.
    host_off = torch.empty((p_rank, nv), dtype=torch.int16, pin_memory=True).numpy().view("uint16")
    pop.read_colors(P.OFFSPRING, host_off)
    e2e_moves = 0
    e2e_gen0 = gen + 1
    barrier()
    pop.timer_start()
    t0 = time.perf_counter()
    for _ in range(a.e2e_steps):
        pop.write_colors(P.OFFSPRING, host_off)
        it, _, _, _ = generation()
        e2e_moves += it
        pop.read_colors(P.OFFSPRING, host_off)
        f, c, iters = pop.stats(P.IMPROVED)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    # the same steps on the stream's clock: e2e / this rate is the host-side cost alone, while e2e / value
    # also carries the search's drift between the timed generations and these later ones (more
    # individuals stop early at f = 0 as the population converges; the generation still lasts as long as
    # its full-budget walks)
    e2e_dev_ms = pop.timer_stop()
    h2d = p_rank * nv * 2
    d2h = p_rank * nv * 2 + p_rank * (4 + 4 + 8)

    tot_moves, tot_e2e = moves, e2e_moves
    t_max, e2e_max = ms, e2e_s
    if dist is not None:
        t = torch.tensor([float(moves), float(e2e_moves)], dtype=torch.float64, device=coll)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        tot_moves, tot_e2e = t.tolist()
        m = torch.tensor([ms, e2e_s], dtype=torch.float64, device=coll)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        t_max, e2e_max = m.tolist()

    if rank == 0:
        peak, peak_src = peaks()
        achieved = alg_bytes / (imp_ms / 1e3) / 1e9
        kernel = "k_plits" if mpma else "k_improve"
        key = f"n{a.n}_r{a.r}_s{a.seed}_p{p_rank}_b{budget}" + ("_lsc" if a.lsc else "")
        prof, prof_src = ncu_profile(kernel, key)
        ctr = pop.counters()
        improve_rate = moves / (imp_ms / 1e3)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": prof.get("dram_bytes_per_launch") if prof else None,
                "kernel": kernel, "peak_source": peak_src, "config_key": key,
                "src_hash": kernel_src_hash(kernel), "profile": prof_src,
                "bytes_def": ("DESIGN.md PLITS byte model summed over every step of the launch" if mpma
                              else "SURVEY 8(d) B_t summed over every step of the launch (int16 gamma rows the "
                                   "reference's step reads; this kernel derives gamma from occupancy masks)"),
                "kernel_share_of_step": imp_ms / ms,
                "binding_limit": ("single-warp step latency: from generation 2 on a generation lasts as long as "
                                  "the ~55 individuals that run the whole budget, one lone warp each (DESIGN.md "
                                  "'PLITS kernel'); DRAM traffic is well under 1% of the algorithmic bytes" if mpma
                                  else "instruction issue (the gamma table is never materialised: measured DRAM "
                                       "traffic is well under 1% of the algorithmic bytes; see roofline.issue)")}
        if prof and prof.get("inst_per_move") and clk.get("sm_mhz"):
            peak_inst = 148 * 4 * clk["sm_mhz"] * 1e6
            ach_inst = prof["inst_per_move"] * improve_rate
            roof["issue"] = {"inst_per_move": prof["inst_per_move"], "achieved_warp_inst_per_s": ach_inst,
                             "peak_warp_inst_per_s": peak_inst, "frac": ach_inst / peak_inst,
                             "peak_def": "148 SMs x 4 schedulers x median SM clock under load",
                             "inst_source": prof_src}
        if prof and prof.get("dram_bytes_per_launch") and prof.get("launch_ms"):
            roof["dram_measured"] = {"gbs": prof["dram_bytes_per_launch"] / (prof["launch_ms"] / 1e3) / 1e9,
                                     "frac": prof["dram_bytes_per_launch"] / (prof["launch_ms"] / 1e3) / 1e9 / peak,
                                     "source": prof_src}
        line = {
            "metric": METRIC, "value": tot_moves / (t_max / 1e3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": t_max / a.steps, "higher_is_better": True,
            "scaling": "weak" if a.weak else "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (generate_instance(60,0.5,12345); random initial population, seeds fixed)",
            "config": {"workload": f"PLSE n={a.n} r={a.r} seed={a.seed}" + (" (LSC builder)" if a.lsc else "") + ", "
                                   + ("MPMA (PLITS) generation" if mpma else "Partial-MPMA generation")
                                   + f" (improve+distances+update+offspring), pop {p_total} = {world} x {p_rank}, "
                                   f"budget {budget}" + (" + 2|V|" if mpma else ""),
                       "variant": a.variant, "tie_break": a.tie,
                       "global_batch": p_total, "per_gpu": p_rank, "vertices": nv, "budget": budget,
                       "parallelism": f"islands x{world}" + (f", {a.elites} elites all-gathered every "
                                                             f"{a.migrate_every} gens as pool candidates"
                                                             if world > 1 else ""),
                       "l2": "inputs larger than L2 (distance blocks + tabu scratch per step)",
                       "improve_launch": {"grid": ctr.grid, "threads": ctr.threads, "warps_per_sm": ctr.warps_per_sm,
                                          "smem_bytes": ctr.smem_bytes}},
            "gpu_launches": launches,
            "clocks": clk,
            "roofline": roof,
            "improve_moves_per_s": improve_rate,
            "phase_ms_per_step": {k: v / a.steps for k, v in timed_phase.items() if k != "k3_ops"},
            "k3_roofline": k3_roofline(timed_phase, pop.counters().k3_tensor_cores),
            "population_rooflines": population_rooflines(timed_phase, p_rank, (nv + 15) // 16 * 16, a.steps,
                                                         peak),
            "best_f_seen": best,
            "e2e": {"value": tot_e2e / e2e_max if e2e_max > 0 else None, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": a.e2e_steps,
                    "generations": [e2e_gen0, e2e_gen0 + a.e2e_steps - 1],
                    "timed_generations": [a.warmup + 1, a.warmup + a.steps],
                    "device_rate_same_steps": (e2e_moves / (e2e_dev_ms / 1e3) if world == 1 and e2e_dev_ms > 0
                                               else None),
                    "host": "pinned u16 rows through write_colors / read_colors"},
            "gen1": gen1,
        }
        if world > 1 and (one_gpu or backend != "nccl"):
            line["functional_check"] = (f"{world} ranks on " + ("one GPU" if one_gpu else "separate GPUs") +
                                        f", {backend} exchange: a code-path check, not a measurement")
        if world == 1 and not a.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(a, grid)
        if world == 1 and not a.no_ttb:
            line["time_to_best"] = ttb(a, P, grid)
            line["time_to_best_multi_generation"] = ttb_hard(a)
        print(json.dumps(line))
    pop.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def cpu_baseline(a, grid):
    import oracle
    if not oracle.Reference.available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": "oracle/_ref not built"}
    ref = oracle.Reference()
    members, budget, threads, s = reference_sample(a, ref, grid)
    if a.variant == "mpma":
        it, secs = ref.plits_phase(grid, members, a.master_seed, 1, a.budget, a.budget2, workers=threads)
    else:
        it, secs = ref.improve_phase(grid, members, a.master_seed, 1, budget, workers=threads)
    return {"value": it / secs, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{s} generation-1 individuals of the C3 population (reference init), budget {budget}: "
                      f"{it} moves in {secs:.1f} s",
            "build": oracle.REF_FLAGS, "lib": os.path.relpath(oracle.REF_LIB, ROOT)}


def ttb(a, P, grid):
    """time-to-reference-best: GPU run() at pop 16384 vs the reference run() on all host cores."""
    out = {}
    import oracle
    target = None
    if oracle.Reference.available():
        ref = oracle.Reference()
        r = ref.run(grid, p=a.ttb_ref_pop, seed=a.master_seed, workers=cpu_threads(), time_limit=300.0,
                    variant=0 if a.variant == "mpma" else 1)
        target = r["best_score"]
        out["reference"] = {"pop": a.ttb_ref_pop, "best_score": r["best_score"], "cores": cpu_threads(),
                            "seconds_to_best": r["first_best_seconds"], "generations": r["generations"],
                            "stop": r["stop_reason"]}
    var = P.MPMA if a.variant == "mpma" else P.PARTIAL
    res = P.run(grid, P.SolverConfig(p=a.pop, master_seed=a.master_seed, target_score=float(target or 0),
                                     time_limit=300.0, variant=var))
    out["ours"] = {"pop": a.pop, "best_score": res.best_score, "seconds_to_best": res.time_to_best_seconds,
                   "generations": res.generations, "stop": res.stop_reason, "moves": res.total_iterations,
                   "mode": "parity (every individual runs its full budget)"}
    if target is not None:
        rr = P.run(grid, P.SolverConfig(p=a.pop, master_seed=a.master_seed, target_score=float(target),
                                        race=True, time_limit=300.0, variant=var))
        out["ours_race"] = {"pop": a.pop, "best_score": rr.best_score, "seconds_to_best": rr.time_to_best_seconds,
                            "generations": rr.generations, "stop": rr.stop_reason, "moves": rr.total_iterations,
                            "mode": "race (device-global early exit at the target)"}
    if target is not None:
        # the SAME computation as the reference run: pop 1024, reference tie-break -> identical
        # trajectory, generations and result (tests/test_gpu_refties.py); only the wall time differs
        rx = P.run(grid, P.SolverConfig(p=a.ttb_ref_pop, master_seed=a.master_seed, time_limit=300.0, variant=var,
                                        tie_mode=P.TIE_REF))
        out["ours_same_computation"] = {
            "pop": a.ttb_ref_pop, "tie_break": "reference (bit-exact)", "best_score": rx.best_score,
            "seconds_to_best": rx.time_to_best_seconds, "seconds_total": rx.elapsed_seconds,
            "generations": rx.generations, "moves": rx.total_iterations, "stop": rx.stop_reason,
            "identical_to_reference": (rx.best_score == r["best_score"] and rx.generations == r["generations"]
                                       and rx.total_iterations == r["total_iterations"]),
            "speedup_vs_reference": (r["elapsed_seconds"] / rx.elapsed_seconds) if rx.elapsed_seconds > 0 else None}
        out["reference"]["seconds_total"] = r["elapsed_seconds"]
        out["reference"]["moves"] = r["total_iterations"]
    if target is not None:
        out["target_score"] = target
        out["ours_reached_target"] = res.best_score >= target
    return out


def ttb_hard(a):
    """time to the reference's best where the generational loop matters (n=60 r=0.7: the reference improves
    for 129 generations in 600 s; C4: optimum in generation 13): live with --ttb-hard, otherwise the committed
    run of tools/ttb_hard.py on a B200 of this pool (profiles/r02_ttb_hard.json), summarised."""
    if a.ttb_hard:
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ttb_hard.py"), "--configs", "hard,c4",
                              "--pops", "16384", "--limit", "600"], capture_output=True, text=True, timeout=3600)
        src, d = "live (tools/ttb_hard.py)", json.loads(out.stdout)
    else:
        try:
            with open(os.path.join(ROOT, "profiles", "r02_ttb_hard.json")) as f:
                d = json.load(f)
            src = "profiles/r02_ttb_hard.json (tools/ttb_hard.py on a B200 of this pool)"
        except (OSError, ValueError):
            return None
    rows = []
    for r in d.get("runs", []):
        ref = r.get("reference", {})
        row = {"instance": r["instance"], "target_score": r["target_score"],
               "reference": {k: ref.get(k) for k in ("pop", "best_score", "seconds_to_best", "generations", "cores")}}
        for k, v in r.items():
            if k.startswith("ours_"):
                row[k] = {x: v.get(x) for x in ("pop", "best_score", "seconds_to_best", "generations", "mode",
                                                 "speedup_vs_reference")}
        rows.append(row)
    return {"source": src, "host_threads": d.get("host_threads"), "runs": rows}


def main():
    a = args_()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
