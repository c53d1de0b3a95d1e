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

N > 1 (torchrun): island model -- every rank evolves its own 16384-individual
island (weak scaling), stream index space gen*p_total + rank*p + i, and the
ranks all-gather 32 elites each over NCCL every 2 generations.

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
    ap.add_argument("--pop", type=int, default=16384)
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
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--migrate-every", type=int, default=2)
    ap.add_argument("--elites", type=int, default=32)
    ap.add_argument("--cpu-per-thread", type=int, default=72, help="individuals per host thread in the CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttb", action="store_true")
    ap.add_argument("--ttb-ref-pop", type=int, default=1024)
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


def ncu_traffic(config_key: str):
    """dram bytes per improve launch from the committed ncu --set full summary, if it matches this config."""
    path = os.path.join(ROOT, "profiles", "improve_ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if d.get("config_key") == config_key:
            return d.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    return None


def lsc_grid(a):
    """C5: the order-n LSC stand-in builders::lsc_instance (tests/support/builders.hpp:46-58), restated with
    the library's xoshiro (same stream as the reference builder)."""
    from paper_2103_10453_b200 import lsc_instance
    return lsc_instance(a.n, a.r, a.seed)


def k3_roofline(ph, tensor_cores):
    """similarity GEMM (one-hot i8 tcgen05): algorithmic ops 2*M*N*Kpad per GEMM over the phase time."""
    if ph["distances"] <= 0 or ph["k3_ops"] <= 0:
        return None
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            bf16 = float(json.load(f)["bf16_tflops"])
        src = "2 x measured bf16 burst (i8 dense rate = 2x bf16 on sm_100; i8 not measured by the driver)"
    except (OSError, KeyError, ValueError):
        bf16, src = 1590.0, "2 x fallback bf16 (B200_PROFILING.md)"
    achieved = ph["k3_ops"] / (ph["distances"] / 1e3) / 1e12
    peak = 2 * bf16
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS", "frac": achieved / peak,
            "kernel": "k_onehot + k_sim_tc" if tensor_cores else "k_hamming (CUDA cores)", "peak_source": src,
            "includes": "one-hot expansion of both operands"}


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
        "ms_per_step": 1000 * secs / a.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic (generate_instance(60,0.5,12345), random initial population)",
        "config": {"workload": f"PLSE n={a.n} r={a.r} seed={a.seed}: reference improve phase "
                               + (f"(plits_run, parallel_for) on {s} individuals, budgets 100|V| + 2|V|" if mpma else
                                  f"(partial_mpma_improve, parallel_for) on {s} individuals x {budget} iterations"),
                   "pop_sample": s, "budget": budget, "variant": a.variant},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{s} generation-1 individuals of the C3 population, budget 100|V|, per step"},
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

    grid = lsc_grid(a) if a.lsc else P.generate_instance(a.n, a.r, a.seed)
    graph = P.preprocess(grid)
    nv = graph.vertex_count
    budget = a.budget if a.budget > 0 else 100 * nv
    mpma = a.variant == "mpma"
    cfg = P.SolverConfig(p=a.pop, master_seed=a.master_seed, phase1_iters=a.budget, device=local,
                         p_total=a.pop * world, offset=a.pop * rank, variant=P.MPMA if mpma else P.PARTIAL,
                         phase2_iters=a.budget2, tie_mode=P.TIE_REF if a.tie == "ref" else P.TIE_CANON)
    pop = P.DevicePopulation(graph, cfg)
    pop.initialize_population()
    pop.offspring = pop.members  # generation-0 offspring are the initial individuals (engine.hpp:163)
    gen = 0
    elite_buf = None
    if world > 1:
        elite_buf = torch.empty((world * a.elites, pop.row_bytes), dtype=torch.uint8, device="cuda")
        my_elites = torch.empty((a.elites, pop.row_bytes), dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    phase = {"improve": 0.0, "distances": 0.0, "update": 0.0, "offspring": 0.0, "k3_ops": 0.0}

    def generation():
        nonlocal gen
        gen += 1
        it, bf, bi = pop.improve(gen)
        ctr = pop.counters()
        pop.compute_cross_distances()
        pop.update_population()
        if world > 1 and gen % a.migrate_every == 0:
            pop.export_elites(a.elites, my_elites.data_ptr())
            torch.cuda.synchronize()
            if coll == "cuda":
                dist.all_gather_into_tensor(elite_buf, my_elites)
            else:
                parts = [torch.empty_like(my_elites, device="cpu") for _ in range(world)]
                dist.all_gather(parts, my_elites.cpu())
                elite_buf.copy_(torch.cat(parts).to("cuda"))
            torch.cuda.synchronize()
            others = torch.cat([elite_buf[r * a.elites:(r + 1) * a.elites] for r in range(world) if r != rank])
            torch.cuda.synchronize()  # the library reads `others` on its own stream
            pop.import_migrants(others.shape[0], others.data_ptr())
        pop.build_offspring(gen)
        c2 = pop.counters()
        phase["improve"] += ctr.improve_ms
        phase["distances"] += c2.distances_ms
        phase["update"] += c2.update_ms
        phase["offspring"] += c2.offspring_ms
        phase["k3_ops"] += c2.k3_ops
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
    launches = pop.counters().kernel_launches - launches0

    timed_phase = dict(phase)
    # e2e through the public API with host buffers: H2D offspring, generation, D2H next offspring + stats
    host_off = pop.offspring
    e2e_moves = 0
    barrier()
    t0 = time.perf_counter()
    for _ in range(a.e2e_steps):
        pop.offspring = host_off
        it, _, _, _ = generation()
        e2e_moves += it
        host_off = pop.offspring
        f, c, iters = pop.stats(P.IMPROVED)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    h2d = a.pop * nv * 2
    d2h = a.pop * nv * 2 + a.pop * (4 + 4 + 8)

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
        key = f"n{a.n}_r{a.r}_s{a.seed}_p{a.pop}_b{budget}"
        ctr = pop.counters()
        line = {
            "metric": METRIC, "value": tot_moves / (t_max / 1e3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": t_max / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (generate_instance(60,0.5,12345); random initial population, seeds fixed)",
            "config": {"workload": f"PLSE n={a.n} r={a.r} seed={a.seed}, "
                                   + ("MPMA (PLITS) generation" if mpma else "Partial-MPMA generation")
                                   + f" (improve+distances+update+offspring), pop {a.pop}/GPU, budget {budget}"
                                   + (" + 2|V|" if mpma else ""),
                       "variant": a.variant, "tie_break": a.tie,
                       "global_batch": a.pop * world, "vertices": nv, "budget": budget,
                       "parallelism": f"islands x{world}" + (f", {a.elites} elites all-gathered every "
                                                             f"{a.migrate_every} gens" if world > 1 else ""),
                       "l2": "inputs larger than L2 (1.5 GB distance blocks + tabu scratch per step)",
                       "improve_launch": {"grid": ctr.grid, "threads": ctr.threads, "warps_per_sm": ctr.warps_per_sm,
                                          "smem_bytes": ctr.smem_bytes}},
            "gpu_launches": launches,
            "clocks": clk,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None if mpma else ncu_traffic(key),
                         "kernel": "k_plits" if mpma else "k_improve",
                         "peak_source": peak_src, "config_key": key,
                         "bytes_def": ("DESIGN.md PLITS byte model summed over every step of the launch" if mpma
                                       else "SURVEY 8(d) B_t summed over every step of the launch"),
                         "kernel_share_of_step": imp_ms / ms},
            "improve_moves_per_s": moves / (imp_ms / 1e3),
            "phase_ms_per_step": {k: v / a.steps for k, v in timed_phase.items() if k != "k3_ops"},
            "k3_roofline": k3_roofline(timed_phase, pop.counters().k3_tensor_cores),
            "best_f_seen": best,
            "e2e": {"value": tot_e2e / e2e_max if e2e_max > 0 else None, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": a.e2e_steps},
            "gen1": gen1,
        }
        if world > 1 and (one_gpu or backend != "nccl"):
            line["functional_check"] = (f"{world} ranks on " + ("one GPU" if one_gpu else "separate GPUs") +
                                        f", {backend} exchange: a code-path check, not a measurement")
        if world == 1 and not a.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(a, grid)
        if world == 1 and not a.no_ttb:
            line["time_to_best"] = ttb(a, P, grid)
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
                      f"{it} moves in {secs:.1f} s"}


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


def main():
    a = args_()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
