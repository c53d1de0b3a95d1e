"""Island model over several GPUs (north star: "the population is sharded across
the GPUs of one 8xB200 box, each GPU evolving its shard, with NCCL all-gather
of the elite or migrant individuals over NVLink every generation block").

One process per GPU.  Rank r of N evolves an island of p individuals with
stream keys gen*p_total + r*p + i (p_total = N*p), so N = 1 is exactly the
reference's single population.  Every `every` generations, after the improve
phase, each rank exports its `n_elite` best members (ascending (illegal, f),
lowest slot first), the ranks all-gather them (NCCL for CUDA tensors, gloo for
CPU tensors), and each rank stages the other ranks' elites, in rank order, as
extra candidates of its next pool: its update_population then
ranks 2p + (N-1)*n_elite candidates (population.hpp:103-183 with pool ids
2p.. for the migrants), so a migrant enters only if it is good and spaced
like any other candidate.  The exchange is the only collective on the data
path; it runs on the population's own CUDA stream (no host synchronisation
for NCCL), and the improve phase and the population phases run locally.
"""
from __future__ import annotations

import dataclasses
import time
from typing import Callable, Optional

import numpy as np


def elite_order(f: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Slots sorted best-first: (illegal, f) ascending, ties by slot (stable)."""
    return np.lexsort((np.arange(len(f)), f, (c != 0).astype(np.int64)))


def allgather_rows(mine, group=None):
    """All-gather equally shaped row blocks; returns (world*rows, width) in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty((world * mine.shape[0],) + tuple(mine.shape[1:]), dtype=mine.dtype, device=mine.device)
    dist.all_gather_into_tensor(out, mine.contiguous(), group=group)
    return out


def others(gathered, rank: int, world: int):
    """Rows of every rank but `rank`, in rank order."""
    import torch
    per = gathered.shape[0] // world
    return torch.cat([gathered[r * per:(r + 1) * per] for r in range(world) if r != rank])


class DeviceIsland:
    """A DevicePopulation shard plus the elite exchange (used by bench.py and run_islands).

    `migrate()` is called between the improve phase and update_population: export (device sort of the
    members) -> all-gather -> stage the other ranks' elites as pool candidates.  Everything is ordered on
    the population's CUDA stream: for NCCL the collective is issued with that stream current, so no host
    synchronisation happens; for gloo the rows cross host memory."""

    def __init__(self, pop, n_elite: int, rank: int, world: int, group=None):
        import torch
        import torch.distributed as dist
        self.pop, self.n_elite, self.rank, self.world, self.group = pop, n_elite, rank, world, group
        self.mine = torch.empty((n_elite, pop.row_bytes), dtype=torch.uint8, device="cuda")
        self.gathered = torch.empty((world * n_elite, pop.row_bytes), dtype=torch.uint8, device="cuda")
        self.rest = torch.empty(((world - 1) * n_elite, pop.row_bytes), dtype=torch.uint8, device="cuda")
        self.nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"
        self.stream = torch.cuda.ExternalStream(pop.stream)

    def migrate(self) -> None:
        import torch
        import torch.distributed as dist
        if self.world < 2:
            return
        per = self.n_elite
        with torch.cuda.stream(self.stream):
            self.pop.export_elites(per, self.mine.data_ptr())
            if self.nccl:
                dist.all_gather_into_tensor(self.gathered, self.mine, group=self.group)
            else:
                host = torch.empty((self.world * per, self.mine.shape[1]), dtype=torch.uint8)
                dist.all_gather_into_tensor(host, self.mine.cpu(), group=self.group)
                self.gathered.copy_(host)
            k = 0
            for r in range(self.world):
                if r != self.rank:
                    self.rest[k * per:(k + 1) * per].copy_(self.gathered[r * per:(r + 1) * per])
                    k += 1
            self.pop.import_migrants(self.rest.shape[0], self.rest.data_ptr())


def exchange_host(islands_members, islands_f, islands_c, n_elite: int):
    """Sequential restatement of one exchange over all islands (the reference for the N>1 tests): for
    every rank, the other ranks' n_elite best members in rank order -- the extra pool candidates of its
    next update."""
    world = len(islands_members)
    elites = [m[elite_order(f, c)[:n_elite]] for m, f, c in zip(islands_members, islands_f, islands_c)]
    return [np.concatenate([elites[q] for q in range(world) if q != r]) if world > 1 else elites[0][:0]
            for r in range(world)]


def stream_coords(rank: int, world: int, p: int, total: Optional[int] = None):
    """(p_total, offset) of a rank's island."""
    return (total or p * world), rank * p


# ------------------------------------------------------------------ the island run (engine.hpp:114-262 per island)
@dataclasses.dataclass
class GenerationReport:
    """One generation of an island run, global over the ranks (rank 0's view)."""
    generation: int
    best_f: int            # global best f so far
    iterations: int        # tabu moves of this generation, summed over the ranks
    total_iterations: int  # summed over the ranks and generations
    elapsed_seconds: float  # max over the ranks
    migrated: bool


def reduce_generation(best_f: int, iterations: int, elapsed: float, group=None, device="cpu"):
    """The per-generation collective of the island run (all-reduce(min) of the best f and
    the stop inputs): returns (global best f, lowest rank holding it, summed iterations, max elapsed)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    key = torch.tensor([best_f * world + rank], dtype=torch.int64, device=device)
    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    it = torch.tensor([iterations], dtype=torch.int64, device=device)
    dist.all_reduce(it, op=dist.ReduceOp.SUM, group=group)
    el = torch.tensor([elapsed], dtype=torch.float64, device=device)
    dist.all_reduce(el, op=dist.ReduceOp.MAX, group=group)
    k = int(key.item())
    return k // world, k % world, int(it.item()), float(el.item())


def run_islands(grid: np.ndarray, config, migrate_every: int = 2, n_elite: int = 32, group=None,
                on_generation: Optional[Callable[[GenerationReport], None]] = None, keep_members: bool = False):
    """The north star's island model as a run: one process per GPU, each evolving a p-individual island
    of the Partial-MPMA generation (engine.hpp:114-262) with stream keys gen*p_total + rank*p + i; every
    `migrate_every` generations, after the improve phase, the ranks all-gather their `n_elite` best
    members (NCCL for the nccl backend, host tensors for gloo) and each ranks the others' elites as extra
    candidates of its pool update (DeviceIsland); every generation
    the best f, the iteration count and the elapsed time are all-reduced so that every rank takes the
    same stop decision (optimal / time / iterations / generations / target, engine.hpp:215-236), and
    the rank holding a new global best broadcasts its colouring.  With torch.distributed not
    initialised (or world size 1) this is exactly `run()`: same colourings, iterations and stop.

    `config` is a SolverConfig whose `p` is the island size (p_total / offset are set here).  The time
    limit is checked between generations (run() also cuts an improve phase at its device deadline).
    Returns the global RunResult on every rank (best_solution broadcast from its owner), and with
    `keep_members` the island's final population as `.members`.
    """
    import torch
    import torch.distributed as dist
    import paper_2103_10453_b200 as P

    on = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if on else 1
    rank = dist.get_rank(group) if on else 0
    coll = "cuda" if on and dist.get_backend(group) == "nccl" else "cpu"
    t0 = time.monotonic()
    grid = np.ascontiguousarray(grid, np.uint16)
    n = grid.shape[0]
    graph = P.preprocess(grid)
    nv, l = graph.vertex_count, graph.l
    p = config.p
    cfg = dataclasses.replace(config, p_total=p * world, offset=p * rank)
    is_opt = (lambda f: f == 1) if l == 1 else (lambda f: f == 0)
    upper = n * n - 2 if l == 1 else n * n - l

    def result(best_f, best, reason, gens, total, ttb, members=None):
        proven = is_opt(best_f)
        out = P.RunResult(best_f, n * n - l - best_f, proven, "optimal" if proven else reason, l, upper, nv, gens,
                          total, time.monotonic() - t0, ttb, best)
        if keep_members:
            out.members = members
        return out

    if nv == 0:
        return result(0, np.zeros(0, np.uint16), "trivial", 0, 0, 0.0)

    def glob(local_f, local_it):
        el = time.monotonic() - t0
        if not on or world == 1:
            return local_f, 0, local_it, el
        return reduce_generation(local_f, local_it, el, group, "cuda" if coll == "cuda" else "cpu")

    best = np.zeros(nv, np.uint16)
    best_f, ttb = nv, 0.0

    def take_best(f_new, owner, row):
        """row: this rank's candidate (None unless rank == owner); broadcast from the owner"""
        nonlocal best, best_f, ttb
        if on and world > 1:
            buf = torch.zeros(nv, dtype=torch.int32, device=coll)
            if rank == owner:
                buf.copy_(torch.from_numpy(row.astype(np.int32)))
            dist.broadcast(buf, src=dist.get_global_rank(group, owner) if group is not None else owner, group=group)
            row = buf.cpu().numpy()
        best = np.asarray(row, np.uint16).copy()
        best_f = f_new
        ttb = time.monotonic() - t0

    with P.DevicePopulation(graph, cfg) as pop:
        pop.initialize_population()
        f, c, _ = pop.stats(P.MEMBERS)
        legal = np.flatnonzero(c == 0)
        loc = int(legal[np.argmin(f[legal])]) if legal.size else -1
        lf = int(f[loc]) if loc >= 0 else nv
        gf, owner, _, _ = glob(lf, 0)
        if gf < best_f:
            take_best(gf, owner, pop.read_row(P.MEMBERS, loc) if rank == owner else None)
        members = lambda: pop.members if keep_members else None
        if not config.disable_optimal_stop and is_opt(best_f):
            return result(best_f, best, "optimal", 0, 0, ttb, members())
        pop.offspring = pop.members
        pop.reset_exclusion()
        isl = DeviceIsland(pop, n_elite, rank, world, group) if world > 1 else None
        total = 0
        gen = 0
        while True:
            gen += 1
            it, bf, bi = pop.improve(gen)
            gf, owner, git, el = glob(bf if bi >= 0 else nv, it)
            total += git
            if gf < best_f:
                take_best(gf, owner, pop.read_row(P.IMPROVED, bi) if rank == owner else None)
            optimal = not config.disable_optimal_stop and is_opt(best_f)
            time_up = config.time_limit > 0 and el >= config.time_limit
            iters_up = config.iteration_limit > 0 and total >= config.iteration_limit
            gens_up = config.generation_limit > 0 and gen >= config.generation_limit
            target = config.target_score > 0 and (n * n - l - best_f) >= config.target_score
            if optimal or time_up or iters_up or gens_up or target:
                reason = ("optimal" if optimal else "time_limit" if time_up else "iteration_limit" if iters_up
                          else "generation_limit" if gens_up else "target")
                if on_generation:
                    on_generation(GenerationReport(gen, best_f, git, total, el, False))
                return result(best_f, best, reason, gen, total, ttb, members())
            migrated = world > 1 and migrate_every > 0 and gen % migrate_every == 0
            if migrated:
                isl.migrate()
            pop.compute_cross_distances()
            pop.update_population(info=False)
            if cfg.exclusion == P.GENERATION:
                pop.reset_exclusion()
            pop.build_offspring(gen)
            if on_generation:
                on_generation(GenerationReport(gen, best_f, git, total, el, migrated))
