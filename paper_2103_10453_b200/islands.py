"""Island model over several GPUs (north star: "the population is sharded across
the GPUs of one 8xB200 box, each GPU evolving its shard, with NCCL all-gather
of the elite or migrant individuals over NVLink every generation block").

One process per GPU.  Rank r of N evolves an island of p individuals with
stream keys gen*p_total + r*p + i (p_total = N*p), so N = 1 is exactly the
reference's single population.  Every `every` generations each rank exports
its `n_elite` best members (ascending (illegal, f), lowest slot first), the
ranks all-gather them (NCCL for CUDA tensors, gloo for CPU tensors), and each
rank replaces its worst (N-1)*n_elite members -- descending (illegal, f, slot)
-- by the other ranks' elites in rank order, then recomputes its distance
matrix.  The exchange is the only collective on the path; the improve phase
and the population phases run locally.
"""
from __future__ import annotations

from typing import Optional

import numpy as np


def elite_order(f: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Slots sorted best-first: (illegal, f) ascending, ties by slot (stable)."""
    return np.lexsort((np.arange(len(f)), f, (c != 0).astype(np.int64)))


def victim_order(f: np.ndarray, c: np.ndarray) -> np.ndarray:
    """Slots sorted worst-first: (illegal, f, slot) descending."""
    return np.lexsort((np.arange(len(f)), f, (c != 0).astype(np.int64)))[::-1]


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
    """A DevicePopulation shard plus the NCCL elite exchange (used by bench.py)."""

    def __init__(self, pop, n_elite: int, rank: int, world: int, group=None):
        import torch
        self.pop, self.n_elite, self.rank, self.world, self.group = pop, n_elite, rank, world, group
        self.mine = torch.empty((n_elite, pop.row_bytes), dtype=torch.uint8, device="cuda")

    def migrate(self) -> None:
        import torch
        self.pop.export_elites(self.n_elite, self.mine.data_ptr())
        torch.cuda.synchronize()
        gathered = allgather_rows(self.mine, self.group)
        torch.cuda.synchronize()
        rest = others(gathered, self.rank, self.world).contiguous()
        self.pop.import_migrants(rest.shape[0], rest.data_ptr())


def migrate_host(members: np.ndarray, f: np.ndarray, c: np.ndarray, incoming: np.ndarray) -> np.ndarray:
    """Host restatement of plse_import_migrants: the worst len(incoming) slots take the migrants."""
    out = members.copy()
    victims = victim_order(f, c)[:len(incoming)]
    for k, slot in enumerate(victims):
        out[slot] = incoming[k]
    return out


def exchange_host(islands_members, islands_f, islands_c, n_elite: int):
    """Sequential restatement of one exchange over all islands (the reference for the N>1 tests)."""
    world = len(islands_members)
    elites = [m[elite_order(f, c)[:n_elite]] for m, f, c in zip(islands_members, islands_f, islands_c)]
    out = []
    for r in range(world):
        incoming = np.concatenate([elites[q] for q in range(world) if q != r]) if world > 1 else elites[0][:0]
        out.append(migrate_host(islands_members[r], islands_f[r], islands_c[r], incoming))
    return out


def stream_coords(rank: int, world: int, p: int, total: Optional[int] = None):
    """(p_total, offset) of a rank's island."""
    return (total or p * world), rank * p
