"""CPU restatement of the island model on top of the oracle.

TEST INFRASTRUCTURE: used by tests/test_islands_gloo.py (world_size 2 over gloo)
and tests/test_gpu_parity.py (two device islands on one GPU)."""
import numpy as np

import oracle
from paper_2103_10453_b200 import islands


def island_init(orc, grid, p, seed, rank, world):
    mem = orc.init_population(grid, p, seed, offset=rank * p)
    return {"members": mem, "dist": orc.full_distances(mem), "offspring": mem.copy(),
            "excl": np.zeros((p, p), np.uint8), "rank": rank, "world": world, "p": p}


def island_improve(orc, grid, st, seed, gen, budget):
    p, world, rank = st["p"], st["world"], st["rank"]
    g = orc.preprocess(grid)
    stop_f = 1 if g.l == 1 else 0
    return np.stack([orc.improve(grid, st["offspring"][i], orc.derive_seed(seed, 2, gen * p * world + rank * p + i),
                                 budget, stop_f=stop_f, tie=oracle.TIE_CANON)["best"] for i in range(p)])


def island_update(orc, grid, st, imp, migrants=None):
    """population.hpp:103-183 with the migrants as extra pool candidates (ids 2p..)"""
    cr, fr = orc.cross_distances(st["members"], imp)
    u = orc.update(grid, st["members"], st["dist"], imp, cr, fr, migrants=migrants)
    st["members"], st["dist"] = u["members"], u["dist"]
    return u


def fc(orc, grid, members):
    out = np.array([orc.eval(grid, m) for m in members], np.int64)
    return out[:, 0], out[:, 1]


def island_offspring(orc, grid, st, seed, gen):
    p, world, rank = st["p"], st["world"], st["rank"]
    st["offspring"], _ = orc.offspring_ex(grid, st["members"], st["dist"], st["excl"], seed, gen * p * world + rank * p)


def simulate(orc, grid, p, world, seed, gens, budget, n_elite, every=1):
    """all islands sequentially in one process: improve, then (every `every` generations) the elite
    exchange staged as pool candidates, then update and offspring"""
    sts = [island_init(orc, grid, p, seed, r, world) for r in range(world)]
    for gen in range(1, gens + 1):
        imps = [island_improve(orc, grid, st, seed, gen, budget) for st in sts]
        incoming = [None] * world
        if world > 1 and every > 0 and gen % every == 0:
            fcs = [fc(orc, grid, st["members"]) for st in sts]
            incoming = islands.exchange_host([st["members"] for st in sts], [x[0] for x in fcs],
                                             [x[1] for x in fcs], n_elite)
        for st, imp, inc in zip(sts, imps, incoming):
            island_update(orc, grid, st, imp, inc)
        for st in sts:
            island_offspring(orc, grid, st, seed, gen)
    return [st["members"] for st in sts]
