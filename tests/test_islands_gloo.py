"""N > 1 island path with world_size 2 over gloo on CPU:
each rank evolves its island with the oracle and exchanges elites through
torch.distributed (the same all-gather bench.py does over NCCL); the result
must equal the sequential island restatement."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, cfg):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import island_sim as S
    import oracle
    from paper_2103_10453_b200 import islands

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.Oracle()
    grid = orc.generate_instance(cfg["n"], cfg["r"], cfg["s"])
    st = S.island_init(orc, grid, cfg["p"], cfg["seed"], rank, world)
    for gen in range(1, cfg["gens"] + 1):
        imp = S.island_improve(orc, grid, st, cfg["seed"], gen, cfg["budget"])
        # the exchange: this island's best members (before its update) all-gathered; the others' elites
        # become extra candidates of this island's pool
        f, c = S.fc(orc, grid, st["members"])
        mine = torch.from_numpy(st["members"][islands.elite_order(f, c)[:cfg["elites"]]].astype(np.int32))
        gathered = islands.allgather_rows(mine)
        incoming = islands.others(gathered, rank, world).numpy().astype(np.uint16)
        S.island_update(orc, grid, st, imp, incoming)
        S.island_offspring(orc, grid, st, cfg["seed"], gen)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), st["members"])
    dist.barrier()
    dist.destroy_process_group()


def test_two_islands_over_gloo_match_sequential_restatement(tmp_path, orc):
    import torch.multiprocessing as mp
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import island_sim as S

    cfg = dict(n=10, r=0.5, s=3, p=12, seed=21, gens=3, budget=400, elites=3)
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), cfg), nprocs=2, join=True,
                       start_method="spawn")
    got = [np.load(tmp_path / f"rank{r}.npy") for r in range(2)]
    grid = orc.generate_instance(cfg["n"], cfg["r"], cfg["s"])
    want = S.simulate(orc, grid, cfg["p"], 2, cfg["seed"], cfg["gens"], cfg["budget"], cfg["elites"])
    for g_, w_ in zip(got, want):
        assert np.array_equal(g_, w_)
    # islands exchanged genetic material: each island holds the other's elites after generation 1
    assert not np.array_equal(got[0], got[1])


def test_single_island_is_the_reference_population(orc):
    """N = 1: stream coordinates reduce to the reference's (gen*p + i) keying"""
    from paper_2103_10453_b200 import islands
    assert islands.stream_coords(0, 1, 64) == (64, 0)
    grid = orc.generate_instance(10, 0.5, 3)
    a = orc.init_population(grid, 8, 5)
    b = orc.init_population(grid, 8, 5, offset=0)
    assert np.array_equal(a, b)


def test_elite_order_and_exchange():
    from paper_2103_10453_b200 import islands
    f = np.array([5, 3, 3, 9, 1])
    c = np.array([0, 0, 0, 0, 2])
    assert islands.elite_order(f, c).tolist() == [1, 2, 0, 3, 4]
    m = [np.arange(10).reshape(5, 2) + 100 * r for r in range(3)]
    inc = islands.exchange_host(m, [f] * 3, [c] * 3, 2)
    assert [x[:, 0].tolist() for x in inc] == [[102, 104, 202, 204], [2, 4, 202, 204], [2, 4, 102, 104]]


def test_update_with_migrants_extends_the_pool(orc):
    """A migrant better than every pool member enters first; with none the update is the reference's."""
    grid = orc.generate_instance(10, 0.5, 3)
    p = 8
    mem = orc.init_population(grid, p, 5)
    dist = orc.full_distances(mem)
    imp = np.stack([orc.improve(grid, mem[i], orc.derive_seed(5, 2, p + i), 300, tie=0)["best"] for i in range(p)])
    cr, fr = orc.cross_distances(mem, imp)
    base = orc.update(grid, mem, dist, imp, cr, fr)
    same = orc.update(grid, mem, dist, imp, cr, fr, migrants=np.zeros((0, mem.shape[1]), np.uint16))
    assert np.array_equal(base["members"], same["members"]) and np.array_equal(base["dist"], same["dist"])
    best = orc.improve(grid, imp[0], orc.derive_seed(9, 2, 0), 5000, tie=0)["best"]
    fb, _ = orc.eval(grid, best)
    if fb < base["pool_best_f"]:
        u = orc.update(grid, mem, dist, imp, cr, fr, migrants=best[None, :])
        assert u["selected"][0] == 2 * p and np.array_equal(u["members"][0], best)
        assert u["pool_best_f"] == fb
    # distances of the new population stay consistent with its rows
    u = orc.update(grid, mem, dist, imp, cr, fr, migrants=imp[:3][::-1].copy())
    assert np.array_equal(u["dist"], orc.full_distances(u["members"]))


def _reduce_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2103_10453_b200 import islands

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # ranks 1 and 2 tie on the best f: the lowest rank owns it
    best_f = [9, 4, 4][rank]
    out = islands.reduce_generation(best_f, 100 * (rank + 1), 0.5 + rank, None, "cpu")
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(out, dtype=np.float64))
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_generation_over_gloo(tmp_path):
    """The island run's per-generation collective: global best f, its lowest owning rank, summed
    iterations, max elapsed -- identical on every rank."""
    import torch.multiprocessing as mp
    mp.start_processes(_reduce_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True,
                       start_method="spawn")
    for r in range(3):
        assert np.load(os.path.join(tmp_path, f"r{r}.npy")).tolist() == [4, 1, 600, 2.5]
