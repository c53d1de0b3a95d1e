"""The island run (islands.run_islands): at world size 1 it is run()
exactly; at world size 2 (two ranks sharing one B200, elites exchanged over gloo -- no kernel
waits on another rank) every island's final population equals the oracle's island restatement
(tests/island_sim.py) and every rank reports the same global best."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("variant", ["partial", "mpma"])
@pytest.mark.parametrize("n,r,s,p,opt_stop", [(12, 0.5, 4, 24, False), (10, 0.6, 7, 16, True), (16, 0.4, 2, 32, False)])
def test_island_run_world1_equals_run(plse, orc, variant, n, r, s, p, opt_stop):
    from paper_2103_10453_b200 import islands
    grid = orc.generate_instance(n, r, s)
    cfg = plse.SolverConfig(p=p, master_seed=5, phase1_iters=300, generation_limit=3,
                            variant=plse.MPMA if variant == "mpma" else plse.PARTIAL,
                            disable_optimal_stop=not opt_stop)
    want = plse.run(grid, cfg)
    got = islands.run_islands(grid, cfg)
    assert (got.best_f, got.generations, got.total_iterations, got.stop_reason, got.proven_optimal) == \
        (want.best_f, want.generations, want.total_iterations, want.stop_reason, want.proven_optimal)
    assert np.array_equal(got.best_solution, want.best_solution)


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def _worker(rank, world, port, out_dir, cfg):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2103_10453_b200 as P
    from paper_2103_10453_b200 import islands
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid = oracle.Oracle().generate_instance(cfg["n"], cfg["r"], cfg["s"])
    sc = P.SolverConfig(p=cfg["p"], master_seed=cfg["seed"], phase1_iters=cfg["budget"],
                        generation_limit=cfg["gens"] + 1, disable_optimal_stop=True)
    reports = []
    res = islands.run_islands(grid, sc, migrate_every=1, n_elite=cfg["elites"], keep_members=True,
                              on_generation=reports.append)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), members=res.members, best=res.best_solution,
             scalars=np.array([res.best_f, res.generations, res.total_iterations]),
             migrated=np.array([r.migrated for r in reports]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_island_run_matches_island_restatement(orc, tmp_path):
    import torch.multiprocessing as mp
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import island_sim as S

    cfg = dict(n=10, r=0.5, s=3, p=12, seed=21, gens=2, budget=400, elites=3)
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), cfg), nprocs=2, join=True,
                       start_method="spawn")
    grid = orc.generate_instance(cfg["n"], cfg["r"], cfg["s"])
    # generation 3 stops after its improve phase: the populations are those after generation 2
    want = S.simulate(orc, grid, cfg["p"], 2, cfg["seed"], cfg["gens"], cfg["budget"], cfg["elites"])
    outs = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(2)]
    for o, w in zip(outs, want):
        assert np.array_equal(o["members"], w)
        assert o["migrated"].tolist() == [True, True, False]  # the stopping generation reports last
    assert np.array_equal(outs[0]["scalars"], outs[1]["scalars"])
    assert np.array_equal(outs[0]["best"], outs[1]["best"])
    best_f = int(outs[0]["scalars"][0])
    f, c = orc.eval(grid, outs[0]["best"])
    assert (f, c) == (best_f, 0)
    # the global best is at least as good as every island's final legal members
    for w in want:
        fc = np.array([orc.eval(grid, m) for m in w])
        assert best_f <= fc[fc[:, 1] == 0, 0].min()
