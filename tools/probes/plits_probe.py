"""PLITS steady-state probe: per-individual iteration histogram and improve time per generation."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2103_10453_b200 as P

p = int(os.environ.get("POP", "16384"))
gens = int(os.environ.get("GENS", "4"))
grid = P.generate_instance(60, 0.5, 12345)
g = P.preprocess(grid)
pop = P.DevicePopulation(g, P.SolverConfig(p=p, master_seed=1, variant=P.MPMA, tie_mode=int(os.environ.get("TIE", "0"))))
pop.initialize_population()
pop.offspring = pop.members
for gen in range(1, gens + 1):
    it, bf, bi = pop.improve(gen)
    ctr = pop.counters()
    f, c, iters = pop.stats(P.IMPROVED)
    q = np.percentile(iters, [50, 90, 99, 99.9, 100])
    print(f"gen {gen} moves {it} improve_ms {ctr.improve_ms:.1f} rate {it / ctr.improve_ms * 1e3:.3g} best_f {bf} "
          f"iters p50/p90/p99/p99.9/max {q.astype(int).tolist()} n_full {(iters >= 180000).sum()} "
          f"mean_f {f.mean():.2f}", flush=True)
    pop.compute_cross_distances()
    pop.update_population()
    pop.build_offspring(gen)
