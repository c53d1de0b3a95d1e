"""PartialCol improve probe on any generated instance: N R SEED POP GENS from the environment."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2103_10453_b200 as P

n, r, seed = int(os.environ.get("N", "50")), float(os.environ.get("R", "0.4")), int(os.environ.get("SEED", "12345"))
p, gens = int(os.environ.get("POP", "8192")), int(os.environ.get("GENS", "2"))
grid = P.generate_instance(n, r, seed)
g = P.preprocess(grid)
pop = P.DevicePopulation(g, P.SolverConfig(p=p, master_seed=1, tie_mode=int(os.environ.get("TIE", "0"))))
pop.initialize_population()
pop.offspring = pop.members
for gen in range(1, gens + 1):
    it, bf, bi = pop.improve(gen)
    ctr = pop.counters()
    f, c, iters = pop.stats(P.IMPROVED)
    print(f"gen {gen} |V| {g.vertex_count} moves {it} improve_ms {ctr.improve_ms:.1f} rate {it / ctr.improve_ms * 1e3:.4g} "
          f"best_f {bf} mean_f {f.mean():.2f} iters p50/max {np.percentile(iters, 50):.0f}/{iters.max()}", flush=True)
    pop.compute_cross_distances()
    pop.update_population()
    pop.build_offspring(gen)
