"""PartialCol improve probe: per-generation rate, with PLSE_PROFILE=1 the dense/sparse split."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2103_10453_b200 as P

p = int(os.environ.get("POP", "16384"))
gens = int(os.environ.get("GENS", "3"))
n, r, s = int(os.environ.get("N", "60")), float(os.environ.get("R", "0.5")), int(os.environ.get("S", "12345"))
grid = P.generate_instance(n, r, s)
g = P.preprocess(grid)
variant = P.MPMA if os.environ.get("VARIANT") == "mpma" else P.PARTIAL
pop = P.DevicePopulation(g, P.SolverConfig(p=p, master_seed=1, tie_mode=int(os.environ.get("TIE", "0")),
                                           variant=variant, phase1_iters=int(os.environ.get("BUDGET", "0"))))
pop.initialize_population()
pop.offspring = pop.members
for gen in range(1, gens + 1):
    it, bf, bi = pop.improve(gen)
    ctr = pop.counters()
    f, c, iters = pop.stats(P.IMPROVED)
    q = np.percentile(iters, [50, 90, 99, 99.9, 100]).astype(int).tolist()
    print(f"gen {gen} moves {it} improve_ms {ctr.improve_ms:.1f} rate {it / ctr.improve_ms * 1e3:.4g} best_f {bf} "
          f"iters p50/p90/p99/p99.9/max {q} n_full {(iters >= iters.max()).sum()} mean_f {f.mean():.2f}", flush=True)
    pop.compute_cross_distances()
    pop.update_population()
    pop.build_offspring(gen)
