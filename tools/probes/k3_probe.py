"""K3 probe: the distance phase at C3 (p = 16384) for an ncu capture of k_onehot / k_sim_tc."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2103_10453_b200 as P

grid = P.generate_instance(60, 0.5, 12345)
g = P.preprocess(grid)
pop = P.DevicePopulation(g, P.SolverConfig(p=16384, master_seed=1, phase1_iters=50))
pop.initialize_population()
pop.offspring = pop.members
pop.improve(1)
for _ in range(2):
    pop.compute_cross_distances()
c = pop.counters()
print(f"distances_ms {c.distances_ms:.2f} k3_ops {c.k3_ops:.3e} tensor_cores {c.k3_tensor_cores} "
      f"TOPS {c.k3_ops / (c.distances_ms / 1e3) / 1e12:.0f}")
