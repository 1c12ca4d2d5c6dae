"""Bench-like C4 run (IslandRunner, migration every 10 with one island) and
an oracle check of the best-ever chromosome and of the best L history."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, oracle, paper_1403_4099_b200 as pga
from paper_1403_4099_b200.islands import GpuIsland, IslandRunner

X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N, P, G = 500, 65536, int(sys.argv[1]) if len(sys.argv) > 1 else 1005
mig = int(sys.argv[2]) if len(sys.argv) > 2 else 10
params = pga.pga_params_default(pop_size=P, elite=10, p_mutation=2.0 / N, tol=-1.0, max_gens=G + 10,
                                migrate_every=mig, migrants=10, seed=2024)
eng = GpuIsland(C, params)
run = IslandRunner(eng)
eng.init(2024)
run.run(G)
torch.cuda.synchronize()
st = eng.state()
h = pga.pga_get_history(eng.ctx, G)
Lb, _ = oracle.log_likelihood(C, st["best_labels"] - 1)
print("gens %d migrate_every %d: state best_L %.6f, oracle L of best labels %.6f" % (G, mig, st["best_L"], Lb))
jumps = np.where(np.diff(h) > 50)[0]
print("history: L[0]=%.3f L[100]=%.3f L[500]=%.3f L[-1]=%.3f; jumps > 50 at %s" % (h[0], h[100], h[500], h[-1], jumps[:10]))
pop, L = pga.pga_get_population(eng.ctx, P, N)
i = int(np.argmax(L))
Lo, _ = oracle.evaluate(C, pop[i:i + 1] - 1)
print("population max L %.6f (idx %d), oracle %.6f" % (L[i], i, Lo[0]))
eng.close()
