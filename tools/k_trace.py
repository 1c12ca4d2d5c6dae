"""Trace the number of distinct labels K per chromosome over a C4 GA run
(measurement tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
import paper_1403_4099_b200 as pga

X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N = C.shape[0]
P = 65536
params = pga.pga_params_default(pop_size=P, elite=10, p_mutation=2.0 / N, tol=-1.0, max_gens=2000, seed=2024)
ctx = pga.pga_create(C, params)
pga.pga_init(ctx, 2024)
pga.pga_profile_enable(ctx, True)
for g in range(1001):
    if g in (0, 5, 10, 25, 50, 100, 200, 300, 500, 750, 1000):
        lab, L = pga.pga_get_population(ctx, P, N)
        K = lab.max(1)
        nontriv = np.array([np.sum(np.bincount(r)[1:] >= 2) for r in lab[::64]])
        st = pga.pga_get_state(ctx, N)
        pr = pga.pga_profile_read(ctx)
        print("gen %4d  K mean %.1f max %d  clusters(n>=2) mean %.1f  bestL %.3f  ms/gen(last) %.3f sweep %.3f"
              % (g, K.mean(), K.max(), nontriv.mean(), st["best_L"], pr["gen_ms"] / max(1, pr["count"]),
                 pr["sweep_ms"] / max(1, pr["count"])), flush=True)
        pga.pga_profile_enable(ctx, True)
    pga.pga_generation(ctx)
Lp = float(pga.pga_evaluate(ctx, planted[None, :] + 1)[0])
print("planted L", Lp)
