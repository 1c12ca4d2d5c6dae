"""Mean label sparsity of the C4 population over a run: sum_s n_s^2 / N^2
(the work of a label-sparse evaluation relative to the dense sweep)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads, paper_1403_4099_b200 as pga
X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N, P = 500, 65536
ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=6000, seed=5))
pga.pga_init(ctx, 5)
done = 0
for g in (0, 5, 20, 50, 100, 200, 500, 1000, 2000, 5000):
    while done < g:
        pga.pga_gen_evaluate(ctx)
        pga.pga_gen_breed(ctx)
        done += 1
    pop, _ = pga.pga_get_population(ctx, P, N)
    sub = pop[::64] - 1
    s2 = np.array([np.bincount(r, minlength=N).astype(np.int64) @ np.bincount(r, minlength=N) for r in sub])
    print("gen %5d: mean sum n_s^2 / N^2 = %.4f (min %.4f max %.4f)" % (g, s2.mean() / N**2, s2.min() / N**2, s2.max() / N**2))
pga.pga_destroy(ctx)
