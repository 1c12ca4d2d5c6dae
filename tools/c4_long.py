"""Long C4 run: best L vs the planted partition over many generations."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads, paper_1403_4099_b200 as pga
gens = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N = C.shape[0]
ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=gens, seed=5))
Lp = pga.pga_evaluate(ctx, planted[None, :] + 1)[0]
t = time.time()
r = pga.pga_run(ctx, gens, 5, N)
h = pga.pga_get_history(ctx, gens)
print("planted L %.4f; %.1f s" % (Lp, time.time() - t))
for g in (100, 300, 1000, 3000, 5000, 10000, 20000, 40000):
    if g <= gens:
        print(g, "%.4f" % h[g - 1])
b = r["best_labels"] - 1
print("best == planted:", np.array_equal(b, planted), "best L %.4f" % r["best_L"])
# how far from planted: adjusted counts of genes whose cluster differs
from collections import Counter
pairs = Counter(zip(b.tolist(), planted.tolist()))
print("clusters in best:", len(set(b.tolist())), "planted:", len(set(planted.tolist())))
pga.pga_destroy(ctx)
