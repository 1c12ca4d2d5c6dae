import sys; sys.path.insert(0,'/root/repo')
import numpy as np, workloads, oracle as orc
import paper_1403_4099_b200 as pga
X, planted = workloads.noh_returns(workloads.CONFIGS["C3"])
C = pga.pga_correlation(X); N=100
params = pga.pga_params_default(pop_size=4096, max_gens=2000, tol=-1.0, seed=1, p_mutation=0.02)
ctx = pga.pga_create(C, params)
r = pga.pga_run(ctx, 2000, 1, N)
b = r["best_labels"]-1
print("best L", repr(r["best_L"]), "K", b.max()+1)
print("planted", planted.tolist())
print("best   ", b.tolist())
Lb,_ = orc.log_likelihood(C, b); Lp,_=orc.log_likelihood(C, planted)
print("oracle L best", repr(Lb), "planted", repr(Lp))
n,c = orc.cluster_stats(C,b); print("n", n.tolist()); print("c", np.round(c,3).tolist())
