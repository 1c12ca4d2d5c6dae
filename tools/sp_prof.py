import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import workloads, paper_1403_4099_b200 as pga
X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N, P = 500, 65536
ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P))
rng = np.random.default_rng(1)
L = torch.zeros(P, dtype=torch.float64, device="cuda")
lab = torch.from_numpy(rng.integers(0, 250, size=(P, N)).astype(np.int16)).cuda()
pga.pga_set_sparse_threshold(ctx, 1.0)
for r in range(2):
    pga.pga_evaluate_device(ctx, lab, L)
torch.cuda.synchronize()
