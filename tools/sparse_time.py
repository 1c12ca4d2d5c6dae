"""Time the fitness path (dense vs label-sparse) on C4-size populations of
given sparsity: uniform labels over [0, K)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_1403_4099_b200 as pga
X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N, P = 500, 65536
ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P))
rng = np.random.default_rng(1)
L = torch.zeros(P, dtype=torch.float64, device="cuda")
for K in (500, 250, 100, 50, 30, 20):
    lab = torch.from_numpy(rng.integers(0, K, size=(P, N)).astype(np.int16)).cuda()
    s2 = np.mean([np.bincount(r, minlength=N) @ np.bincount(r, minlength=N) for r in lab[:64].cpu().numpy().astype(np.int64)]) / N**2
    out = []
    for theta in (0.0, 1.0):
        pga.pga_set_sparse_threshold(ctx, theta)
        ts = []
        st = torch.cuda.Stream()
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record(st)
                pga.pga_evaluate_device(ctx, lab, L, stream=st.cuda_stream)
                e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out.append(np.median(ts[1:]))
    print("K=%3d sum n^2/N^2 = %.4f: dense %.3f ms, sparse %.3f ms" % (K, s2, out[0], out[1]))
pga.pga_destroy(ctx)
# sanity: device results vs host path on a few rows
ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P))
lab = torch.from_numpy(rng.integers(0, 50, size=(P, N)).astype(np.int16)).cuda()
for theta in (0.0, 1.0):
    pga.pga_set_sparse_threshold(ctx, theta)
    pga.pga_evaluate_device(ctx, lab, L)
    torch.cuda.synchronize()
    print(theta, L[:4].cpu().numpy(), pga.pga_evaluate(ctx, lab[:4].cpu().numpy().astype(np.int32) + 1))
pga.pga_destroy(ctx)
