"""Where the host-buffer pga_batch_run call spends its time (F1 e2e)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import workloads
import paper_1403_4099_b200 as pga

f1 = workloads.F1
B, N, T = f1["B"], f1["N"], f1["T"]
X, _ = workloads.window_returns(B, N, T, f1["seed0"])
dX = torch.from_numpy(X).cuda()
dC = torch.empty((B, N, N), dtype=torch.float64, device="cuda")
st = torch.zeros(B, dtype=torch.int32, device="cuda")
for b in range(B):
    pga.pga_correlation_device(dX[b], dC[b], st[b:b + 1])
torch.cuda.synchronize()
params = pga.pga_params_default(pop_size=f1["pop"], max_gens=f1["gens"], seed=2024)
Cp = torch.from_numpy(dC.cpu().numpy()).pin_memory()
Cn = dC.cpu().numpy()
for name, C in (("pinned", Cp.numpy()), ("pageable", Cn)):
    for r in range(3):
        t0 = time.perf_counter()
        res = pga.pga_batch_run(C, params)
        dt = time.perf_counter() - t0
        print(name, r, "%.1f ms" % (dt * 1e3))
lab = torch.zeros((B, N), dtype=torch.int32, device="cuda")
bL = torch.zeros(B, dtype=torch.float64, device="cuda")
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pga.pga_batch_run_device(dC, params, lab, bL, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize(); print("device", r, "%.1f ms" % ((time.perf_counter() - t0) * 1e3))
