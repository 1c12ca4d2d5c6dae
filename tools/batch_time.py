"""Time the batched GA (pga_batch_run, device path) on the F1 windows.

python tools/batch_time.py [--B 1760] [--pop 1000] [--gens 400] [--reps 3]
Prints matrices/s, generations run, and how often the planted partition is
the GA's best (C by the product's own pga_correlation_device)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
import paper_1403_4099_b200 as pga  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=workloads.F1["B"])
    ap.add_argument("--N", type=int, default=workloads.F1["N"])
    ap.add_argument("--pop", type=int, default=workloads.F1["pop"])
    ap.add_argument("--gens", type=int, default=workloads.F1["gens"])
    ap.add_argument("--tol", type=float, default=1e-5)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    X, planted = workloads.window_returns(a.B, a.N, workloads.F1["T"])
    dX = torch.from_numpy(X).cuda()
    dC = torch.empty((a.B, a.N, a.N), dtype=torch.float64, device="cuda")
    st = torch.zeros(a.B, dtype=torch.int32, device="cuda")
    for b in range(a.B):
        pga.pga_correlation_device(dX[b], dC[b], st[b:b + 1])
    torch.cuda.synchronize()
    assert int(st.sum()) == 0
    p = pga.pga_params_default(pop_size=a.pop, max_gens=a.gens, tol=a.tol, seed=1)
    lab = torch.zeros((a.B, a.N), dtype=torch.int32, device="cuda")
    bl = torch.zeros(a.B, dtype=torch.float64, device="cuda")
    gens = torch.zeros(a.B, dtype=torch.int32, device="cuda")
    print("smem/CTA", pga.pga_batch_smem_bytes(a.N, a.pop, p.elite))
    times = []
    for r in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pga.pga_batch_run_device(dC, p, lab, bl, gens, stream=torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    g = gens.cpu().numpy()
    same = np.mean([np.array_equal(lab[b].cpu().numpy() - 1, planted[b]) for b in range(a.B)])
    print("B=%d N=%d P=%d: %.2f ms per batch -> %.1f matrices/s; gens mean %.1f max %d; "
          "planted==best %.3f; evals/s %.3g" % (a.B, a.N, a.pop, ms, a.B / ms * 1e3, g.mean(), g.max(),
                                               same, g.sum() * a.pop / ms * 1e3))


if __name__ == "__main__":
    main()
