"""Timed C4 generations: cached graphs (profiling off) vs plain launches with
the bench's profiling events (profiling on).  Same seed, same population."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_1403_4099_b200 as pga
from paper_1403_4099_b200.islands import GpuIsland, IslandRunner

X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 500
for prof in (1, 0, 1, 0):
    params = pga.pga_params_default(pop_size=65536, p_mutation=2.0 / 500, tol=-1.0, max_gens=10 ** 6, seed=5)
    eng = GpuIsland(C, params)
    r = IslandRunner(eng)
    eng.init(5)
    for _ in range(5):
        r.step()
    pga.pga_profile_enable(eng.ctx, prof)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    for _ in range(K):
        r.step()
    e1.record(eng.stream)
    torch.cuda.synchronize()
    print("prof" if prof else "graph", e0.elapsed_time(e1) / K, "ms/gen", "best", eng.state()["best_L"], flush=True)
    eng.close()
