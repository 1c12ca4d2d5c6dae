"""Whole-run time of C4 (5000 generations from random init) per sparse threshold.
argv: [G] [theta,theta,...] [cache|nocache]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_1403_4099_b200 as pga
X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N, P, G = 500, 65536, int(sys.argv[1]) if len(sys.argv) > 1 else 5000
for theta in [float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "0.02", "0.04", "0.07", "0.1"])]:
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=G, seed=5))
    pga.pga_set_sparse_threshold(ctx, theta)
    pga.pga_set_cluster_cache(ctx, not (len(sys.argv) > 3 and sys.argv[3] == "nocache"))
    pga.pga_profile_enable(ctx, 1)
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = pga.pga_run(ctx, G, 5, N)
    dt = time.perf_counter() - t
    h = pga.pga_get_history(ctx, G)
    pr = pga.pga_profile_read(ctx)
    hits, saved = pga.pga_profile_cache(ctx)
    blocks, gathered = pga.pga_profile_sparse(ctx)
    print("theta %.3f: %d gens %.3f s (%.3f ms/gen), best L %.4f, L@%d %.3f, sparse blocks %d, gathered %.3g, "
          "cache hits %d saving %.3g pairs" % (theta, G, dt, 1e3 * dt / G, r["best_L"], min(G, 1000),
                                               h[min(G, 1000) - 1], blocks, gathered, hits, saved), flush=True)
    pga.pga_destroy(ctx)
