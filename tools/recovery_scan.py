"""Planted-cluster recovery vs generation budget on the GPU (measurement tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads
import paper_1403_4099_b200 as pga

def scan(cfg, P, gens_list, seeds, pm=None):
    X, planted = workloads.noh_returns(workloads.CONFIGS[cfg])
    C = pga.pga_correlation(X)
    N = C.shape[0]
    Lp = float(pga.pga_evaluate(pga.pga_create(C, pga.pga_params_default(pop_size=16, elite=2)), planted[None] + 1)[0])
    for G in gens_list:
        rec = 0; Ls = []; t = time.time()
        for seed in seeds:
            params = pga.pga_params_default(pop_size=P, max_gens=G, tol=-1.0, seed=seed,
                                            p_mutation=(pm if pm is not None else 2.0 / N))
            ctx = pga.pga_create(C, params)
            r = pga.pga_run(ctx, G, seed, N)
            pga.pga_destroy(ctx)
            rec += np.array_equal(r["best_labels"] - 1, planted)
            Ls.append(r["best_L"])
        print("%s P=%d gens=%d pm=%s: recovered %d/%d  planted L %.4f  best L min/median %.4f/%.4f  K(last)=%d  %.1fs"
              % (cfg, P, G, pm, rec, len(seeds), Lp, min(Ls), float(np.median(Ls)), r["best_labels"].max(), time.time() - t), flush=True)

scan("C1", 128, [100, 300], range(1, 11), pm=0.1)
scan("C3", 4096, [500, 2000, 5000], range(1, 4))
scan("C4", 65536, [3000], range(1, 2))
