"""How many of a generation's cluster evaluations repeat one from the
previous generation (C4)?  For each generation g listed, the clusters
(n >= 2) of population g+1 are looked up, by member set, among those of
population g; printed weighted by the pair updates n(n-1)/2 a label-sparse
evaluation would gather.  Decides whether a cluster cache pays."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads, paper_1403_4099_b200 as pga

X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N, P = 500, 65536
keys = np.random.default_rng(123).integers(0, 2**63, N, dtype=np.uint64) * np.uint64(2) + np.uint64(1)


def clusters(pop):
    lab = pop.astype(np.int64)                     # 1-based labels, [P][N]
    idx = (np.arange(P, dtype=np.int64)[:, None] * (N + 1) + lab).ravel()
    h = np.zeros(P * (N + 1), np.uint64)
    np.add.at(h, idx, np.tile(keys, P))
    n = np.bincount(idx, minlength=P * (N + 1))
    m = n >= 2
    return h[m], n[m]


ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=8000, seed=5))
pga.pga_init(ctx, 5)
done = 0
for g in (5, 50, 200, 500, 1000, 1500, 2000, 3000, 5000):
    while done < g:
        pga.pga_gen_evaluate(ctx)
        pga.pga_gen_breed(ctx)
        done += 1
    pa, _ = pga.pga_get_population(ctx, P, N)
    pga.pga_gen_evaluate(ctx)
    pga.pga_gen_breed(ctx)
    done += 1
    ch, _ = pga.pga_get_population(ctx, P, N)
    hp, npar = clusters(pa)
    hc, nc = clusters(ch)
    hit = np.isin(hc, np.unique(hp))
    pairs = nc * (nc - 1) // 2
    out = ["gen %4d: pairs/chrom %7.0f (dense %d)" % (g, pairs.sum() / P, N * (N - 1) // 2),
           "hit by pairs %.3f, by clusters %.3f" % (pairs[hit].sum() / pairs.sum(), hit.mean())]
    for nmin in (4, 8, 16):
        big = nc >= nmin
        out.append("n>=%d: %.3f of pairs, hit %.3f" % (nmin, pairs[big].sum() / pairs.sum(),
                                                        pairs[big & hit].sum() / max(1, pairs[big].sum())))
    u = np.unique(hc).size
    out.append("distinct %d of %d" % (u, hc.size))
    print("; ".join(out), flush=True)
pga.pga_destroy(ctx)
