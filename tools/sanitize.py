"""Small invocations of every kernel family, checked against the oracle and,
with the device-check build (PGA_LIB=paper_1403_4099_b200/libpga_check.so,
-DPGA_DEVICE_CHECKS), against the hot kernels' index/range invariants
(SURVEY §4 layer 6; compute-sanitizer itself is closed on the GPU pool, where
it can also be run as
    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize.py)
Covers k_fitness (TMA sweep + last-CTA fold), k_fitness_sparse (counting
sort, L2 gathers, cluster-cache CAS / relaxed loads, clear path), k_stats
(multi-CTA last-CTA reduction), the order sort and merge levels, selection
(small one-CTA path and the multi-kernel path), k_breed2 / k_breed, k_batch,
k_gram (Pearson) and the correlation stream.  Results are checked against
the oracle so a run that silently does nothing fails."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle as orc  # noqa: E402
import workloads  # noqa: E402
import paper_1403_4099_b200 as pga  # noqa: E402


def close(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.all(np.abs(a - b) <= 1e-9 * np.maximum(1.0, np.abs(b)))


def main():
    import torch
    what = sys.argv[1:] or ["all"]
    X, planted = workloads.noh_returns(workloads.CONFIGS["C3"])
    C = pga.pga_correlation(X)                                   # k_colstats / k_gram
    assert np.abs(C - orc.pearson(X)).max() <= 1e-12
    N = C.shape[0]
    # dense path (theta = 0): k_pack, k_fitness with its fused last-CTA fold
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=2048, p_mutation=2.0 / N, tol=-1.0, seed=3))
    try:
        lab = workloads.population_mix(4, planted, 700)
        pga.pga_set_sparse_threshold(ctx, 0.0)
        assert close(pga.pga_evaluate(ctx, lab + 1), orc.evaluate(C, lab)[0])
        # sparse path with the cluster cache (theta = 1 forces it at N = 100)
        pga.pga_set_sparse_threshold(ctx, 1.0)
        for _ in range(2):                                       # second pass: cache hits
            assert close(pga.pga_evaluate(ctx, lab + 1), orc.evaluate(C, lab)[0])
        # GA generations (multi-kernel selection at P = 2048 > 1024, k_breed2,
        # k_stats, sparse pass with hysteresis, graph replay)
        pga.pga_init(ctx, 3)
        for _ in range(6):
            pga.pga_gen_evaluate(ctx)
            pga.pga_gen_breed(ctx)
        pop, L = pga.pga_get_population(ctx)
        st = pga.pga_get_state(ctx)
        assert st["generation"] == 6 and np.isfinite(L).all()
    finally:
        pga.pga_destroy(ctx)
    # tiny cache table: force clears (4096 slots, many distinct clusters)
    spec = workloads.CONFIGS["C4"]
    X4, pl4 = workloads.noh_returns(spec)
    C4 = orc.pearson(X4)
    ctx = pga.pga_create(C4, pga.pga_params_default(pop_size=64, p_mutation=0.05, tol=-1.0, seed=5))
    try:
        pga.pga_init(ctx, 5)
        for _ in range(12):
            pga.pga_gen_evaluate(ctx)
            pga.pga_gen_breed(ctx)
        pop, L = pga.pga_get_population(ctx)
        assert np.isfinite(L).all()
        print("cache", pga.pga_cache_stats(ctx))
    finally:
        pga.pga_destroy(ctx)
    # C4-size GA (N = 500): automatic label-sparse pass with the cache,
    # cluster selection (P = 4096), and the N = 2000 instantiation of the pass
    ctx = pga.pga_create(C4, pga.pga_params_default(pop_size=4096, p_mutation=0.004, tol=-1.0, seed=6))
    try:
        pga.pga_init(ctx, 6)
        for _ in range(8):
            pga.pga_gen_evaluate(ctx)
            pga.pga_gen_breed(ctx)
        pga.pga_gen_evaluate(ctx)
        pop, L = pga.pga_get_population(ctx)
        idx = np.arange(0, 4096, 97)
        assert close(L[idx], orc.evaluate(C4, pop[idx] - 1)[0])
    finally:
        pga.pga_destroy(ctx)
    X5, pl5 = workloads.noh_returns(workloads.CONFIGS["C5"])
    C5 = orc.pearson(X5)
    ctx = pga.pga_create(C5, pga.pga_params_default(pop_size=96, seed=8))
    try:
        lab5 = workloads.population_mix(9, pl5, 96)
        pga.pga_set_sparse_threshold(ctx, 1.0)
        assert close(pga.pga_evaluate(ctx, lab5 + 1), orc.evaluate(C5, lab5, nthreads=8)[0])
    finally:
        pga.pga_destroy(ctx)
    # small single-CTA selection path, k_stats with a stall stop
    C1, p1 = workloads.noh_returns(workloads.CONFIGS["C1"])
    C1 = orc.pearson(C1)
    ctx = pga.pga_create(C1, pga.pga_params_default(pop_size=128, seed=7))
    try:
        r = pga.pga_run(ctx, 30, 7)
        assert r["gens_run"] == 30
    finally:
        pga.pga_destroy(ctx)
    # wide N: k_breed (N > 1024) through the operator hook
    Nw, P = 1100, 24
    rng = np.random.default_rng(1)
    popw = orc.canonicalize(rng.integers(0, 40, (P, Nw)))
    top = popw[:, 0].copy()
    Lw = rng.random(P)
    params = pga.pga_params_default(pop_size=P, elite=4, p_mutation=0.01, seed=9)
    o, sel = orc.select(Lw, 4, seed=9)
    sig = orc.mates(len(sel), seed=9)
    assert np.array_equal(pga.pga_op_breed(popw, top, o, sel, sig, params),
                          orc.breed(popw, top, o, 4, sel, sig, 0.9, 0.01, 0.9, seed=9))
    # multi-kernel selection hook (P > 4096: run sort + merge levels + scan + SUS)
    Ls = np.round(rng.random(5000) * 10, 2)
    p5 = pga.pga_params_default(pop_size=5000, elite=10, seed=4)
    og, sg = pga.pga_op_select(Ls, p5)
    oo, so = orc.select(Ls, 10, seed=4)
    assert np.array_equal(og, oo) and np.array_equal(sg, so)
    # batched GA (k_batch) and the correlation stream (k_ewma, k_clean)
    Xw, _ = workloads.window_returns(4)
    Cw = np.stack([orc.pearson(Xw[b]) for b in range(4)])
    res = pga.pga_batch_run(Cw, pga.pga_params_default(pop_size=64, max_gens=15, seed=11))
    for b in range(4):
        ref = orc.run(Cw[b], orc.default_params(pop=64, max_gens=15, seed=11 + b))
        assert np.array_equal(res["best_labels"][b] - 1, ref["best_labels"])
    Xs, _ = workloads.stream_returns(200, 18, seed=3)
    Cs = pga.pga_corr_stream(Xs, warm=160, stride=20, q=0.0)
    assert np.isfinite(Cs).all()
    torch.cuda.synchronize()
    v = pga.pga_debug_violations()
    print("sanitize workload ok; device invariant violations: %d" % v)
    if v > 0:
        sys.exit(3)


if __name__ == "__main__":
    main()
