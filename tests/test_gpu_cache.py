"""Cluster cache of the label-sparse pass (pga_set_cluster_cache): a cached
c_s is the exact fixed-point sum of its member set, so L, top and the whole
GA trajectory are bit-identical with the cache on or off, and identical to
the oracle within the parity tolerance.  Covers repeated evaluation (every
cluster a hit), GA generations (mostly hits), the table clearing itself
when half full (small P: 4096 slots), and the cache's hit counters."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def pga():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1403_4099_b200 import build
    build.build()
    import paper_1403_4099_b200 as p
    return p


def _assert_L(Lg, Lo):
    err = np.abs(np.asarray(Lg) - np.asarray(Lo)) / np.maximum(1.0, np.abs(Lo))
    assert err.max() <= TOL, "max rel err %g at %d" % (err.max(), int(err.argmax()))


def test_repeat_evaluation_hits_and_matches_oracle(pga, orc):
    X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
    C = orc.pearson(X)
    N, P = C.shape[0], 1024
    rng = np.random.default_rng(4)
    lab = np.concatenate([workloads.population_mix(4, planted, P // 2),
                          workloads.random_labels(rng, P // 2, N, K=60)])
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P))
    try:
        pga.pga_set_sparse_threshold(ctx, 1.0)
        pga.pga_profile_enable(ctx, 1)
        a = pga.pga_evaluate(ctx, lab + 1)          # misses: gathered and inserted
        h1, _ = pga.pga_profile_cache(ctx)
        b = pga.pga_evaluate(ctx, lab + 1)          # the same clusters again: hits
        h2, saved = pga.pga_profile_cache(ctx)
        pga.pga_set_cluster_cache(ctx, False)
        c = pga.pga_evaluate(ctx, lab + 1)
        pga.pga_profile_enable(ctx, 0)
    finally:
        pga.pga_destroy(ctx)
    assert np.array_equal(a, b) and np.array_equal(a, c)
    _assert_L(a, orc.evaluate(C, lab, nthreads=8)[0])
    assert h2 - h1 > 0 and saved > 0


def _trajectory(pga, C, P, N, G, seed, cache, theta=1.0):
    params = pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=G + 5, seed=seed)
    ctx = pga.pga_create(C, params)
    try:
        pga.pga_set_sparse_threshold(ctx, theta)
        pga.pga_set_cluster_cache(ctx, cache)
        pga.pga_profile_enable(ctx, 1)
        pga.pga_init(ctx, seed)
        for _ in range(G):
            pga.pga_gen_evaluate(ctx)
            pga.pga_gen_breed(ctx)
        pga.pga_gen_evaluate(ctx)
        pop, L, top = pga.pga_get_population(ctx, P, N, with_top=True)
        hits = pga.pga_profile_cache(ctx)[0]
    finally:
        pga.pga_destroy(ctx)
    return pop, L, top, hits


@pytest.mark.parametrize("P,G", [(2048, 60), (64, 400)])
def test_ga_trajectory_identical_with_and_without_cache(pga, orc, P, G):
    """P = 64 gets the smallest table (4096 slots), which fills past half
    and is cleared by the pass several times in 400 generations."""
    X, _ = workloads.noh_returns(workloads.CONFIGS["C4"])
    C = orc.pearson(X)
    N = C.shape[0]
    pa, La, ta, hits = _trajectory(pga, C, P, N, G, 31, True)
    pb, Lb, tb, none = _trajectory(pga, C, P, N, G, 31, False)
    assert np.array_equal(pa, pb) and np.array_equal(La, Lb) and np.array_equal(ta, tb)
    assert hits > 0 and none == 0
    _assert_L(La, orc.evaluate(C, pa - 1, nthreads=8)[0])


def test_cache_lockstep_with_oracle(pga, orc):
    """Default threshold and cache: GPU L and the oracle's operators agree
    generation by generation (bit-exact populations)."""
    X, _ = workloads.noh_returns(workloads.CONFIGS["C3"])
    C = orc.pearson(X)
    N, P = C.shape[0], 512
    params = pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=50, seed=8)
    ctx = pga.pga_create(C, params)
    try:
        pga.pga_set_sparse_threshold(ctx, 1.0)
        pga.pga_init(ctx, 8)
        op = orc.default_params(pop=P, p_m=2.0 / N, tol=-1.0, max_gens=50, seed=8)
        for g in range(6):
            pga.pga_gen_evaluate(ctx)
            pop, L, top = pga.pga_get_population(ctx, P, N, with_top=True)
            _assert_L(L, orc.evaluate(C, pop - 1, nthreads=8)[0])
            nxt = orc.step(op, pop - 1, L, top, g)
            pga.pga_gen_breed(ctx)
            pop2, _ = pga.pga_get_population(ctx, P, N)
            assert np.array_equal(pop2 - 1, nxt), g
    finally:
        pga.pga_destroy(ctx)
