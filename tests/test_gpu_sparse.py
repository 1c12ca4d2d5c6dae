"""Label-sparse fitness (pga_set_sparse_threshold) vs the
oracle and vs the dense sweep: the same Eq. 5/6/8 values within the parity
tolerance whichever path evaluates a block, deterministic run to run, and
the GA stays bit-exact in lockstep with the oracle's operators."""
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


def _pops(N, planted, P, seed):
    rng = np.random.default_rng(seed)
    mix = workloads.population_mix(seed, planted, P)
    rnd = workloads.random_labels(rng, P, N)                       # sparse
    few = workloads.random_labels(rng, P, N, K=max(2, N // 40))    # few big clusters: dense
    return {"mix": mix, "random": rnd, "few": few}


@pytest.mark.parametrize("cfg,P", [("C1", 100), ("C3", 700), ("C4", 1000)])
@pytest.mark.parametrize("theta", [0.0, 1.0, 0.03])
def test_sparse_and_dense_paths_match_oracle(pga, orc, cfg, P, theta):
    X, planted = workloads.noh_returns(workloads.CONFIGS[cfg])
    C = orc.pearson(X)
    N = C.shape[0]
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, elite=min(10, P - 1)))
    try:
        pga.pga_set_sparse_threshold(ctx, theta)
        for name, lab in _pops(N, planted, P, 7).items():
            Lg = pga.pga_evaluate(ctx, lab + 1)
            Lo, _ = orc.evaluate(C, lab, nthreads=8)
            _assert_L(Lg, Lo)
    finally:
        pga.pga_destroy(ctx)


def test_sparse_path_is_deterministic_and_close_to_dense(pga, orc):
    X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
    C = orc.pearson(X)
    lab = workloads.population_mix(3, planted, 2048)
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=2048))
    try:
        pga.pga_set_sparse_threshold(ctx, 1.0)
        a = pga.pga_evaluate(ctx, lab + 1)
        b = pga.pga_evaluate(ctx, lab + 1)
        pga.pga_set_sparse_threshold(ctx, 0.0)
        d = pga.pga_evaluate(ctx, lab + 1)
    finally:
        pga.pga_destroy(ctx)
    assert np.array_equal(a, b)
    _assert_L(a, d)


def test_sparse_threshold_validation(pga):
    ctx = pga.pga_create(np.eye(4), pga.pga_params_default(pop_size=8, elite=2))
    try:
        with pytest.raises(pga.PgaError):
            pga.pga_set_sparse_threshold(ctx, 1.5)
    finally:
        pga.pga_destroy(ctx)


@pytest.mark.parametrize("N,P", [(640, 100), (641, 64), (1100, 40), (2048, 33), (2049, 32), (37, 33), (2, 5)])
def test_sparse_edges_match_oracle(pga, orc, N, P):
    """The two instantiations of the label-sparse pass (16 warps up to
    N = 640, 8 warps with 32 label registers per lane up to 2048) at their
    edges, the first N without a pass (2049), ragged P (not a multiple of
    32), N = 2: every path vs the oracle."""
    rng = np.random.default_rng(N + P)
    X = rng.standard_normal((max(3 * N, 40), N))
    k = max(1, N // 6)
    X += 0.8 * rng.standard_normal((X.shape[0], k))[:, rng.integers(0, k, N)]
    C = orc.pearson(X)
    labs = [workloads.random_labels(rng, P, N), workloads.random_labels(rng, P, N, K=max(2, N // 50))]
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, elite=min(10, P - 1)))
    try:
        for theta in (1.0, 0.0):
            pga.pga_set_sparse_threshold(ctx, theta)
            for lab in labs:
                _assert_L(pga.pga_evaluate(ctx, lab + 1), orc.evaluate(C, lab, nthreads=8)[0])
    finally:
        pga.pga_destroy(ctx)


@pytest.mark.parametrize("theta", [0.0, 1.0, 0.04])
def test_ga_recovers_C1_any_path(pga, orc, theta):
    """The GA recovers C1's planted partition whichever fitness path runs
    (forced dense, forced label-sparse, default)."""
    X, planted = workloads.noh_returns(workloads.CONFIGS["C1"])
    C = orc.pearson(X)
    ok = 0
    for seed in range(1, 6):
        ctx = pga.pga_create(C, pga.pga_params_default(pop_size=128, max_gens=300, tol=-1.0, seed=seed))
        try:
            pga.pga_set_sparse_threshold(ctx, theta)
            r = pga.pga_run(ctx, 300, seed, 18)
            Lr, _ = orc.log_likelihood(C, r["best_labels"] - 1)
            _assert_L([r["best_L"]], [Lr])
            ok += np.array_equal(r["best_labels"] - 1, planted)
        finally:
            pga.pga_destroy(ctx)
    assert ok >= 4, ok


def test_sparse_pass_in_lockstep_with_oracle(pga, orc):
    """C4-size GA generations with the default label-sparse pass: at every
    generation the GPU's L matches the oracle and, fed the GPU's L and top,
    the oracle's operators breed the GPU's next population bit for bit."""
    X, _ = workloads.noh_returns(workloads.CONFIGS["C4"])
    C = orc.pearson(X)
    P, N = 2048, 500
    params = pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=50, seed=21)
    ctx = pga.pga_create(C, params)
    try:
        pga.pga_init(ctx, 21)
        op = orc.default_params(pop=P, p_m=2.0 / N, tol=-1.0, max_gens=50, seed=21)
        for g in range(4):
            pga.pga_gen_evaluate(ctx)
            pop, L, top = pga.pga_get_population(ctx, P, N, with_top=True)
            _assert_L(L, orc.evaluate(C, pop - 1, nthreads=8)[0])
            nxt = orc.step(op, pop - 1, L, top, g)
            pga.pga_gen_breed(ctx)
            pop2, _ = pga.pga_get_population(ctx, P, N)
            assert np.array_equal(pop2 - 1, nxt), g
        assert pga.pga_profile_sparse_blocks(ctx) >= 0
    finally:
        pga.pga_destroy(ctx)


@pytest.mark.parametrize("theta", [0.0, 1.0])
def test_out_of_range_device_label_is_contained(pga, orc, theta):
    """A label >= N in one chromosome (device fast path, unchecked input)
    must not disturb the other chromosomes' L on either fitness path."""
    import torch
    X, planted = workloads.noh_returns(workloads.CONFIGS["C3"])
    C = orc.pearson(X)
    N, P = C.shape[0], 96
    lab = workloads.population_mix(5, planted, P)
    bad = lab.copy()
    bad[7, 3] = N + 5
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P))
    try:
        pga.pga_set_sparse_threshold(ctx, theta)
        L = torch.zeros(P, dtype=torch.float64, device="cuda")
        s = torch.cuda.Stream()
        pga.pga_evaluate_device(ctx, torch.from_numpy(bad.astype(np.int16)).cuda(), L, stream=s.cuda_stream)
        s.synchronize()
        Lg = L.cpu().numpy()
    finally:
        pga.pga_destroy(ctx)
    Lo, _ = orc.evaluate(C, lab)
    keep = np.arange(P) != 7
    _assert_L(Lg[keep], Lo[keep])


def test_switching_the_sparse_pass_off_mid_run(pga, orc):
    """While the label-sparse pass runs, the breed leaves the gene-major copy
    to it; switching the pass off between generations must hand the dense
    sweep a current copy (the L of the next evaluation matches the oracle)."""
    X, _ = workloads.noh_returns(workloads.CONFIGS["C4"])
    C = orc.pearson(X)
    P, N = 2048, 500
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=60, seed=4))
    try:
        pga.pga_init(ctx, 4)
        for _ in range(12):
            pga.pga_gen_evaluate(ctx)
            pga.pga_gen_breed(ctx)
        pga.pga_set_sparse_threshold(ctx, 0.0)
        pga.pga_gen_evaluate(ctx)
        pop, L = pga.pga_get_population(ctx, P, N)
        _assert_L(L, orc.evaluate(C, pop - 1, nthreads=8)[0])
        pga.pga_gen_breed(ctx)
        pga.pga_set_sparse_threshold(ctx, -1.0)     # and back on (automatic)
        pga.pga_gen_evaluate(ctx)
        pop, L = pga.pga_get_population(ctx, P, N)
        _assert_L(L, orc.evaluate(C, pop - 1, nthreads=8)[0])
    finally:
        pga.pga_destroy(ctx)


def test_sparse_pass_C5_ga_lockstep(pga, orc):
    """N = 2000 (C5's stocks) GA generations with the automatic label-sparse
    pass (early generations: every block sparse) and the cluster cache: L
    matches the oracle and the bred population equals orc_step on the GPU's
    L and top; the pass evaluated blocks."""
    X, _ = workloads.noh_returns(workloads.CONFIGS["C5"])
    C = orc.pearson(X)
    N, P, gens = C.shape[0], 256, 4
    params = pga.pga_params_default(pop_size=P, max_gens=gens + 1, tol=-1.0, p_mutation=2.0 / N, seed=21)
    op = orc.default_params(pop=P, max_gens=gens + 1, tol=-1.0, p_m=2.0 / N, seed=21)
    ctx = pga.pga_create(C, params)
    try:
        pga.pga_init(ctx, 21)
        pop, _ = pga.pga_get_population(ctx)
        for g in range(gens):
            pga.pga_generation(ctx)
            nxt, L, top = pga.pga_get_population(ctx, with_top=True)
            _assert_L(L, orc.evaluate(C, pop - 1, nthreads=8)[0])
            assert np.array_equal(nxt - 1, orc.step(op, pop - 1, L, top, gen=g)), g
            pop = nxt
        blocks, _ = pga.pga_profile_sparse(ctx)
        assert blocks > 0
    finally:
        pga.pga_destroy(ctx)
