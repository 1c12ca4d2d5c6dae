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
