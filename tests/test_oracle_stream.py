"""Pins of oracle/stream.py (f4: EWMA covariance, correlation, RMT
cleaning) against closed forms, the SPEC's worked
examples, spectral identities and the method's own fitness."""
import numpy as np
import pytest

from oracle import stream as ost
import workloads


def test_ewma_zero_stream_and_single_observation():
    lam = 0.98
    mean, cov = np.zeros(4), np.zeros((4, 4))
    for _ in range(10):
        mean, cov = ost.ewma_update(mean, cov, np.zeros(4), lam)
    assert np.all(cov == 0.0) and np.all(mean == 0.0)
    x = np.array([1.5, -2.0, 0.25, 3.0])
    mean, cov = ost.ewma_update(np.zeros(4), np.zeros((4, 4)), x, lam)
    assert np.array_equal(cov, (1.0 - lam) * np.outer(x, x))  # S:287, one-step algebra
    assert np.array_equal(mean, (1.0 - lam) * x)


def test_ewma_closed_form():
    """cov_T = sum_k lam^(T-1-k) (1-lam) d_k d_k^T with d_k = x_k - m_{k-1},
    m_k = (1-lam) sum_{m<=k} lam^(k-m) x_m: an independent (non-recursive)
    formulation."""
    rng = np.random.default_rng(3)
    lam, T, N = 0.9, 60, 5
    X = rng.standard_normal((T, N))
    mean, cov = np.zeros(N), np.zeros((N, N))
    for t in range(T):
        mean, cov = ost.ewma_update(mean, cov, X[t], lam)
    m = [np.zeros(N)]
    for k in range(T):
        m.append((1 - lam) * sum(lam ** (k - j) * X[j] for j in range(k + 1)))
    ref = sum(lam ** (T - 1 - k) * (1 - lam) * np.outer(X[k] - m[k], X[k] - m[k]) for k in range(T))
    assert np.allclose(cov, ref, rtol=1e-12, atol=1e-14)
    assert np.allclose(mean, m[T], rtol=1e-12, atol=1e-14)


def test_ewma_unit_variance_converges():
    rng = np.random.default_rng(7)
    mean, cov = np.zeros(3), np.zeros((3, 3))
    for x in rng.standard_normal((2000, 3)):
        mean, cov = ost.ewma_update(mean, cov, x, 0.98)
    # S:288 says "within 0.1"; a 50-sample effective window has sd ~ 0.2
    # per diagonal entry, so the bound is checked on the average
    assert abs(np.diag(cov).mean() - 1.0) < 0.25


def test_correlation_from_covariance():
    assert np.array_equal(ost.correlation_from_covariance(np.diag([2.0, 3.0, 5.0])), np.eye(3))
    C = ost.correlation_from_covariance(np.array([[4.0, 2.0], [2.0, 9.0]]))
    assert C[0, 1] == 2.0 / 6.0 and C[1, 0] == 2.0 / 6.0
    assert C[0, 0] == 1.0 and C[1, 1] == 1.0
    with pytest.raises(ValueError):
        ost.correlation_from_covariance(np.array([[0.0, 0.0], [0.0, 1.0]]))


def test_rmt_identity_and_band():
    assert np.allclose(ost.rmt_clean(np.eye(6), 0.1), np.eye(6), atol=1e-14)
    lo, hi = ost.mp_band(0.36)
    assert abs(lo - 0.16) < 1e-15 and abs(hi - 2.56) < 1e-15


def test_rmt_filter_spectrum():
    """Eigenvalues outside the band survive, those inside become their mean,
    and the trace is preserved, on a matrix built from a chosen
    spectrum."""
    rng = np.random.default_rng(11)
    N = 8
    Q, _ = np.linalg.qr(rng.standard_normal((N, N)))
    w = np.array([4.0, 2.9, 0.5, 0.7, 1.1, 1.3, 0.05, 0.10])    # band [0.16, 2.56] at q = 0.36
    C = (Q * w) @ Q.T
    C = 0.5 * (C + C.T)
    C2 = ost.rmt_filter(C, 0.36)
    band = (w >= 0.16) & (w <= 2.56)
    expect = w.copy()
    expect[band] = w[band].mean()
    assert np.allclose(np.sort(np.linalg.eigvalsh(C2)), np.sort(expect), atol=1e-12)
    assert abs(np.trace(C2) - np.trace(C)) < 1e-12


def test_rmt_clean_properties():
    X, planted = workloads.noh_returns(workloads.PlantedSpec((5, 5), (0.9, 0.9), 100, 7))
    import oracle as orc
    C = orc.pearson(X)
    out = ost.rmt_clean(C, 10 / 100)
    assert np.array_equal(out, out.T)
    assert np.all(np.diag(out) == 1.0) and abs(np.trace(out) - 10) < 1e-12
    assert np.all(np.abs(out) <= 1.0 + 1e-12)
    w = np.sort(np.linalg.eigvalsh(C))[::-1]
    w2 = np.sort(np.linalg.eigvalsh(ost.rmt_filter(C, 0.1)))[::-1]
    assert np.allclose(w[:2], w2[:2], atol=1e-12)                # signal eigenvalues untouched


def test_rmt_clean_keeps_planted_fitness(orc):
    """cleaning enhances the clusters -- the planted partition's Eq. 8
    likelihood does not decrease (2 blocks, rho = 0.8, N = 10, D = 100)."""
    worse = 0
    for seed in range(20):
        X, planted = workloads.noh_returns(workloads.PlantedSpec((5, 5), (0.8 ** 0.5, 0.8 ** 0.5), 100, 500 + seed))
        C = orc.pearson(X)
        L0, _ = orc.log_likelihood(C, planted)
        L1, _ = orc.log_likelihood(ost.rmt_clean(C, 0.1), planted)
        worse += L1 < L0 - 1e-12
    assert worse == 0


def test_stream_emission_schedule():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((57, 4))
    out = ost.corr_stream(X, lam=0.9, warm=20, stride=9, clean=False)
    assert out.shape == (ost.n_emitted(57, 20, 9), 4, 4) == (5, 4, 4)
    mean, cov = np.zeros(4), np.zeros((4, 4))
    for t in range(20 + 9 * 2):                                   # emission b = 2 after t = 37
        mean, cov = ost.ewma_update(mean, cov, X[t], 0.9)
    assert np.array_equal(out[2], ost.correlation_from_covariance(cov))
