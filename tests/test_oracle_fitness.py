"""Pins for the oracle's fitness (Eq. 5, 6, 8) against things other than itself:
worked values, closed forms, an independent numpy formulation, invariants and
exhaustive search.  CPU only."""
import math

import numpy as np
import pytest

from conftest import golden
from oracle import npref


def _rand_corr(rng, N, T=None):
    T = T or 3 * N
    X = rng.standard_normal((T, N))
    X -= X.mean(0)
    X /= np.linalg.norm(X, axis=0)
    C = X.T @ X
    C = 0.5 * (C + C.T)
    np.fill_diagonal(C, 1.0)
    return C


def _block_corr(N, members, rho):
    C = np.eye(N)
    for i in members:
        for j in members:
            if i != j:
                C[i, j] = rho
    return C


def _read_examples():
    rows = []
    for line in open(golden("likelihood_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, n, rho, val = line.split()[:4]
        rows.append((name, int(n), float(rho), float(val)))
    return rows


@pytest.mark.parametrize("name,n,rho,expected", _read_examples())
def test_worked_examples(orc, name, n, rho, expected):
    # embed the cluster among singletons at scattered positions
    N = n + 5
    members = list(range(1, 2 * n, 2))[:n] if 2 * n <= N else list(range(n))
    C = _block_corr(N, members, rho)
    lab = np.arange(N, dtype=np.int32) + 1
    lab[members] = 0
    L, top = orc.log_likelihood(C, lab)
    # fp64 summation of n(n-1) equal terms: relative error grows ~n^2 eps
    assert L == pytest.approx(expected, rel=1e-12, abs=1e-15)
    assert top == 0


def test_triple_spec_value_is_wrong(orc):
    """SPEC S:70 prints 1.787780; the expression it gives evaluates to
    1.78777538 (difference 4.6e-6) -- the oracle follows the expression."""
    C = _block_corr(3, [0, 1, 2], 0.9)
    L, _ = orc.log_likelihood(C, [0, 0, 0])
    assert abs(L - 0.5 * (math.log(3 / 8.4) + 2 * math.log(6 / 0.6))) < 1e-14
    assert abs(L - 1.787780) > 4e-6


@pytest.mark.parametrize("n", [2, 3, 5, 10, 37])
@pytest.mark.parametrize("rho", [0.05, 0.3, 0.64, 0.81])
def test_block_closed_form(orc, n, rho):
    C = _block_corr(n, range(n), rho)
    L, _ = orc.log_likelihood(C, np.zeros(n, np.int32))
    assert L == pytest.approx(npref.block_closed_form(n, rho), rel=1e-12)


def test_two_blocks_add(orc):
    """Eq. 8 is a sum over clusters: two planted blocks give the sum of their
    closed forms (and the cross-block zeros do not leak in)."""
    N = 12
    C = _block_corr(N, [0, 2, 4, 6], 0.5)
    C2 = _block_corr(N, [1, 3, 5], 0.7)
    C = C + C2 - np.eye(N)
    lab = np.arange(N, dtype=np.int32)
    lab[[0, 2, 4, 6]] = 0
    lab[[1, 3, 5]] = 1
    L, top = orc.log_likelihood(C, lab)
    want = npref.block_closed_form(4, 0.5) + npref.block_closed_form(3, 0.7)
    assert L == pytest.approx(want, rel=1e-13)
    # the triple at 0.7 has the larger per-cluster term
    assert top == (1 if npref.block_closed_form(3, 0.7) > npref.block_closed_form(4, 0.5) else 0)


def test_singletons_zero(orc):
    rng = np.random.default_rng(3)
    C = _rand_corr(rng, 15)
    L, top = orc.log_likelihood(C, np.arange(15))
    assert L == 0.0 and top == -1


def test_identity_zero(orc):
    rng = np.random.default_rng(4)
    C = np.eye(20)
    for _ in range(20):
        L, top = orc.log_likelihood(C, rng.integers(0, 5, 20))
        assert L == 0.0 and top == -1  # c_s = n_s for every cluster


def test_c_equals_n_zero(orc):
    """A cluster whose off-diagonal correlations cancel has c_s = n_s and
    contributes 0 ("c_s = n_s")."""
    C = np.eye(3)
    C[0, 1] = C[1, 0] = 0.5
    C[0, 2] = C[2, 0] = -0.5
    L, top = orc.log_likelihood(C, [0, 0, 0])
    assert L == 0.0 and top == -1


def test_anticorrelated_pair_zero(orc):
    """Reading Q2: raw Eq. 8 gives ln(4/3)/2 for rho = -0.5 as well (it is
    symmetric in rho); the constrained MLE (g* in [0,1], Eq. 4) gives 0."""
    C = np.array([[1.0, -0.5], [-0.5, 1.0]])
    L, _ = orc.log_likelihood(C, [0, 0])
    assert L == 0.0
    raw = 0.5 * (math.log(2 / 1.0) + math.log(2 / 3.0))
    assert raw == pytest.approx(0.5 * math.log(4 / 3))


def test_cluster_term_continuous_at_c_eq_n(orc):
    for n in (2, 3, 7):
        assert orc.cluster_term(n, n) == 0.0
        assert 0.0 < orc.cluster_term(n, n + 1e-6) < 1e-9


def test_clamp_near_perfect_correlation(orc):
    """Q3: duplicated series (rho = 1) give a finite value, equal to the
    clamped formula at c = n^2 - 1e-9."""
    C = np.ones((4, 4))
    L, _ = orc.log_likelihood(C, [0, 0, 0, 0])
    n = 4.0
    ch = n * n - 1e-9
    assert math.isfinite(L)
    assert L == pytest.approx(0.5 * (math.log(n / ch) + (n - 1) * math.log((n * n - n) / 1e-9)),
                              rel=1e-6)


def test_clamp_region_properties(orc):
    """Q3 pinned by properties a wrong clamp would break, not by retyping it:
    (a) the term is constant for c in [n^2 - 1e-9, n^2] (the clamp is active
    exactly there); (b) it is continuous at the clamp boundary from below;
    (c) it increases strictly in c on (n, n^2 - 1e-9) (a dropped term or a
    sign error in either log breaks this); (d) for a pair the clamped value
    equals the pair closed form -ln(1 - rho^2) at rho = 1 - 5e-10 (c = 2 + 2 rho
    = 4 - 1e-9), independent of Eq. 8's algebra."""
    for n in (2, 3, 5, 40):
        n2 = float(n * n)
        top = orc.cluster_term(n, n2)
        for c in (n2 - 1e-9, n2 - 5e-10, n2 - 1e-12, n2):
            assert orc.cluster_term(n, c) == top
        # below the boundary the second log is ~(n-1) ln(1/(n^2 - c)): the gap to
        # the clamped value is ~(n-1) d / 1e-9 for small d, so it vanishes
        d3 = max(1e-13, 8 * np.spacing(n2))      # resolvable below n^2 - 1e-9
        below = [orc.cluster_term(n, n2 - 1e-9 - d) for d in (1e-7, 1e-11, d3)]
        gaps = [top - b for b in below]
        assert all(g > 0 for g in gaps) and gaps[0] > gaps[1] > gaps[2]
        assert gaps[1] < 0.02 * (n - 1) and gaps[2] < 2.0 * (n - 1) * d3 / 1e-9
        cs = np.linspace(n + 1e-3, n2 - 2e-9, 200)
        f = [orc.cluster_term(n, float(c)) for c in cs]
        assert all(b > a for a, b in zip(f, f[1:]))
    rho = 1.0 - 5e-10
    assert orc.cluster_term(2, 4.0) == pytest.approx(-math.log1p(-rho * rho), rel=1e-7)


@pytest.mark.parametrize("seed", range(6))
def test_cross_oracle_one_hot(orc, seed):
    """Eq. 5/6 double loop vs numpy diag(Z^T C Z)."""
    rng = np.random.default_rng(100 + seed)
    N = int(rng.integers(5, 60))
    C = _rand_corr(rng, N)
    lab = rng.integers(0, max(1, N // 3), N).astype(np.int32)
    n1, c1 = orc.cluster_stats(C, lab)
    n2, c2 = npref.cluster_stats(C, lab)
    assert np.array_equal(n1, n2)
    assert n1.sum() == N
    np.testing.assert_allclose(c1, c2, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(5))
def test_permutation_invariance(orc, seed):
    rng = np.random.default_rng(200 + seed)
    N = 30
    C = _rand_corr(rng, N, T=40)
    lab = rng.integers(0, 6, N).astype(np.int32)
    L0, _ = orc.log_likelihood(C, lab)
    relabel = rng.permutation(6).astype(np.int32)
    L1, _ = orc.log_likelihood(C, relabel[lab])
    assert L1 == pytest.approx(L0, rel=1e-14, abs=1e-15)
    perm = rng.permutation(N)
    L2, _ = orc.log_likelihood(C[np.ix_(perm, perm)], lab[perm])
    assert L2 == pytest.approx(L0, rel=1e-12, abs=1e-14)


def test_nonnegative(orc):
    rng = np.random.default_rng(7)
    for _ in range(50):
        N = int(rng.integers(2, 25))
        C = _rand_corr(rng, N, T=int(rng.integers(N, 4 * N)))
        L, _ = orc.log_likelihood(C, rng.integers(0, N, N))
        assert L >= 0.0


def test_monotone_pair_response(orc):
    vals = []
    for rho in np.linspace(0.01, 0.99, 40):
        C = np.array([[1.0, rho], [rho, 1.0]])
        vals.append(orc.log_likelihood(C, [0, 0])[0])
    assert all(b > a for a, b in zip(vals, vals[1:]))


def test_evaluate_batch_matches_single(orc):
    rng = np.random.default_rng(11)
    N, P = 23, 40
    C = _rand_corr(rng, N)
    lab = rng.integers(0, 8, (P, N)).astype(np.int32)
    L1, t1 = orc.evaluate(C, lab, nthreads=1)
    L4, t4 = orc.evaluate(C, lab, nthreads=4)
    assert np.array_equal(L1, L4) and np.array_equal(t1, t4)
    for p in range(P):
        L, t = orc.log_likelihood(C, lab[p])
        assert L == L1[p] and t == t1[p]


def test_bell_numbers(orc):
    want = [int(v) for v in open(golden("bell_numbers.txt")).read().split("\n")[-2].split()]
    assert npref.bell(12)[1:] == want
    for n in range(1, 11):
        C = np.eye(n)
        _, _, count = orc.brute_force(C)
        assert count == want[n - 1]


def test_brute_force_planted_blocks(orc):
    """Two 4-blocks at rho = 0.7: the planted partition is the
    exhaustive argmax."""
    N = 8
    C = _block_corr(N, [0, 1, 2, 3], 0.7) + _block_corr(N, [4, 5, 6, 7], 0.7) - np.eye(N)
    best, L, count = orc.brute_force(C)
    assert count == 4140
    assert list(best) == [0, 0, 0, 0, 1, 1, 1, 1]
    assert L == pytest.approx(2 * npref.block_closed_form(4, 0.7), rel=1e-12)


def test_brute_force_identity_tie(orc):
    best, L, count = orc.brute_force(np.eye(4))
    assert L == 0.0 and count == 15
    # every partition ties at 0; the first visited string (all zeros) is kept
    assert list(best) == [0, 0, 0, 0]


def test_brute_force_is_max_over_random(orc):
    rng = np.random.default_rng(12)
    C = _rand_corr(rng, 8, T=12)
    _, Lb, _ = orc.brute_force(C)
    lab = rng.integers(0, 8, (2000, 8)).astype(np.int32)
    L, _ = orc.evaluate(C, lab)
    assert L.max() <= Lb + 1e-12
