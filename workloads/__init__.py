"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it draws returns from the
Noh generative model (Eq. 2, the data model the paper assumes) and
label populations, with numpy's PCG64.  Correlation matrices are computed
from these returns by each side separately (``oracle.pearson`` /
``pga_correlation``), and fitness is never computed here.

Recipes follow SURVEY.md §8(d): cluster sizes, loadings g_s,
sample lengths T and seeds per BASELINE.json config.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class PlantedSpec:
    sizes: tuple
    g: tuple
    T: int
    seed: int
    singletons: int = 0          # extra independent assets (g = 0), Q25
    shuffle: bool = True         # scatter cluster members over asset indices

    @property
    def N(self) -> int:
        return int(sum(self.sizes)) + self.singletons


def _c5_sizes():
    return (250, 222, 197, 174, 154, 137, 121, 107, 95, 84, 75, 66, 58, 52, 46,
            41, 36, 32, 28, 25)


CONFIGS = {
    # BASELINE.json configs[0..4]; SURVEY.md §8(d)
    "C1": PlantedSpec((7, 6, 5), (0.8, 0.7, 0.6), 250, 1801),
    "C2": PlantedSpec((4, 3, 2), (0.8, 0.7, 0.6), 250, 1001, singletons=1),
    "C3": PlantedSpec((30, 25, 20, 15, 10), (0.8, 0.75, 0.7, 0.65, 0.6), 2000, 10002),
    "C4": PlantedSpec((100, 90, 80, 70, 60, 50, 25, 15, 10),
                      tuple(np.linspace(0.85, 0.55, 9).tolist()), 2000, 50004),
    "C5": PlantedSpec(_c5_sizes(), tuple(np.linspace(0.85, 0.55, 20).tolist()), 4000, 200005),
}

# GA settings per config: population per run, generations.
GA_SETTINGS = {
    "C1": dict(pop=128, gens=100),
    "C2": dict(pop=1024, gens=400),
    "C3": dict(pop=4096, gens=500),
    "C4": dict(pop=65536, gens=1000),
    "C5": dict(pop=262144, gens=0),
}


def noh_returns(spec: PlantedSpec):
    """Draw X [T][N] from Eq. 2: x_i = g_s eta_s + sqrt(1 - g_s^2) eps_i.

    Returns (X, planted) where planted[i] is the 0-based cluster of asset i
    in first-occurrence canonical order (independent assets get their own
    singleton label).
    """
    rng = np.random.Generator(np.random.PCG64(spec.seed))
    N, T = spec.N, spec.T
    k = len(spec.sizes)
    cluster = np.concatenate([np.full(n, c) for c, n in enumerate(spec.sizes)]
                             + [np.arange(k, k + spec.singletons)]).astype(np.int64)
    gs = np.concatenate([np.asarray(spec.g, np.float64), np.zeros(spec.singletons)])
    if spec.shuffle:
        cluster = cluster[rng.permutation(N)]
    eta = rng.standard_normal((T, k + spec.singletons))
    eps = rng.standard_normal((T, N))
    g = gs[cluster]
    X = np.ascontiguousarray(g[None, :] * eta[:, cluster] + np.sqrt(1.0 - g * g)[None, :] * eps)
    # first-occurrence relabelling of the planted partition (pure bookkeeping)
    first = {}
    planted = np.empty(N, np.int32)
    for i, c in enumerate(cluster):
        planted[i] = first.setdefault(int(c), len(first))
    return X, planted


# C2's exhaustive-check set (SPEC S:536 acceptance 2):
# 50 matrices, n in {6, 8, 10}, GA seeds / matrix seeds 2000..2049.  Every
# fifth matrix is pure noise (independent assets); the others plant 1..3
# clusters of 2..n/2 stocks with loadings g ~ U(0.55, 0.85), the remaining
# assets independent.  T = 250 as in C1/C2.
C2_SET = dict(count=50, seed0=2000, sizes=(6, 8, 10), T=250)


def c2_set_spec(k: int) -> PlantedSpec:
    seed = C2_SET["seed0"] + k
    n = C2_SET["sizes"][k % 3]
    if k % 5 == 4:
        return PlantedSpec((), (), C2_SET["T"], seed, singletons=n)
    rng = np.random.Generator(np.random.PCG64(seed))
    sizes = []
    for _ in range(int(rng.integers(1, 4))):
        m = int(rng.integers(2, n // 2 + 1))
        if sum(sizes) + m > n:
            break
        sizes.append(m)
    g = tuple(float(x) for x in rng.uniform(0.55, 0.85, len(sizes)))
    return PlantedSpec(tuple(sizes), g, C2_SET["T"], seed, singletons=n - sum(sizes))


def random_labels(rng, P, N, K=None):
    """Labels uniform over [0, K) (K = N: 'looks like initialisation')."""
    K = N if K is None else K
    return rng.integers(0, K, size=(P, N), dtype=np.int64).astype(np.int32)


def perturbed_planted(rng, planted, P, frac=0.05):
    """The planted partition with a fraction of genes re-drawn over [0, N)."""
    N = planted.shape[0]
    lab = np.tile(planted.astype(np.int32), (P, 1))
    mask = rng.random((P, N)) < frac
    lab[mask] = rng.integers(0, N, size=int(mask.sum()), dtype=np.int64).astype(np.int32)
    return lab


def population_mix(seed, planted, P):
    """Equal thirds: uniform over [0,N), planted with 5%
    re-drawn, uniform over 20 labels.  Rows are interleaved so every block of
    consecutive chromosomes sees all three kinds."""
    rng = np.random.Generator(np.random.PCG64(seed))
    N = planted.shape[0]
    parts = [random_labels(rng, P, N), perturbed_planted(rng, planted, P),
             random_labels(rng, P, N, K=min(20, N))]
    kind = np.arange(P) % 3
    out = np.empty((P, N), np.int32)
    for k in range(3):
        out[kind == k] = parts[k][kind == k]
    return out


def adversarial_population(N):
    """Edge populations: all singletons, one big cluster, every gene on the
    largest label, alternating two labels, a single pair."""
    rows = [np.arange(N), np.zeros(N), np.full(N, N - 1), np.arange(N) % 2]
    pair = np.arange(N)
    if N >= 2:
        pair[1] = 0
    rows.append(pair)
    return np.asarray(rows, np.int32)


# ---------------------------------------------------------------------------
# F1: the paper's test-set shape -- many windows of
# 18 stocks, each clustered by its own GA (1760 matrices from 3-minute
# bars; Table 3 GA configuration).  Reading Q29: the
# paper does not give the window length; a trading day of 3-minute bars
# (8 h -> T = 160) is used.  Per window: 2..4 planted clusters of 2..7 stocks,
# loadings g ~ U(0.55, 0.85), the remaining stocks independent.
# ---------------------------------------------------------------------------
F1 = dict(B=1760, N=18, T=160, seed0=1_760_000, pop=1000, gens=400)


def window_spec(b: int, N: int = 18, T: int = 160, seed0: int = 1_760_000) -> PlantedSpec:
    rng = np.random.Generator(np.random.PCG64(seed0 + b))
    k = int(rng.integers(2, 5))
    sizes = []
    for _ in range(k):
        n = int(rng.integers(2, 8))
        if sum(sizes) + n > N:
            break
        sizes.append(n)
    g = tuple(float(x) for x in rng.uniform(0.55, 0.85, len(sizes)))
    return PlantedSpec(tuple(sizes), g, T, seed0 + b, singletons=N - sum(sizes))


def window_returns(B: int, N: int = 18, T: int = 160, seed0: int = 1_760_000):
    """Returns X [B][T][N] and planted labels [B][N] (0-based canonical)."""
    X = np.empty((B, T, N))
    planted = np.empty((B, N), np.int32)
    for b in range(B):
        X[b], planted[b] = noh_returns(window_spec(b, N, T, seed0))
    return X, planted


def stream_returns(T: int, N: int = 18, seed: int = 1_800_000):
    """A continuous return stream for the correlation stream (f4): the Noh
    model (Eq. 2) with one fixed planted structure drawn like an F1 window
    (window_spec), T observations.  Returns (X [T][N], planted [N])."""
    spec = window_spec(0, N, T, seed)
    return noh_returns(spec)
