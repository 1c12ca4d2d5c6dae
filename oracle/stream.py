"""Oracle of the on-device correlation stream.

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may use it; the product path never does).  Plain numpy fp64,
one function per step of the paper's pre-processing (§4.2.5):
"a covariance matrix was then computed using an iterative online
exponentially-weighted moving average (EWMA) filter with a default forgetting
factor of lambda = 0.98.  The correlation matrix was computed from the
covariance matrix and was cleaned using random matrix theory methods ...
eliminating eigenvalues in the Wishart range in a trace-preserving manner."
The operations and their order follow SPEC.md: ewma_update,
correlation_from_covariance, rmt_clean.  Readings (Q31-Q33): zero
initial state; emission after observation t = warm-1 + b*stride; the
Marchenko-Pastur ratio q = N (1 - lambda) (effective sample 1/(1-lambda),
S:307) unless given; in-band eigenvalues replaced by their mean; the
reconstruction renormalised to a unit diagonal from its upper triangle.
numpy.linalg.eigh is the library step for the eigendecomposition.
"""
import numpy as np


def ewma_update(mean, cov, x, lam):
    """d = x - mean_prev; cov <- lam cov + (1-lam) d d^T;
    mean <- lam mean + (1-lam) x.  Elementwise in this exact operation order
    (no fused multiply-add)."""
    oml = 1.0 - lam
    d = x - mean
    cov = lam * cov + oml * np.outer(d, d)
    mean = lam * mean + oml * x
    return mean, cov


def correlation_from_covariance(cov):
    """C_ij = cov_ij / sqrt(cov_ii cov_jj), unit diagonal exactly."""
    dg = np.diag(cov).copy()
    if np.any(~(dg > 0)):
        raise ValueError("non-positive variance at index %d" % int(np.argmin(dg)))
    C = cov / np.sqrt(np.outer(dg, dg))
    np.fill_diagonal(C, 1.0)
    return C


def mp_band(q):
    """Marchenko-Pastur support [(1 - sqrt q)^2, (1 + sqrt q)^2]."""
    r = np.sqrt(q)
    return (1.0 - r) ** 2, (1.0 + r) ** 2


def rmt_filter(C, q):
    """eigenvalues inside the Marchenko-Pastur band are replaced by
    their average (trace preserving); returns V diag(w') V^T."""
    w, V = np.linalg.eigh(C)
    lo, hi = mp_band(q)
    band = (w >= lo) & (w <= hi)
    w2 = w.copy()
    if band.any():
        w2[band] = w[band].mean()
    return (V * w2) @ V.T


def unit_diagonal(C2):
    """C''_ij = C'_ij / sqrt(C'_ii C'_jj) from the upper triangle,
    mirrored, unit diagonal."""
    dg = np.diag(C2).copy()
    N = C2.shape[0]
    out = np.eye(N)
    iu = np.triu_indices(N, 1)
    out[iu] = C2[iu] / np.sqrt(dg[iu[0]] * dg[iu[1]])
    out[(iu[1], iu[0])] = out[iu]
    return out


def rmt_clean(C, q):
    """rmt_filter then unit_diagonal."""
    return unit_diagonal(rmt_filter(C, q))


def n_emitted(T, warm, stride):
    return 0 if T < warm else (T - warm) // stride + 1


def corr_stream(X, lam=0.98, warm=160, stride=10, q=None, clean=True):
    """Returns X [T][N] -> C [B][N][N]: the EWMA state after observation
    t = warm-1 + b*stride, converted to a correlation matrix and (clean=True)
    RMT-cleaned.  q=None: q = N (1 - lam)."""
    X = np.asarray(X, np.float64)
    T, N = X.shape
    B = n_emitted(T, warm, stride)
    q = N * (1.0 - lam) if q is None else q
    mean = np.zeros(N)
    cov = np.zeros((N, N))
    out = np.zeros((B, N, N))
    b = 0
    for t in range(T):
        mean, cov = ewma_update(mean, cov, X[t], lam)
        if b < B and t == warm - 1 + b * stride:
            C = correlation_from_covariance(cov)
            out[b] = rmt_clean(C, q) if clean else C
            b += 1
    return out
