"""Independent numpy formulation of Eq. 5/6 used to pin the C oracle.

TEST INFRASTRUCTURE ONLY.  With Z the N x K one-hot membership matrix of a
partition, n = Z^T 1 (Eq. 5) and c = diag(Z^T C Z) (Eq. 6,
P:96-99).  This is a different formulation from oracle.c's double loop, so a
dropped diagonal, a transposed index or a wrong membership test in either
would show up as a mismatch.
"""
import numpy as np


def one_hot(labels, K=None):
    labels = np.asarray(labels, np.int64)
    K = int(labels.max()) + 1 if K is None else K
    Z = np.zeros((labels.shape[0], K), np.float64)
    Z[np.arange(labels.shape[0]), labels] = 1.0
    return Z


def cluster_stats(C, labels):
    Z = one_hot(labels)
    n = Z.sum(axis=0).astype(np.int64)
    c = np.einsum("ik,ij,jk->k", Z, np.asarray(C, np.float64), Z)
    return n, c


def block_closed_form(n, rho):
    """L of one planted block of size n with constant off-diagonal rho
    (c = n + n(n-1) rho in Eq. 8):  1/2 [-(n-1) ln(1-rho) - ln(1+(n-1) rho)].
    Derived by hand from Eq. 8; valid for rho > 0."""
    return 0.5 * (-(n - 1) * np.log1p(-rho) - np.log1p((n - 1) * rho))


def bell(n):
    """Bell numbers via the Bell triangle (pins the partition enumeration)."""
    row = [1]
    out = [1]
    for _ in range(n):
        nxt = [row[-1]]
        for v in row:
            nxt.append(nxt[-1] + v)
        row = nxt
        out.append(row[0])
    return out
