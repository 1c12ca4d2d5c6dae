"""CPU oracle for the Giada–Marsili PGA hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1403_4099_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``oracle.c`` (plain fp64 C, each function
citing PAPER.md); this module only marshals arguments through ctypes, and
``npref.py`` holds an independent numpy one-hot formulation used as a pin.

Parity-unpinned items: GPU-vs-oracle parity inside the
c_s -> n_s^2 clamp region (Q3; the oracle's clamp itself is pinned by
properties) and the knowledge-based crossover's fidelity to the
(unavailable) thesis operator (Q12).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

TAG_INIT, TAG_SUS, TAG_PERM, TAG_TOUR, TAG_XO, TAG_MUT, TAG_MUTV = 1, 2, 3, 4, 5, 6, 7


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc (no -ffast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call([
            "gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off",
            "-fno-fast-math", "-Wall", "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


class Params(ct.Structure):
    """Mirror of the oracle's own ``orc_params`` (Table 3 defaults)."""
    _fields_ = [
        ("pop", ct.c_int32), ("elite", ct.c_int32), ("p_c", ct.c_double),
        ("p_m", ct.c_double), ("p_kb", ct.c_double), ("tol", ct.c_double),
        ("stall_gens", ct.c_int32), ("max_gens", ct.c_int32),
        ("selection", ct.c_int32), ("tour_k", ct.c_int32), ("scaling", ct.c_int32),
        ("n_islands", ct.c_int32), ("migrate_every", ct.c_int32),
        ("migrants", ct.c_int32), ("seed", ct.c_uint64),
    ]


def default_params(**kw) -> Params:
    p = Params(pop=1000, elite=10, p_c=0.9, p_m=0.1, p_kb=0.9, tol=1e-5,
               stall_gens=50, max_gens=400, selection=0, tour_k=2, scaling=0,
               n_islands=1, migrate_every=10, migrants=10, seed=1)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


_lib = None


def lib():
    global _lib
    if _lib is None:
        l = ct.CDLL(build())
        D, I32, I64, U32, U64 = ct.c_double, ct.c_int32, ct.c_int64, ct.c_uint32, ct.c_uint64
        P = ct.c_void_p
        sig = {
            "orc_philox4x32_10": (None, [P, P, P]),
            "orc_cluster_stats": (None, [P, I32, P, I32, P, P]),
            "orc_cluster_term": (D, [I64, D]),
            "orc_log_likelihood": (D, [P, I32, P, P]),
            "orc_evaluate": (None, [P, I32, P, I64, P, P, I32]),
            "orc_canonicalize_batch": (None, [P, I64, I32]),
            "orc_brute_force": (I64, [P, I32, P, P]),
            "orc_init_population": (None, [U64, I32, I64, I64, U32, P]),
            "orc_order": (None, [P, I32, P]),
            "orc_num_offspring": (I32, [I32, I32]),
            "orc_select": (None, [P, P, I32, I32, I32, I32, I32, U64, U32, U32, P]),
            "orc_mates": (None, [I32, U64, U32, U32, P]),
            "orc_breed": (None, [P, P, P, I32, I32, I32, P, P, D, D, D, U64, U32, U32, I64, P]),
            "orc_step": (None, [P, I32, P, P, P, U32, U32, I64, P]),
            "orc_migrate": (None, [I32, I32, I32, I32, P, P, P]),
            "orc_run": (I32, [P, I32, P, P, P, P, P, P, I32]),
            "orc_pearson": (I32, [P, I32, I32, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ct.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# thin marshalling wrappers (no arithmetic here)
# ---------------------------------------------------------------------------

def philox(ctr, key) -> np.ndarray:
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def cluster_stats(C, labels):
    C = _c(C, np.float64)
    s = _c(labels, np.int32)
    K = int(s.max()) + 1
    n = np.zeros(K, np.int64)
    c = np.zeros(K, np.float64)
    lib().orc_cluster_stats(_p(C), C.shape[0], _p(s), K, _p(n), _p(c))
    return n, c


def cluster_term(n_s: int, c_s: float) -> float:
    return lib().orc_cluster_term(int(n_s), float(c_s))


def log_likelihood(C, labels):
    """(L, top) for one chromosome; top = -1 if no cluster has f_s > 0."""
    C = _c(C, np.float64)
    s = _c(labels, np.int32)
    top = ct.c_int32(0)
    L = lib().orc_log_likelihood(_p(C), C.shape[0], _p(s), ct.byref(top))
    return L, top.value


def evaluate(C, labels, nthreads: int = 1):
    C = _c(C, np.float64)
    lab = _c(labels, np.int32)
    P, N = lab.shape
    L = np.zeros(P, np.float64)
    top = np.zeros(P, np.int32)
    lib().orc_evaluate(_p(C), N, _p(lab), P, _p(L), _p(top), int(nthreads))
    return L, top


def canonicalize(labels) -> np.ndarray:
    lab = np.array(labels, dtype=np.int32, copy=True, order="C")
    two_d = lab.ndim == 2
    if not two_d:
        lab = lab[None, :]
    lib().orc_canonicalize_batch(_p(lab), lab.shape[0], lab.shape[1])
    return lab if two_d else lab[0]


def brute_force(C):
    C = _c(C, np.float64)
    N = C.shape[0]
    best = np.zeros(N, np.int32)
    L = ct.c_double(0)
    count = lib().orc_brute_force(_p(C), N, _p(best), ct.byref(L))
    return best, L.value, count


def init_population(seed: int, N: int, P: int, p_off: int = 0, island: int = 0):
    out = np.zeros((P, N), np.int32)
    lib().orc_init_population(seed, N, P, p_off, island, _p(out))
    return out


def order(L):
    L = _c(L, np.float64)
    o = np.zeros(L.shape[0], np.int32)
    lib().orc_order(_p(L), L.shape[0], _p(o))
    return o


def num_offspring(P: int, E: int) -> int:
    return lib().orc_num_offspring(P, E)


def select(L, E, selection=0, tour_k=2, scaling=0, seed=1, gen=0, island=0):
    L = _c(L, np.float64)
    P = L.shape[0]
    o = order(L)
    M = num_offspring(P, E)
    sel = np.zeros(M, np.int32)
    lib().orc_select(_p(L), _p(o), P, E, selection, tour_k, scaling, seed, gen, island, _p(sel))
    return o, sel


def mates(M, seed=1, gen=0, island=0):
    sigma = np.zeros(M, np.int32)
    lib().orc_mates(M, seed, gen, island, _p(sigma))
    return sigma


def breed(pop, top, order_, E, sel, sigma, p_c, p_m, p_kb, seed=1, gen=0, island=0, p_off=0):
    pop = _c(pop, np.int32)
    P, N = pop.shape
    top = _c(top, np.int32)
    order_ = _c(order_, np.int32)
    sel = _c(sel, np.int32)
    sigma = _c(sigma, np.int32)
    nxt = np.zeros_like(pop)
    lib().orc_breed(_p(pop), _p(top), _p(order_), P, N, E, _p(sel), _p(sigma),
                    p_c, p_m, p_kb, seed, gen, island, p_off, _p(nxt))
    return nxt


def step(params: Params, pop, L, top, gen, island=0, p_off=0):
    pop = _c(pop, np.int32)
    L = _c(L, np.float64)
    top = _c(top, np.int32)
    nxt = np.zeros_like(pop)
    lib().orc_step(ct.byref(params), pop.shape[1], _p(pop), _p(L), _p(top), gen, island,
                   p_off, _p(nxt))
    return nxt


def migrate(pops, Ls, tops, migrants):
    """In place on lists of numpy arrays (one per island)."""
    G = len(pops)
    P, N = pops[0].shape
    arrs = [(_c(p, np.int32), _c(l, np.float64), _c(t, np.int32)) for p, l, t in zip(pops, Ls, tops)]
    PP = (ct.c_void_p * G)(*[a[0].ctypes.data for a in arrs])
    LL = (ct.c_void_p * G)(*[a[1].ctypes.data for a in arrs])
    TT = (ct.c_void_p * G)(*[a[2].ctypes.data for a in arrs])
    lib().orc_migrate(G, P, N, migrants, PP, LL, TT)
    return [a[0] for a in arrs], [a[1] for a in arrs], [a[2] for a in arrs]


def run(C, params: Params, nthreads: int = 1):
    C = _c(C, np.float64)
    N = C.shape[0]
    best = np.zeros(N, np.int32)
    L = ct.c_double(0)
    gens = ct.c_int32(0)
    reason = ct.c_int32(0)
    hist = np.zeros(max(1, params.max_gens), np.float64)
    rc = lib().orc_run(_p(C), N, ct.byref(params), _p(best), ct.byref(L), ct.byref(gens),
                       ct.byref(reason), _p(hist), int(nthreads))
    if rc != 0:
        raise ValueError("orc_run rejected its arguments")
    return dict(best_labels=best, best_L=L.value, gens_run=gens.value,
                reason=reason.value, history=hist[: gens.value].copy())


def pearson(X):
    X = _c(X, np.float64)
    T, N = X.shape
    C = np.zeros((N, N), np.float64)
    rc = lib().orc_pearson(_p(X), T, N, _p(C))
    if rc != 0:
        raise ValueError("zero-variance or non-finite column")
    return C
