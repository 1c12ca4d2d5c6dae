"""Thin ctypes binding of libpga.so (include/pga.h) — argument marshalling only.

Every function here has the name of the C entry point it wraps and does no
arithmetic of the method: it converts numpy / torch arguments to pointers,
calls the library and turns negative return codes into ``PgaError``.  There
is no CPU fallback: if libpga.so is missing or no CUDA device exists the
calls fail loudly.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PGA_LIB") or os.path.join(_HERE, "libpga.so")

PGA_OK, PGA_EINVAL, PGA_ENOMEM, PGA_EDEVICE, PGA_ENUMERIC, PGA_ESTATE = 0, -1, -2, -3, -4, -5
PGA_SEL_SUS, PGA_SEL_TOURNAMENT = 0, 1
PGA_SCALE_RANK, PGA_SCALE_NONE = 0, 1
_CODES = {-1: "PGA_EINVAL", -2: "PGA_ENOMEM", -3: "PGA_EDEVICE", -4: "PGA_ENUMERIC", -5: "PGA_ESTATE"}


class PgaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s: %s" % (_CODES.get(code, code), msg))
        self.code = code


class pga_params(ct.Structure):
    _fields_ = [
        ("pop_size", ct.c_int32), ("elite", ct.c_int32), ("p_crossover", ct.c_double),
        ("p_mutation", ct.c_double), ("p_kb", ct.c_double), ("tol", ct.c_double),
        ("stall_gens", ct.c_int32), ("max_gens", ct.c_int32), ("selection", ct.c_int32),
        ("tournament_k", ct.c_int32), ("scaling", ct.c_int32), ("device", ct.c_int32),
        ("island", ct.c_int32), ("n_islands", ct.c_int32), ("migrate_every", ct.c_int32),
        ("migrants", ct.c_int32), ("seed", ct.c_uint64),
    ]


_lib = None

_SIGS = {
    "pga_params_default": (ct.c_int, [ct.c_void_p]),
    "pga_create": (ct.c_int, [ct.c_void_p, ct.c_int32, ct.c_void_p, ct.c_void_p]),
    "pga_destroy": (None, [ct.c_void_p]),
    "pga_last_error": (ct.c_char_p, []),
    "pga_evaluate": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_void_p]),
    "pga_evaluate_device": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_void_p,
                                       ct.c_void_p, ct.c_void_p]),
    "pga_init": (ct.c_int, [ct.c_void_p, ct.c_uint64]),
    "pga_gen_evaluate": (ct.c_int, [ct.c_void_p, ct.c_void_p]),
    "pga_gen_breed": (ct.c_int, [ct.c_void_p]),
    "pga_generation": (ct.c_int, [ct.c_void_p, ct.c_void_p]),
    "pga_run": (ct.c_int, [ct.c_void_p, ct.c_int32, ct.c_uint64, ct.c_void_p, ct.c_void_p,
                           ct.c_void_p, ct.c_void_p]),
    "pga_get_state": (ct.c_int, [ct.c_void_p] + [ct.c_void_p] * 6),
    "pga_get_history": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_int32]),
    "pga_get_population": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p]),
    "pga_profile_enable": (ct.c_int, [ct.c_void_p, ct.c_int32]),
    "pga_profile_read": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                    ct.c_void_p]),
    "pga_profile_phases": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p]),
    "pga_set_population": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_int32]),
    "pga_migrant_bytes": (ct.c_int, [ct.c_void_p, ct.c_void_p]),
    "pga_export_migrants": (ct.c_int, [ct.c_void_p, ct.c_void_p]),
    "pga_import_migrants": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_int32]),
    "pga_get_stream": (ct.c_int, [ct.c_void_p, ct.c_void_p]),
    "pga_correlation": (ct.c_int, [ct.c_void_p, ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_int32]),
    "pga_correlation_device": (ct.c_int, [ct.c_void_p, ct.c_int32, ct.c_int32, ct.c_void_p,
                                          ct.c_void_p, ct.c_void_p]),
    "pga_op_select": (ct.c_int, [ct.c_void_p, ct.c_int64, ct.c_void_p, ct.c_int32, ct.c_int32,
                                 ct.c_void_p, ct.c_void_p]),
    "pga_op_mates": (ct.c_int, [ct.c_int64, ct.c_void_p, ct.c_int32, ct.c_int32, ct.c_void_p]),
    "pga_op_breed": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_int32,
                                ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_int32, ct.c_int32,
                                ct.c_int64, ct.c_void_p]),
    "pga_op_canonicalize": (ct.c_int, [ct.c_void_p, ct.c_int64, ct.c_int32, ct.c_int32]),
    "pga_op_init": (ct.c_int, [ct.c_uint64, ct.c_int32, ct.c_int64, ct.c_int64, ct.c_int32,
                               ct.c_int32, ct.c_void_p]),
    "pga_launch_count": (ct.c_int64, []),
    "pga_get_dims": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p]),
    "pga_debug_violations": (ct.c_int64, []),
    "pga_op_fast_ln": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_void_p]),
    "pga_cache_stats": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p]),
    "pga_set_sparse_threshold": (ct.c_int, [ct.c_void_p, ct.c_double]),
    "pga_profile_sparse_blocks": (ct.c_int, [ct.c_void_p, ct.c_void_p]),
    "pga_profile_sparse": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p]),
    "pga_set_cluster_cache": (ct.c_int, [ct.c_void_p, ct.c_int32]),
    "pga_profile_cache": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p]),
    "pga_rep_evaluate": (ct.c_int, [ct.c_void_p, ct.c_int64, ct.c_int64, ct.c_void_p, ct.c_void_p]),
    "pga_rep_commit": (ct.c_int, [ct.c_void_p, ct.c_void_p, ct.c_void_p]),
    "pga_stream_count": (ct.c_int, [ct.c_int32, ct.c_int32, ct.c_int32]),
    "pga_corr_stream": (ct.c_int, [ct.c_void_p, ct.c_int32, ct.c_int32, ct.c_double, ct.c_int32,
                                   ct.c_int32, ct.c_double, ct.c_int32, ct.c_void_p, ct.c_void_p,
                                   ct.c_int32, ct.c_void_p]),
    "pga_batch_run": (ct.c_int, [ct.c_void_p, ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_int32,
                                 ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                 ct.c_void_p]),
    "pga_batch_smem_bytes": (ct.c_int, [ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_void_p]),
    "pga_batch_op_evaluate": (ct.c_int, [ct.c_void_p, ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_int32,
                                         ct.c_int32, ct.c_void_p, ct.c_void_p]),
    "pga_batch_op_step": (ct.c_int, [ct.c_int32, ct.c_int32, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                     ct.c_void_p, ct.c_int32, ct.c_void_p]),
}


def lib():
    """Load libpga.so (no fallback: raises if it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libpga.so not built: run `python -m paper_1403_4099_b200.build` "
                              "(there is no CPU fallback)")
        l = ct.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def _check(rc):
    if rc != PGA_OK:
        raise PgaError(rc, lib().pga_last_error().decode())
    return rc


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ct.c_void_p)
    if hasattr(a, "data_ptr"):  # torch tensor (device pointer)
        if not a.is_contiguous():
            raise ValueError("tensors passed to libpga must be contiguous (row-major)")
        return ct.c_void_p(a.data_ptr())
    return a


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def pga_get_dims(ctx):
    """(N, pop_size, capacity) of a ctx."""
    n, p, c = ct.c_int32(), ct.c_int64(), ct.c_int64()
    _check(lib().pga_get_dims(ctx, ct.byref(n), ct.byref(p), ct.byref(c)))
    return n.value, p.value, c.value


def _need(cond, msg):
    if not cond:
        raise ValueError(msg)


def _dev_tensor(t, dtypes, numel, what):
    """Check a torch CUDA tensor argument before its pointer crosses the ABI."""
    _need(hasattr(t, "data_ptr") and getattr(t, "is_cuda", False), "%s must be a CUDA tensor" % what)
    _need(str(t.dtype).replace("torch.", "") in dtypes, "%s must have dtype %s (got %s)"
          % (what, "/".join(dtypes), t.dtype))
    _need(t.numel() >= numel, "%s holds %d elements, needs %d" % (what, t.numel(), numel))


def pga_params_default(**kw) -> pga_params:
    p = pga_params()
    _check(lib().pga_params_default(ct.byref(p)))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise AttributeError(k)
        setattr(p, k, v)
    return p


def pga_create(C, params: pga_params):
    C = _c(C, np.float64)
    ctx = ct.c_void_p()
    _check(lib().pga_create(_p(C), C.shape[0], ct.byref(params), ct.byref(ctx)))
    return ctx


def pga_destroy(ctx):
    lib().pga_destroy(ctx)


def pga_evaluate(ctx, labels_1based) -> np.ndarray:
    lab = _c(labels_1based, np.int32)
    if lab.ndim == 1:
        lab = lab[None, :]
    N = pga_get_dims(ctx)[0]
    _need(lab.ndim == 2 and lab.shape[1] == N, "labels must be [P][%d]" % N)
    L = np.zeros(lab.shape[0], np.float64)
    _check(lib().pga_evaluate(ctx, _p(lab), lab.shape[0], _p(L)))
    return L


CUDA_STREAM_LEGACY = 1   # cudaStreamLegacy: the legacy default stream as an explicit handle


def _caller_stream(stream):
    """The stream a device-pointer call is ordered on: the caller's, else
    torch's current stream (the legacy default stream is passed as
    cudaStreamLegacy, since NULL means the ctx's own stream at this ABI)."""
    if stream is None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream
    return stream if stream else CUDA_STREAM_LEGACY


def pga_evaluate_device(ctx, labels_dev, L_dev, top_dev=None, stream=None):
    """labels_dev: torch uint16-compatible (int16) CUDA tensor [P][N] 0-based.
    Ordered on `stream` (default: torch's current stream, so tensors made
    just before are complete); the library joins it to the ctx's stream."""
    N, _, cap = pga_get_dims(ctx)
    _need(labels_dev.dim() == 2 and labels_dev.shape[1] == N, "labels_dev must be [P][%d]" % N)
    P = labels_dev.shape[0]
    _need(1 <= P <= cap, "P must lie in [1, %d]" % cap)
    _dev_tensor(labels_dev, ("int16", "uint16"), P * N, "labels_dev")
    _need(labels_dev.is_contiguous(), "labels_dev must be contiguous")
    _dev_tensor(L_dev, ("float64",), P, "L_dev")
    if top_dev is not None:
        _dev_tensor(top_dev, ("int16", "uint16"), P, "top_dev")
    _check(lib().pga_evaluate_device(ctx, _p(labels_dev), P, _p(L_dev), _p(top_dev),
                                     ct.c_void_p(_caller_stream(stream))))


def pga_init(ctx, seed: int):
    _check(lib().pga_init(ctx, seed))


def pga_gen_evaluate(ctx) -> bool:
    m = ct.c_int32(0)
    _check(lib().pga_gen_evaluate(ctx, ct.byref(m)))
    return bool(m.value)


def pga_gen_breed(ctx):
    _check(lib().pga_gen_breed(ctx))


def pga_generation(ctx) -> bool:
    d = ct.c_int32(0)
    _check(lib().pga_generation(ctx, ct.byref(d)))
    return bool(d.value)


def pga_run(ctx, gens: int, seed: int, N: int = None):
    N = pga_get_dims(ctx)[0] if N is None else N
    _need(N == pga_get_dims(ctx)[0], "N differs from the ctx's")
    best = np.zeros(N, np.int32)
    L = ct.c_double(0)
    g = ct.c_int32(0)
    r = ct.c_int32(0)
    _check(lib().pga_run(ctx, gens, seed, _p(best), ct.byref(L), ct.byref(g), ct.byref(r)))
    return dict(best_labels=best, best_L=L.value, gens_run=g.value, reason=r.value)


def pga_get_state(ctx, N: int = None):
    N = pga_get_dims(ctx)[0] if N is None else N
    _need(N == pga_get_dims(ctx)[0], "N differs from the ctx's")
    gen, done, reason = ct.c_int32(), ct.c_int32(), ct.c_int32()
    best, mean = ct.c_double(), ct.c_double()
    lab = np.zeros(N, np.int32)
    _check(lib().pga_get_state(ctx, ct.byref(gen), ct.byref(done), ct.byref(reason),
                               ct.byref(best), ct.byref(mean), _p(lab)))
    return dict(generation=gen.value, done=done.value, reason=reason.value, best_L=best.value,
                mean_L=mean.value, best_labels=lab)


def pga_get_history(ctx, n: int) -> np.ndarray:
    h = np.zeros(n, np.float64)
    _check(lib().pga_get_history(ctx, _p(h), n))
    return h


def pga_get_population(ctx, P: int = None, N: int = None, with_top: bool = False):
    Nc, Pc, _ = pga_get_dims(ctx)
    P, N = (Pc if P is None else P), (Nc if N is None else N)
    _need((P, N) == (Pc, Nc), "population is [%d][%d], not [%d][%d]" % (Pc, Nc, P, N))
    lab = np.zeros((P, N), np.int32)
    L = np.zeros(P, np.float64)
    top = np.zeros(P, np.int32)
    _check(lib().pga_get_population(ctx, _p(lab), _p(L), _p(top)))
    return (lab, L, top) if with_top else (lab, L)


def pga_profile_enable(ctx, on=True):
    """on: False/0 off, True/1 fitness + generation events, 2 every phase."""
    _check(lib().pga_profile_enable(ctx, int(on)))


PHASES = ["fitness", "sparse_pass", "stats", "order_sort", "selection", "mates", "breed", "advance"]


def pga_profile_phases(ctx):
    ms = np.zeros(len(PHASES), np.float64)
    n = ct.c_int32()
    _check(lib().pga_profile_phases(ctx, _p(ms), ct.byref(n)))
    return dict(zip(PHASES, ms.tolist())), n.value


def pga_profile_read(ctx):
    s, f, g = ct.c_double(), ct.c_double(), ct.c_double()
    n = ct.c_int32()
    _check(lib().pga_profile_read(ctx, ct.byref(s), ct.byref(f), ct.byref(g), ct.byref(n)))
    return dict(sweep_ms=s.value, fold_ms=f.value, gen_ms=g.value, count=n.value)


def pga_set_population(ctx, labels_1based, generation: int = 0):
    lab = _c(labels_1based, np.int32)
    N, P, _ = pga_get_dims(ctx)
    _need(lab.shape == (P, N), "labels must be [%d][%d]" % (P, N))
    _check(lib().pga_set_population(ctx, _p(lab), generation))


def pga_migrant_bytes(ctx) -> int:
    b = ct.c_int64(0)
    _check(lib().pga_migrant_bytes(ctx, ct.byref(b)))
    return b.value


def pga_export_migrants(ctx, dev_send):
    _check(lib().pga_export_migrants(ctx, _p(dev_send)))


def pga_import_migrants(ctx, dev_recv, n_islands: int):
    _check(lib().pga_import_migrants(ctx, _p(dev_recv), n_islands))


def pga_get_stream(ctx) -> int:
    s = ct.c_void_p()
    _check(lib().pga_get_stream(ctx, ct.byref(s)))
    return s.value or 0


def pga_correlation(returns, device: int = 0) -> np.ndarray:
    X = _c(returns, np.float64)
    T, N = X.shape
    C = np.zeros((N, N), np.float64)
    _check(lib().pga_correlation(_p(X), T, N, _p(C), device))
    return C


def pga_correlation_device(X_dev, C_dev, status_dev, stream=None):
    T, N = X_dev.shape
    _check(lib().pga_correlation_device(_p(X_dev), T, N, _p(C_dev), _p(status_dev),
                                        None if stream is None else ct.c_void_p(stream)))


def pga_op_select(L, params: pga_params, gen: int = 0, island: int = 0):
    L = _c(L, np.float64)
    P = L.shape[0]
    M = 2 * ((P - params.elite + 1) // 2)
    order = np.zeros(P, np.int32)
    sel = np.zeros(M, np.int32)
    _check(lib().pga_op_select(_p(L), P, ct.byref(params), gen, island, _p(order), _p(sel)))
    return order, sel


def pga_op_mates(M: int, params: pga_params, gen: int = 0, island: int = 0):
    sigma = np.zeros(M, np.int32)
    _check(lib().pga_op_mates(M, ct.byref(params), gen, island, _p(sigma)))
    return sigma


def pga_op_breed(pop, top, order, sel, sigma, params: pga_params, gen=0, island=0, p_off=0):
    pop = _c(pop, np.int32)
    P, N = pop.shape
    nxt = np.zeros_like(pop)
    _check(lib().pga_op_breed(_p(pop), _p(_c(top, np.int32)), _p(_c(order, np.int32)), P, N,
                              _p(_c(sel, np.int32)), _p(_c(sigma, np.int32)), ct.byref(params),
                              gen, island, p_off, _p(nxt)))
    return nxt


def pga_op_fast_ln(ctx, x):
    """The sparse pass's table-driven ln (test hook)."""
    x = _c(x, np.float64)
    out = np.zeros_like(x)
    _check(lib().pga_op_fast_ln(ctx, _p(x), x.size, _p(out)))
    return out


def pga_op_canonicalize(labels, device: int = 0):
    lab = np.array(labels, dtype=np.int32, copy=True, order="C")
    two = lab.ndim == 2
    if not two:
        lab = lab[None, :]
    _check(lib().pga_op_canonicalize(_p(lab), lab.shape[0], lab.shape[1], device))
    return lab if two else lab[0]


def pga_op_init(seed: int, N: int, P: int, p_off: int = 0, island: int = 0, device: int = 0):
    out = np.zeros((P, N), np.int32)
    _check(lib().pga_op_init(seed, N, P, p_off, island, device, _p(out)))
    return out


def pga_profile_sparse_blocks(ctx) -> int:
    v = ct.c_int64()
    _check(lib().pga_profile_sparse_blocks(ctx, ct.byref(v)))
    return v.value


def pga_profile_sparse(ctx):
    """(blocks evaluated by the label-sparse pre-pass, C entries it gathered)."""
    v, g = ct.c_int64(), ct.c_int64()
    _check(lib().pga_profile_sparse(ctx, ct.byref(v), ct.byref(g)))
    return v.value, g.value


def pga_set_sparse_threshold(ctx, theta: float):
    """theta: 0 = dense sweep only; 1 = label-sparse whenever N <= 640."""
    _check(lib().pga_set_sparse_threshold(ctx, float(theta)))


def pga_set_cluster_cache(ctx, on: bool):
    """Cluster cache of the label-sparse pass (default on); results are identical either way."""
    _check(lib().pga_set_cluster_cache(ctx, 1 if on else 0))


def pga_cache_stats(ctx):
    """dict(fill, slots, clears) of the cluster cache (slots 0: no cache)."""
    f, s, c = ct.c_int64(), ct.c_int64(), ct.c_int64()
    _check(lib().pga_cache_stats(ctx, ct.byref(f), ct.byref(s), ct.byref(c)))
    return dict(fill=f.value, slots=s.value, clears=c.value)


def pga_profile_cache(ctx):
    """(cluster-cache hits, pair updates they replaced) since profiling was enabled."""
    h, v = ct.c_int64(), ct.c_int64()
    _check(lib().pga_profile_cache(ctx, ct.byref(h), ct.byref(v)))
    return h.value, v.value


def pga_rep_evaluate(ctx, begin: int, end: int, L_dev, top_dev):
    """Fitness of chromosomes [begin, end) into device buffers (torch tensors:
    float64 [end-begin], int16/uint16 [end-begin])."""
    _dev_tensor(L_dev, ("float64",), max(0, end - begin), "L_dev")
    _dev_tensor(top_dev, ("int16", "uint16"), max(0, end - begin), "top_dev")
    _check(lib().pga_rep_evaluate(ctx, begin, end, _p(L_dev), _p(top_dev)))


def pga_rep_commit(ctx, L_dev, top_dev):
    P = pga_get_dims(ctx)[1]
    _dev_tensor(L_dev, ("float64",), P, "L_dev")
    _dev_tensor(top_dev, ("int16", "uint16"), P, "top_dev")
    _check(lib().pga_rep_commit(ctx, _p(L_dev), _p(top_dev)))


def pga_stream_count(T: int, warm: int, stride: int) -> int:
    rc = lib().pga_stream_count(T, warm, stride)
    if rc < 0:
        _check(rc)
    return rc


def pga_corr_stream(X, lam: float = 0.98, warm: int = 160, stride: int = 10, q: float = 0.0,
                    device: int = 0):
    """Host returns X [T][N] -> cleaned correlation windows [B][N][N]
    (include/pga.h pga_corr_stream; q = 0: N (1 - lam), q < 0: no cleaning)."""
    X = _c(X, np.float64)
    T, N = X.shape
    B = pga_stream_count(T, warm, stride)
    out = np.zeros((B, N, N))
    st = ct.c_int32(0)
    _check(lib().pga_corr_stream(_p(X), T, N, lam, warm, stride, q, 0, _p(out), ct.byref(st),
                                 device, None))
    return out


def pga_corr_stream_device(X_dev, C_dev, status_dev, lam: float = 0.98, warm: int = 160,
                           stride: int = 10, q: float = 0.0, device: int = 0, stream=None):
    T, N = X_dev.shape
    _check(lib().pga_corr_stream(_p(X_dev), T, N, lam, warm, stride, q, 1, _p(C_dev), _p(status_dev),
                                 device, None if stream is None else ct.c_void_p(stream)))


def pga_batch_run(C, params: pga_params, history: bool = False):
    """Batched GA over host matrices C [B][N][N] (include/pga.h pga_batch_run).
    Returns dict(best_labels [B][N] 1-based, best_L [B], gens [B], reason [B],
    history [B][max_gens] or None)."""
    C = _c(C, np.float64)
    B, N = C.shape[0], C.shape[1]
    out = dict(best_labels=np.zeros((B, N), np.int32), best_L=np.zeros(B),
               gens=np.zeros(B, np.int32), reason=np.zeros(B, np.int32),
               history=np.zeros((B, params.max_gens)) if history else None)
    _check(lib().pga_batch_run(_p(C), B, N, ct.byref(params), 0, _p(out["best_labels"]),
                               _p(out["best_L"]), _p(out["gens"]), _p(out["reason"]),
                               _p(out["history"]), None))
    return out


def pga_batch_run_device(C_dev, params: pga_params, best_labels_dev, best_L_dev, gens_dev=None,
                         reason_dev=None, history_dev=None, stream=None):
    """Device variant (torch tensors / raw pointers), stream-ordered."""
    B, N = C_dev.shape[0], C_dev.shape[1]
    _check(lib().pga_batch_run(_p(C_dev), B, N, ct.byref(params), 1, _p(best_labels_dev),
                               _p(best_L_dev), _p(gens_dev), _p(reason_dev), _p(history_dev),
                               None if stream is None else ct.c_void_p(stream)))


def pga_batch_smem_bytes(N: int, pop_size: int, elite: int, device: int = 0) -> int:
    v = ct.c_int64()
    _check(lib().pga_batch_smem_bytes(N, pop_size, elite, device, ct.byref(v)))
    return v.value


def pga_batch_op_evaluate(C, labels, device: int = 0):
    C = _c(C, np.float64)
    labels = _c(labels, np.int32)
    B, P, N = labels.shape
    L = np.zeros((B, P))
    top = np.zeros((B, P), np.int32)
    _check(lib().pga_batch_op_evaluate(_p(C), B, N, _p(labels), P, device, _p(L), _p(top)))
    return L, top


def pga_batch_op_step(params: pga_params, pop, L, top, gen: int):
    pop = _c(pop, np.int32)
    B, P, N = pop.shape
    L = _c(L, np.float64)
    top = _c(top, np.int32)
    nxt = np.zeros_like(pop)
    _check(lib().pga_batch_op_step(B, N, ct.byref(params), _p(pop), _p(L), _p(top), gen, _p(nxt)))
    return nxt


def pga_debug_violations() -> int:
    """Device invariant violations so far (-1: product build, checks compiled out)."""
    return lib().pga_debug_violations()


def pga_launch_count() -> int:
    return lib().pga_launch_count()
