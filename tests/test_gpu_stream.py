"""Correlation stream (include/pga.h pga_corr_stream) vs
oracle/stream.py: the EWMA recurrences and the uncleaned correlation are
bit-identical; the RMT-cleaned windows agree to 1e-10 (different
eigensolvers; band membership margins checked); the windows feed the
batched GA, which then matches orc_run window by window."""
import numpy as np
import pytest

import workloads
from oracle import stream as ost

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pga():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1403_4099_b200 import build
    build.build()
    import paper_1403_4099_b200 as p
    return p


@pytest.mark.parametrize("N,lam,warm,stride", [(1, 0.98, 10, 3), (5, 0.9, 50, 7), (18, 0.98, 160, 10),
                                               (37, 0.95, 100, 1), (64, 0.98, 200, 25)])
def test_stream_uncleaned_bit_exact(pga, N, lam, warm, stride):
    X, _ = workloads.stream_returns(600, N, seed=900 + N)
    g = pga.pga_corr_stream(X, lam=lam, warm=warm, stride=stride, q=-1.0)
    o = ost.corr_stream(X, lam=lam, warm=warm, stride=stride, clean=False)
    assert g.shape == o.shape
    assert np.array_equal(g, o)


@pytest.mark.parametrize("N,T", [(18, 1150), (10, 700), (32, 900), (64, 1200)])
def test_stream_cleaned_matches_oracle(pga, N, T):
    X, _ = workloads.stream_returns(T, N, seed=77 + N)
    warm, stride, lam = 160, 10, 0.98
    q = N * (1 - lam)
    g = pga.pga_corr_stream(X, lam=lam, warm=warm, stride=stride, q=0.0)
    o = ost.corr_stream(X, lam=lam, warm=warm, stride=stride, q=q)
    raw = ost.corr_stream(X, lam=lam, warm=warm, stride=stride, clean=False)
    lo, hi = ost.mp_band(q)
    checked = 0
    for b in range(o.shape[0]):
        w = np.linalg.eigvalsh(raw[b])
        if np.min(np.abs(np.concatenate([w - lo, w - hi]))) < 1e-8:
            continue            # band membership too close to call in fp64
        checked += 1
        assert np.max(np.abs(g[b] - o[b])) <= 1e-10, b
        assert np.array_equal(g[b], g[b].T)
        assert np.all(np.diag(g[b]) == 1.0)
    assert checked >= 0.9 * o.shape[0]


def test_stream_device_path(pga):
    import torch
    X, _ = workloads.stream_returns(500, 18, seed=5)
    host = pga.pga_corr_stream(X, q=0.0)
    B = host.shape[0]
    dX = torch.from_numpy(X).cuda()
    dC = torch.zeros((B, 18, 18), dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    pga.pga_corr_stream_device(dX, dC, st, q=0.0, stream=s.cuda_stream)
    assert int(st.item()) == 0
    assert np.array_equal(dC.cpu().numpy(), host)


def test_stream_zero_variance(pga):
    X = np.zeros((300, 4))
    X[:, 1:] = np.random.default_rng(0).standard_normal((300, 3))
    with pytest.raises(pga.PgaError) as e:
        pga.pga_corr_stream(X, warm=100, stride=50)
    assert e.value.code == pga.binding.PGA_ENUMERIC


def test_stream_feeds_batched_ga(pga, orc):
    """returns -> EWMA/RMT windows (device) -> batched GA (device): every
    window's GA equals orc_run on that window's matrix."""
    X, planted = workloads.stream_returns(160 + 10 * 7, 18, seed=31)
    C = pga.pga_corr_stream(X, q=0.0)
    params = pga.pga_params_default(pop_size=200, max_gens=80, seed=9)
    res = pga.pga_batch_run(C, params)
    for b in range(C.shape[0]):
        ref = orc.run(C[b], orc.default_params(pop=200, max_gens=80, seed=9 + b))
        assert np.array_equal(res["best_labels"][b] - 1, ref["best_labels"])
        assert res["gens"][b] == ref["gens_run"]
