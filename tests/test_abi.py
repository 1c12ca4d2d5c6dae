"""The C-ABI library loads, exports every symbol include/pga.h declares, and
validates arguments before touching a device (CPU only, no compute calls)."""
import ctypes as ct
import os
import re

import numpy as np
import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def pga():
    from paper_1403_4099_b200 import build
    build.build()
    import paper_1403_4099_b200 as p
    p.lib()
    return p


def _declared():
    src = open(os.path.join(ROOT, "include", "pga.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pga_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_survey_boundary():
    names = _declared()
    for n in ["pga_create", "pga_evaluate", "pga_generation", "pga_run", "pga_correlation",
              "pga_destroy", "pga_last_error", "pga_params_default"]:
        assert n in names


def test_every_declared_symbol_is_exported(pga):
    raw = ct.CDLL(pga.binding.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(raw, n)]
    assert not missing, missing


def test_binding_covers_every_symbol(pga):
    for n in _declared():
        assert n in pga.binding._SIGS, n


def test_params_default_is_table3(pga):
    p = pga.pga_params_default()
    assert (p.elite, p.p_crossover, p.p_mutation, p.p_kb, p.tol, p.stall_gens, p.max_gens) == \
        (10, 0.9, 0.1, 0.9, 1e-5, 50, 400)


@pytest.mark.parametrize("kw,msg", [
    (dict(pop_size=1), "pop_size"),
    (dict(elite=1000), "elite"),
    (dict(p_mutation=1.5), "probabilities"),
    (dict(selection=7), "selection"),
    (dict(tournament_k=9), "tournament_k"),
    (dict(n_islands=9), "n_islands"),
    (dict(island=3, n_islands=2), "island"),
])
def test_param_validation(pga, kw, msg):
    with pytest.raises(pga.PgaError) as e:
        pga.pga_create(np.eye(4), pga.pga_params_default(**kw))
    assert e.value.code == pga.binding.PGA_EINVAL and msg in str(e.value)


def test_corr_validation(pga):
    bad = np.eye(4)
    bad[0, 1] = 0.3            # not symmetric
    with pytest.raises(pga.PgaError, match="symmetric"):
        pga.pga_create(bad, pga.pga_params_default())
    bad = np.eye(4) * 1.1      # diagonal != 1
    with pytest.raises(pga.PgaError, match="C_ii"):
        pga.pga_create(bad, pga.pga_params_default())
    bad = np.eye(4)
    bad[1, 2] = bad[2, 1] = 1.5
    with pytest.raises(pga.PgaError, match=r"\|C_ij\|"):
        pga.pga_create(bad, pga.pga_params_default())
    with pytest.raises(pga.PgaError, match="N must"):
        pga.pga_create(np.eye(1), pga.pga_params_default())


def test_no_cpu_fallback(pga):
    """Without a CUDA device the library refuses to compute."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(pga.PgaError) as e:
        pga.pga_create(np.eye(4), pga.pga_params_default())
    assert e.value.code == pga.binding.PGA_EDEVICE
    with pytest.raises(pga.PgaError) as e:
        pga.pga_correlation(np.random.default_rng(0).standard_normal((10, 3)))
    assert e.value.code == pga.binding.PGA_EDEVICE


@pytest.mark.parametrize("N,kw,msg", [
    (33, {}, "2 <= N <= 32"),
    (8, dict(pop_size=4096), "pop_size <= 2048"),
    (8, dict(n_islands=2), "one island per matrix"),
    (8, dict(elite=100), "elite"),
])
def test_batch_validation(pga, N, kw, msg):
    """pga_batch_run validates before touching a device."""
    kw.setdefault("pop_size", 100)
    with pytest.raises(pga.PgaError) as e:
        pga.pga_batch_run(np.stack([np.eye(N)] * 2), pga.pga_params_default(**kw))
    assert e.value.code == pga.binding.PGA_EINVAL and msg in str(e.value)
    bad = np.stack([np.eye(4), np.eye(4)])
    bad[1, 0, 1] = 0.5        # matrix 1 not symmetric
    with pytest.raises(pga.PgaError, match="matrix 1"):
        pga.pga_batch_run(bad, pga.pga_params_default(pop_size=10, elite=2))


def test_corr_stream_validation(pga):
    X = np.random.default_rng(0).standard_normal((50, 4))
    for kw, msg in [(dict(lam=1.0), "lambda"), (dict(warm=0), "warm"), (dict(warm=60), "T >= warm"),
                    (dict(stride=0), "stride")]:
        with pytest.raises(pga.PgaError) as e:
            pga.pga_corr_stream(X, **{**dict(warm=10, stride=5), **kw})
        assert e.value.code == pga.binding.PGA_EINVAL
    with pytest.raises(pga.PgaError, match="1 <= N <= 64"):
        pga.pga_corr_stream(np.zeros((20, 65)), warm=5, stride=5)
    assert pga.pga_stream_count(57, 20, 9) == 5
