"""Device-side invariant checks -- the substitute for compute-sanitizer,
which the GPU pool does not allow (SURVEY §4 layer 6).
The library is rebuilt with -DPGA_DEVICE_CHECKS (paper_1403_4099_b200/
libpga_check.so, built by __graft_entry__.build()); every hot kernel counts
violated index/range invariants (shared-memory table indices, ordinals,
walk ranges, ranks, merge positions, SUS segments) in device counters.
tools/sanitize.py drives every kernel family on small inputs, checks the
results against the oracle, and must end with zero violations.  A second
part checks run-to-run bit-identity of the kernels that use atomics and
last-CTA reductions (a race would show as nondeterminism)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pga():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1403_4099_b200 import build
    build.build()
    import paper_1403_4099_b200 as p
    return p


def test_device_invariants_clean():
    from paper_1403_4099_b200 import build
    lib = build.build_check()
    env = dict(os.environ, PGA_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py")], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "device invariant violations: 0" in r.stdout, r.stdout[-1000:]


@pytest.mark.parametrize("cfg,P,theta", [("C4", 8192, -1.0), ("C4", 2048, 1.0), ("C3", 4096, 0.0),
                                         ("C5", 512, 1.0)])
def test_atomic_kernels_bit_identical_run_to_run(pga, orc, cfg, P, theta):
    """k_fitness (last-CTA fold with shared atomics), k_fitness_sparse
    (shared atomics, cache CAS, relaxed loads), k_stats (last-CTA
    reduction), the breed's last-CTA advance: ten GA generations twice
    from the same seed give bit-identical populations, L and state."""
    X, _ = workloads.noh_returns(workloads.CONFIGS[cfg])
    C = orc.pearson(X)
    N = C.shape[0]
    out = []
    for _ in range(2):
        ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=50,
                                                       seed=77))
        try:
            pga.pga_set_sparse_threshold(ctx, theta)
            pga.pga_init(ctx, 77)
            for _ in range(10):
                pga.pga_gen_evaluate(ctx)
                pga.pga_gen_breed(ctx)
            pga.pga_gen_evaluate(ctx)
            lab, L, top = pga.pga_get_population(ctx, with_top=True)
            st = pga.pga_get_state(ctx)
            out.append((lab, L, top, st["best_L"], st["mean_L"], st["generation"]))
        finally:
            pga.pga_destroy(ctx)
    a, b = out
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_fast_ln_matches_libm(pga):
    """The label-sparse pass's table-driven ln (fitness.cu fast_ln) against
    numpy's correctly rounded log over the range the Eq. 8 terms use
    (c in (2, 4.2e6), n^2 - c down to 1e-9): a few ulp of the result, far
    inside the 1e-9 max(1, |L|) parity bound."""
    rng = np.random.default_rng(5)
    x = np.concatenate([np.exp(rng.uniform(np.log(1e-9), np.log(5e6), 200000)),
                        2.0 ** np.arange(-30, 23), np.nextafter(2.0 ** np.arange(-30, 23), 0),
                        1.0 + (np.arange(129) / 128.0), 1.0 + (np.arange(128) + 0.5) / 128.0,
                        np.array([1.0, 2.0, 3.0, 1e-9, 4.2e6])])
    ctx = pga.pga_create(np.eye(4), pga.pga_params_default(pop_size=4, elite=1))
    try:
        got = pga.pga_op_fast_ln(ctx, x)
    finally:
        pga.pga_destroy(ctx)
    want = np.log(x)
    err = np.abs(got - want)
    assert err.max() <= 4e-16 * np.maximum(1.0, np.abs(want)).max()
    assert (err <= 8 * np.spacing(np.maximum(np.abs(want), 1e-300)) + 3e-16).all()
