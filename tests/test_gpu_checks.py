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
