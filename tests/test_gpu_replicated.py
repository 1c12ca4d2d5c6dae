"""Replicated master-slave on one GPU: W replica contexts
in ONE process, driven step by step in sequence (no rank waits on another),
each evaluating only its shard through pga_rep_evaluate; the shards are
concatenated (what the all-gather produces) and committed to every replica.
Every replica must reproduce the single-GPU pga_run bit for bit (history,
best labels, population)."""
import numpy as np
import pytest

import workloads

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


@pytest.mark.parametrize("cfg,P,W,gens", [("C1", 128, 2, 40), ("C1", 100, 3, 20),
                                         ("C3", 4096, 2, 15), ("C4", 8192, 4, 6)])
def test_replicas_equal_single_gpu_run(pga, orc, cfg, P, W, gens):
    import torch
    from paper_1403_4099_b200.replicated import GpuReplica, shard
    X, _ = workloads.noh_returns(workloads.CONFIGS[cfg])
    C = orc.pearson(X)
    N = C.shape[0]
    pm = 0.1 if N <= 40 else 2.0 / N
    params = pga.pga_params_default(pop_size=P, p_mutation=pm, max_gens=gens, tol=-1.0, seed=3)
    ref_ctx = pga.pga_create(C, params)
    try:
        # bit-identity with one GPU needs the path choice to be a function of
        # the block alone: the label-sparse pass's launch-history shortcuts are off
        pga.pga_set_sparse_threshold(ref_ctx, 0.0)
        ref = pga.pga_run(ref_ctx, gens, 3, N)
        ref_hist = pga.pga_get_history(ref_ctx, gens)
        ref_pop, ref_L = pga.pga_get_population(ref_ctx, P, N)
    finally:
        pga.pga_destroy(ref_ctx)

    reps = [GpuReplica(C, params) for _ in range(W)]
    try:
        for r in reps:
            pga.pga_set_sparse_threshold(r.ctx, 0.0)
            r.init(3)
        S = shard(P, W, 0)[2]
        L_all = torch.zeros(S * W, dtype=torch.float64, device="cuda")
        t_all = torch.zeros(S * W, dtype=torch.int16, device="cuda")
        for g in range(gens):
            for k, r in enumerate(reps):
                b, e, _ = shard(P, W, k)
                if e > b:
                    with torch.cuda.stream(r.stream):
                        r.rep_evaluate(b, e, L_all[k * S:k * S + (e - b)], t_all[k * S:k * S + (e - b)])
                    r.stream.synchronize()
            for r in reps:
                r.rep_commit(L_all[:P], t_all[:P])
                r.gen_breed()
                r.stream.synchronize()
        for r in reps:
            hist = pga.pga_get_history(r.ctx, gens)
            assert np.array_equal(hist, ref_hist)
            st = r.state()
            assert st["best_L"] == ref["best_L"]
            assert np.array_equal(st["best_labels"], ref["best_labels"])
            pop, L = pga.pga_get_population(r.ctx, P, N)
            assert np.array_equal(pop, ref_pop)
            assert np.array_equal(L, ref_L)
    finally:
        for r in reps:
            r.close()


def test_rep_validation(pga, orc):
    import torch
    C = np.eye(6)
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=64))
    try:
        L = torch.zeros(64, dtype=torch.float64, device="cuda")
        t = torch.zeros(64, dtype=torch.int16, device="cuda")
        with pytest.raises(pga.PgaError):            # no population yet
            pga.pga_rep_evaluate(ctx, 0, 32, L, t)
        pga.pga_init(ctx, 1)
        with pytest.raises(pga.PgaError):            # begin not a multiple of 32
            pga.pga_rep_evaluate(ctx, 5, 40, L, t)
        with pytest.raises(pga.PgaError):            # end beyond pop_size
            pga.pga_rep_evaluate(ctx, 32, 96, L, t)
    finally:
        pga.pga_destroy(ctx)
