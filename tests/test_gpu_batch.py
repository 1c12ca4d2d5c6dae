"""Batched GA (include/pga.h pga_batch_*) vs the
oracle: one independent GA per correlation matrix, matrix b under seed + b.

- fitness: |dL| <= 1e-9 max(1, |L|), top label exact (BASELINE.json);
- one generation of operators in lockstep with orc_step: bit-exact;
- whole runs: orc_run(C_b, seed + b) per matrix -- generations, stop
  reason, best labels and best L;
- end to end: planted clusters of the F1 windows recovered."""
import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-9


@pytest.fixture(scope="module")
def pga():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1403_4099_b200 import build
    build.build()
    import paper_1403_4099_b200 as p
    return p


def _windows(orc, B, N=18, T=160, seed0=workloads.F1["seed0"]):
    X, planted = workloads.window_returns(B, N, T, seed0)
    C = np.stack([orc.pearson(X[b]) for b in range(B)])
    return C, planted


def _assert_L(Lg, Lo):
    err = np.abs(np.asarray(Lg) - np.asarray(Lo)) / np.maximum(1.0, np.abs(Lo))
    assert err.max() <= TOL, "max rel err %g at %d" % (err.max(), int(err.argmax()))


def _oparams(orc, P, seed, **kw):
    kw.setdefault("elite", min(10, P - 1))
    return orc.default_params(pop=P, seed=seed, **kw)


def _gparams(pga, P, seed, **kw):
    kw.setdefault("elite", min(10, P - 1))
    return pga.pga_params_default(pop_size=P, seed=seed, **kw)


@pytest.mark.parametrize("N,P", [(2, 3), (5, 64), (18, 1000), (31, 77), (32, 256)])
def test_batch_evaluate_parity(pga, orc, N, P):
    B = 3
    C, planted = _windows(orc, B, N=N, T=max(3 * N, 40))
    labs = np.stack([workloads.population_mix(100 + b, planted[b], P) for b in range(B)])
    adv = workloads.adversarial_population(N)
    labs[:, : min(P, adv.shape[0])] = adv[: min(P, adv.shape[0])]
    Lg, tg = pga.pga_batch_op_evaluate(C, labs)
    for b in range(B):
        Lo, to = orc.evaluate(C[b], labs[b])
        _assert_L(Lg[b], Lo)
        assert np.array_equal(tg[b], to)


def test_batch_evaluate_noncanonical_labels(pga, orc):
    """Labels up to 2N, not canonical: n_s, c_s and the top label (by label
    value, smallest wins ties) follow the definition, not label order."""
    N, P, B = 18, 50, 2
    C, _ = _windows(orc, B, N=N)
    rng = np.random.default_rng(5)
    labs = rng.integers(0, 2 * N + 1, size=(B, P, N)).astype(np.int32)
    labs[:, :, : N // 2] = rng.integers(30, 37, size=(B, P, N // 2))
    Lg, tg = pga.pga_batch_op_evaluate(C, labs)
    for b in range(B):
        Lo, to = orc.evaluate(C[b], labs[b])
        _assert_L(Lg[b], Lo)
        assert np.array_equal(tg[b], to)


@pytest.mark.parametrize("P,E,sel,scal", [(1000, 10, 0, 0), (128, 9, 0, 0), (77, 0, 1, 0),
                                          (64, 5, 0, 1), (2, 1, 0, 0), (2048, 10, 0, 0)])
def test_batch_step_lockstep(pga, orc, P, E, sel, scal):
    """Generations 0..3 in lockstep: the oracle evaluates, both sides breed
    from the same (pop, L, top); children must be identical."""
    B, N, seed = 3, 18, 4242
    C, _ = _windows(orc, B)
    op = [_oparams(orc, P, seed + b, elite=E, selection=sel, scaling=scal) for b in range(B)]
    gp = _gparams(pga, P, seed, elite=E, selection=sel, scaling=scal)
    pops = np.stack([orc.init_population(seed + b, N, P) for b in range(B)])
    for gen in range(4):
        L = np.zeros((B, P))
        top = np.zeros((B, P), np.int32)
        for b in range(B):
            L[b], top[b] = orc.evaluate(C[b], pops[b])
        nxt_g = pga.pga_batch_op_step(gp, pops, L, top, gen)
        nxt_o = np.stack([orc.step(op[b], pops[b], L[b], top[b], gen) for b in range(B)])
        assert np.array_equal(nxt_g, nxt_o), "generation %d differs" % gen
        pops = nxt_o


@pytest.mark.parametrize("P,gens,tol,pm", [(128, 100, 1e-5, 0.1), (300, 60, -1.0, 0.05),
                                           (1000, 400, 1e-5, 0.1)])
def test_batch_run_matches_oracle(pga, orc, P, gens, tol, pm):
    B, seed = 6, 777
    C, _ = _windows(orc, B)
    g = _gparams(pga, P, seed, max_gens=gens, tol=tol, p_mutation=pm)
    res = pga.pga_batch_run(C, g, history=True)
    for b in range(B):
        ref = orc.run(C[b], _oparams(orc, P, seed + b, max_gens=gens, tol=tol, p_m=pm))
        assert res["gens"][b] == ref["gens_run"], b
        assert res["reason"][b] == ref["reason"], b
        assert np.array_equal(res["best_labels"][b] - 1, ref["best_labels"]), b
        _assert_L([res["best_L"][b]], [ref["best_L"]])
        _assert_L(res["history"][b, : ref["gens_run"]], ref["history"])
        assert np.all(res["history"][b, ref["gens_run"]:] == 0.0)
        # the reported L is the fitness of the reported labels
        Lo, _ = orc.log_likelihood(C[b], res["best_labels"][b] - 1)
        _assert_L([res["best_L"][b]], [Lo])


def test_batch_device_path_matches_host(pga, orc):
    import torch
    B, P = 5, 200
    C, _ = _windows(orc, B)
    g = _gparams(pga, P, 31, max_gens=50)
    host = pga.pga_batch_run(C, g, history=True)
    dC = torch.from_numpy(C).cuda()
    lab = torch.zeros((B, 18), dtype=torch.int32, device="cuda")
    bl = torch.zeros(B, dtype=torch.float64, device="cuda")
    gens = torch.zeros(B, dtype=torch.int32, device="cuda")
    reason = torch.zeros(B, dtype=torch.int32, device="cuda")
    hist = torch.zeros((B, 50), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pga.pga_batch_run_device(dC, g, lab, bl, gens, reason, hist, stream=s.cuda_stream)
    s.synchronize()
    assert np.array_equal(lab.cpu().numpy(), host["best_labels"])
    assert np.array_equal(bl.cpu().numpy(), host["best_L"])
    assert np.array_equal(gens.cpu().numpy(), host["gens"])
    assert np.array_equal(hist.cpu().numpy(), host["history"])


def _single_move_improves(orc, C, lab):
    """True if moving one gene to another existing or a fresh cluster raises
    L (the local-optimality certificate of SURVEY.md §8(c))."""
    N = lab.shape[0]
    L0, _ = orc.log_likelihood(C, lab)
    cand = []
    for i in range(N):
        for k in range(int(lab.max()) + 2):
            if k != lab[i]:
                m = lab.copy()
                m[i] = k
                cand.append(m)
    L, _ = orc.evaluate(C, np.asarray(cand, np.int32))
    return bool(np.any(L > L0 + 1e-12 * max(1.0, abs(L0))))


def _ari(a, b):
    """Adjusted Rand index of two labellings (textbook contingency form)."""
    from math import comb
    ct = {}
    for x, y in zip(a, b):
        ct[(x, y)] = ct.get((x, y), 0) + 1
    sa, sb = {}, {}
    for (x, y), n in ct.items():
        sa[x] = sa.get(x, 0) + n
        sb[y] = sb.get(y, 0) + n
    idx = sum(comb(n, 2) for n in ct.values())
    ea = sum(comb(n, 2) for n in sa.values())
    eb = sum(comb(n, 2) for n in sb.values())
    tot = comb(len(a), 2)
    exp = ea * eb / tot
    den = 0.5 * (ea + eb) - exp
    return 1.0 if den == 0 else (idx - exp) / den


def test_batch_recovers_planted_windows(pga, orc):
    """End to end on F1 windows (Table 3 configuration).  Eq. 8 rewards any
    positively correlated pair, so at T = 160 the maximum-likelihood
    partition is not the planted one (noise pairs merge).  What must hold:
    the GA's best scores at least the planted partition, it is a local
    optimum under single-gene moves, and it agrees with the planted
    structure (ARI)."""
    B = 64
    C, planted = _windows(orc, B)
    res = pga.pga_batch_run(C, _gparams(pga, 1000, 99))
    best = res["best_labels"] - 1
    Lp = np.array([orc.log_likelihood(C[b], planted[b])[0] for b in range(B)])
    ge = res["best_L"] >= Lp - 1e-9 * np.maximum(1, Lp)
    local = np.array([not _single_move_improves(orc, C[b], best[b]) for b in range(B)])
    ari = np.array([_ari(best[b], planted[b]) for b in range(B)])
    print("best>=planted %.3f local-opt %.3f mean ARI %.3f" % (ge.mean(), local.mean(), ari.mean()))
    assert ge.mean() >= 0.95, ge.mean()
    assert local.mean() >= 0.95, local.mean()
    assert ari.mean() >= 0.8, ari.mean()     # oracle GA on the same windows: 0.894


def test_batch_validation(pga):
    C = np.stack([np.eye(33)])
    with pytest.raises(pga.PgaError):
        pga.pga_batch_run(C, pga.pga_params_default(pop_size=100))
    with pytest.raises(pga.PgaError):
        pga.pga_batch_run(np.stack([np.eye(8)]), pga.pga_params_default(pop_size=4096))
    with pytest.raises(pga.PgaError):
        pga.pga_batch_run(np.stack([np.eye(8)]), pga.pga_params_default(pop_size=100, n_islands=2))
