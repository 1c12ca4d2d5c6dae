"""GPU parity for paths the round-1 suite ran but did not check (VERDICT r01
"What's weak" 1-2): the wide-N breed kernel, the island stall rule with a
live tolerance and bit-exact populations after every migrant import, the
single-population GA run free against the oracle, the full-size C4 GA after
cache clears, replicated master-slave with the default label-sparse
threshold, the C2 exhaustive set, and C5 fitness at its full size on a
1024-row sample.  Everything goes through the C ABI; tolerances as in
test_gpu_parity.py (L: 1e-9 max(1, |L|); labels, operators: bit-exact)."""
import os

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-9
NT = os.cpu_count() or 1


@pytest.fixture(scope="module")
def pga():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1403_4099_b200 import build
    build.build()
    import paper_1403_4099_b200 as p
    return p


def _par(pga, P, **kw):
    kw.setdefault("elite", min(10, P - 1))
    return pga.pga_params_default(pop_size=P, **kw)


def _assert_L(Lg, Lo):
    err = np.abs(np.asarray(Lg) - np.asarray(Lo)) / np.maximum(1.0, np.abs(Lo))
    assert err.max() <= TOL, "max rel err %g at %d" % (err.max(), int(err.argmax()))


def _corr(orc, spec):
    X, planted = workloads.noh_returns(spec)
    return orc.pearson(X), planted


# ---------------------------------------------------------------------------
# k_breed (N > 1024: the chunk-sequential breed kernel; the C5 GA path)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("N,P,pc,pm,pkb", [(1025, 64, 0.9, 0.002, 0.9), (2000, 48, 0.9, 0.001, 0.5),
                                           (1100, 37, 1.0, 0.3, 0.0), (2000, 20, 0.5, 1.0, 1.0)])
def test_op_breed_wide(pga, orc, N, P, pc, pm, pkb):
    rng = np.random.default_rng(N + P)
    planted = orc.canonicalize(rng.integers(0, 12, N))
    pop = orc.canonicalize(workloads.perturbed_planted(rng, planted, P, frac=0.05))
    pop[::3] = orc.canonicalize(rng.integers(0, N, (len(pop[::3]), N)))
    # KB tops: any label present in the row, some rows without a top
    top = np.array([int(pop[p][rng.integers(0, N)]) for p in range(P)], np.int32)
    top[::7] = -1
    L = np.round(rng.random(P) * 100, 2)
    E = min(10, P - 1)
    params = _par(pga, P, elite=E, p_crossover=pc, p_mutation=pm, p_kb=pkb, seed=77)
    o, sel = orc.select(L, E, seed=77, gen=9, island=1)
    sig = orc.mates(len(sel), seed=77, gen=9, island=1)
    ng = pga.pga_op_breed(pop, top, o, sel, sig, params, gen=9, island=1, p_off=3 * P)
    no = orc.breed(pop, top, o, E, sel, sig, pc, pm, pkb, seed=77, gen=9, island=1, p_off=3 * P)
    assert np.array_equal(ng, no)


def test_generation_lockstep_wide_N(pga, orc):
    """GA generations at N = 1100 (k_breed inside pga_generation, dense
    fitness): populations bit-exact given the GPU's own L and top."""
    spec = workloads.PlantedSpec((300, 250, 200, 150, 100, 100), (0.8, 0.75, 0.7, 0.65, 0.6, 0.6),
                                 3000, 11001)
    C, _ = _corr(orc, spec)
    N, P, gens = C.shape[0], 96, 3
    params = _par(pga, P, max_gens=gens + 1, tol=-1.0, p_mutation=2.0 / N, seed=6)
    op = orc.default_params(pop=P, max_gens=gens + 1, tol=-1.0, p_m=2.0 / N, seed=6)
    ctx = pga.pga_create(C, params)
    try:
        pga.pga_init(ctx, 6)
        pop, _ = pga.pga_get_population(ctx)
        for g in range(gens):
            pga.pga_generation(ctx)
            nxt, L, top = pga.pga_get_population(ctx, with_top=True)
            _assert_L(L, orc.evaluate(C, pop - 1, nthreads=NT)[0])
            assert np.array_equal(nxt - 1, orc.step(op, pop - 1, L, top, gen=g)), g
            pop = nxt
    finally:
        pga.pga_destroy(ctx)


@pytest.mark.parametrize("path", ["rank_count", "cluster_or_sort"])
@pytest.mark.parametrize("P,sel,scal,E", [(1025, 0, 0, 10), (1500, 0, 1, 7), (4096, 1, 0, 10),
                                          (8192, 0, 0, 10), (16384, 0, 1, 0), (16383, 0, 0, 10),
                                          (20001, 0, 0, 10), (20000, 0, 1, 10)])
def test_generation_lockstep_cluster_select(pga, orc, P, sel, scal, E, path, monkeypatch):
    """1024 < P <= 8192: order, scaling and selection by rank counting in
    one launch (k_rank_sel: chunk sorts + binary searches, per-tile
    finalisers, fused SUS; the default there) or, with PGA_NO_RANKC=1, in
    one thread-block-cluster launch (k_select_cluster); P > 8192: the run
    sort + merge tree on both (path is then moot).
    Generations in lockstep with the oracle's operators: bit-exact
    populations given the GPU's L and top, for SUS RANK / NONE and
    tournament, ragged P, E = 0 (M = P + 1 for odd P - E)."""
    if path != "rank_count":
        monkeypatch.setenv("PGA_NO_RANKC", "1")
    C, _ = _corr(orc, workloads.CONFIGS["C3"])
    N, gens = C.shape[0], 3
    params = _par(pga, P, elite=E, selection=sel, scaling=scal, tournament_k=3, max_gens=gens + 1,
                  tol=-1.0, p_mutation=0.02, seed=17)
    op = orc.default_params(pop=P, elite=E, selection=sel, scaling=scal, tour_k=3, max_gens=gens + 1,
                            tol=-1.0, p_m=0.02, seed=17)
    ctx = pga.pga_create(C, params)
    try:
        pga.pga_init(ctx, 17)
        pop, _ = pga.pga_get_population(ctx)
        for g in range(gens):
            pga.pga_generation(ctx)
            nxt, L, top = pga.pga_get_population(ctx, with_top=True)
            _assert_L(L, orc.evaluate(C, pop - 1, nthreads=NT)[0])
            assert np.array_equal(nxt - 1, orc.step(op, pop - 1, L, top, gen=g)), g
            pop = nxt
    finally:
        pga.pga_destroy(ctx)


@pytest.mark.parametrize("path", ["rank_count", "cluster_or_sort"])
@pytest.mark.parametrize("P,kind", [(2048, "identical"), (5000, "singletons"), (12000, "two_values")])
def test_generation_lockstep_selection_ties(pga, orc, P, kind, path, monkeypatch):
    """Selection with massive L ties (1024 < P <= 16384; k_rank_sel up to 8192): every individual
    the same chromosome (all L equal), every individual all singletons (L =
    0 everywhere: the sort key equals the padding key of k_rank_sel's
    chunks), or two distinct chromosomes alternating.  The order must break
    ties by index across chunks and tiles; one generation in lockstep with
    orc_step (bit-exact), by rank counting and by the cluster / sort path."""
    if path != "rank_count":
        monkeypatch.setenv("PGA_NO_RANKC", "1")
    C, planted = _corr(orc, workloads.CONFIGS["C3"])
    N = C.shape[0]
    if kind == "identical":
        pop = np.tile(planted, (P, 1))
    elif kind == "singletons":
        pop = np.tile(np.arange(N), (P, 1))
    else:
        alt = orc.canonicalize(np.where(np.arange(N) % 2 == 0, planted, 0)[None, :])[0]
        pop = np.where((np.arange(P) % 2 == 0)[:, None], planted[None, :], alt[None, :])
    pop = pop.astype(np.int32)
    params = _par(pga, P, max_gens=4, tol=-1.0, p_mutation=0.02, seed=23)
    op = orc.default_params(pop=P, max_gens=4, tol=-1.0, p_m=0.02, seed=23)
    ctx = pga.pga_create(C, params)
    try:
        pga.pga_init(ctx, 23)
        pga.pga_set_population(ctx, pop + 1, 0)
        pga.pga_generation(ctx)
        nxt, L, top = pga.pga_get_population(ctx, with_top=True)
        Lo = orc.evaluate(C, pop, nthreads=NT)[0]
        _assert_L(L, Lo)
        if kind == "singletons":
            assert np.all(L == 0.0)
        assert np.array_equal(nxt - 1, orc.step(op, pop, L, top, gen=0))
    finally:
        pga.pga_destroy(ctx)


# ---------------------------------------------------------------------------
# islands: the Q28 stall rule with tol >= 0, bit-exact after every import
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("cfg,P,M,S,pm", [("C1", 64, 4, 8, 0.1), ("C3", 256, 5, 10, 0.02)])
def test_islands_stall_and_import_lockstep(pga, orc, cfg, P, M, S, pm):
    """Two islands as two contexts on one device (the all-gather emulated by
    concatenating the send buffers; the migration kernels run unchanged),
    tol = 1e-5 and a short stall window so the run ends by stall.  Every
    generation: (a) L matches the oracle; (b) after pga_import_migrants each
    island's population, L and top equal the oracle's orc_migrate applied to
    the GPU's pre-import state; (c) the bred population equals orc_step on
    the GPU's post-import state; (d) the GPU stops at the generation and
    with the reason the Q28 rule gives on the GPU's own
    per-generation global best."""
    import torch
    C, _ = _corr(orc, workloads.CONFIGS[cfg])
    N, G, tol = C.shape[0], 2, 1e-5
    kw = dict(max_gens=400, tol=tol, stall_gens=S, p_mutation=pm, seed=41, n_islands=G,
              migrate_every=M, migrants=5)
    ctxs = [pga.pga_create(C, _par(pga, P, island=g, **kw)) for g in range(G)]
    op = orc.default_params(pop=P, max_gens=400, tol=tol, stall_gens=S, p_m=pm, seed=41,
                            n_islands=G, migrate_every=M, migrants=5)
    stall, prev, expect_stop = 0, 0.0, None
    try:
        for c in ctxs:
            pga.pga_init(c, 41)
        pops = [pga.pga_get_population(c)[0] - 1 for c in ctxs]
        nb = pga.pga_migrant_bytes(ctxs[0])
        send = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(G)]
        imports = 0
        for g in range(400):
            mig = [pga.pga_gen_evaluate(c) for c in ctxs]
            assert all(m == ((g + 1) % M == 0) for m in mig)
            st = [pga.pga_get_population(c, with_top=True) for c in ctxs]
            for k in range(G):
                assert np.array_equal(st[k][0] - 1, pops[k])
                _assert_L(st[k][1], orc.evaluate(C, pops[k], nthreads=NT)[0])
            Ls = [s[1].copy() for s in st]
            tops = [s[2].copy() for s in st]
            if mig[0]:
                for c, s in zip(ctxs, send):
                    pga.pga_export_migrants(c, s)
                torch.cuda.synchronize()
                recv = torch.cat(send)
                for c in ctxs:
                    pga.pga_import_migrants(c, recv, G)
                want_p, want_L, want_t = orc.migrate([p.copy() for p in pops], Ls, tops, 5)
                for k, c in enumerate(ctxs):
                    lab, L, top = pga.pga_get_population(c, with_top=True)
                    assert np.array_equal(lab - 1, want_p[k]), "import, island %d gen %d" % (k, g)
                    assert np.array_equal(L, want_L[k]) and np.array_equal(top, want_t[k])
                pops, Ls, tops = list(want_p), list(want_L), list(want_t)
                imports += 1
                gbest = max(float(x.max()) for x in Ls)
                if g + 1 > M:
                    stall = stall + M if gbest - prev < tol else 0
                prev = gbest
            if stall >= S and expect_stop is None:
                expect_stop = g + 1
            states = [pga.pga_get_state(c) for c in ctxs]
            done = [s["done"] for s in states]
            assert done[0] == done[1] == (1 if expect_stop is not None else 0), g
            if done[0]:
                assert all(s["reason"] == 1 for s in states)
                break
            for k, c in enumerate(ctxs):
                pga.pga_gen_breed(c)
                nxt = pga.pga_get_population(c)[0] - 1
                want = orc.step(op, pops[k], Ls[k], tops[k], gen=g, island=k, p_off=k * P)
                assert np.array_equal(nxt, want), "breed, island %d gen %d" % (k, g)
                pops[k] = nxt
        assert expect_stop is not None and imports >= 3
        # a driver that keeps stepping after the stop (through at least one
        # more migration generation: export, all-gather, import) leaves the
        # final population, L and best state alone
        final = [pga.pga_get_population(c) for c in ctxs]
        best = [pga.pga_get_state(c)["best_L"] for c in ctxs]
        for c in ctxs:
            pga.pga_gen_breed(c)
        for _ in range(M):
            mig = [pga.pga_gen_evaluate(c) for c in ctxs]
            if mig[0]:
                for c, s in zip(ctxs, send):
                    pga.pga_export_migrants(c, s)
                torch.cuda.synchronize()
                recv = torch.cat(send)
                for c in ctxs:
                    pga.pga_import_migrants(c, recv, G)
            for c in ctxs:
                pga.pga_gen_breed(c)
        for c, f, b in zip(ctxs, final, best):
            lab, L = pga.pga_get_population(c)
            assert np.array_equal(lab, f[0]) and np.array_equal(L, f[1])
            assert pga.pga_get_state(c)["best_L"] == b
    finally:
        for c in ctxs:
            pga.pga_destroy(c)


# ---------------------------------------------------------------------------
# the single-population GA run free against the oracle
# ---------------------------------------------------------------------------
def test_run_C1_free_running_equals_oracle(pga, orc):
    """C1 at its stated 100 generations, GA seeds 1..20: pga_run (CUDA graph
    replay, nothing fed back from the oracle) and orc_run end with the same
    best labelling in >= 19 of 20 seeds (a last-bit near-tie of two distinct
    L values may flip a rank and split a trajectory).  The planted partition
    is recovered in the same seeds on both sides; the rate itself (~10/20
    here, 62% over 1000 seeds, profiles/r02_pairing_tradeoff.json) is the
    method's at this budget, reported in DESIGN.md §6."""
    C, planted = _corr(orc, workloads.CONFIGS["C1"])
    N = C.shape[0]
    same = rec_g = rec_o = 0
    for seed in range(1, 21):
        ctx = pga.pga_create(C, _par(pga, 128, max_gens=100, tol=-1.0, seed=seed))
        try:
            r = pga.pga_run(ctx, 100, seed)
        finally:
            pga.pga_destroy(ctx)
        ro = orc.run(C, orc.default_params(pop=128, max_gens=100, tol=-1.0, seed=seed))
        eq = np.array_equal(r["best_labels"] - 1, ro["best_labels"])
        same += eq
        if eq:
            assert abs(r["best_L"] - ro["best_L"]) <= TOL * max(1.0, ro["best_L"])
            assert r["gens_run"] == ro["gens_run"] == 100
        rec_g += np.array_equal(r["best_labels"] - 1, planted)
        rec_o += np.array_equal(ro["best_labels"], planted)
    assert same >= 19, same
    assert abs(rec_g - rec_o) <= 20 - same
    assert rec_o >= 6


def test_run_table3_termination_equals_oracle(pga, orc):
    """Table 3 termination (tol 1e-5, stall 50, <= 400 generations) free
    running on C1 and C2: generations run, stop reason and best labels agree
    with orc_run in >= 5 of the 6 runs (a near-tie can split a trajectory,
    see the free-running C1 test), and every run stops by stall."""
    agree = 0
    for cfg, P in (("C1", 1000), ("C2", 1024)):
        C, _ = _corr(orc, workloads.CONFIGS[cfg])
        for seed in (1, 2, 3):
            ctx = pga.pga_create(C, _par(pga, P, seed=seed))
            try:
                    r = pga.pga_run(ctx, 0, seed)
            finally:
                pga.pga_destroy(ctx)
            ro = orc.run(C, orc.default_params(pop=P, seed=seed))
            agree += ((r["gens_run"], r["reason"]) == (ro["gens_run"], ro["reason"]) and
                      np.array_equal(r["best_labels"] - 1, ro["best_labels"]))
            assert r["reason"] == 1 and r["gens_run"] <= 400
    assert agree >= 5, agree


# ---------------------------------------------------------------------------
# C4 at full size, mid-run, across cluster-cache clears
# ---------------------------------------------------------------------------
def test_C4_full_size_midrun_sample(pga, orc):
    """C4 (N = 500, P = 65536, p_m = 2/N) after ~800 generations with the
    automatic label-sparse pass and the cluster cache, including at least
    one cache clear and the pass's unchecked launches: 1024 sampled
    chromosomes of the evaluated generation (plus both ends) against the
    oracle, and the next population (all 65536 rows) equal to orc_step on
    the GPU's L and top."""
    C, _ = _corr(orc, workloads.CONFIGS["C4"])
    N, P = C.shape[0], 65536
    params = _par(pga, P, max_gens=4000, tol=-1.0, p_mutation=2.0 / N, seed=12)
    ctx = pga.pga_create(C, params)
    try:
        pga.pga_init(ctx, 12)
        gens, after = 0, None
        # run until the cache table has been cleared (half full: ~700
        # generations at C4), then 60 generations more
        while gens < 3500 and (after is None or gens < after + 60):
            for _ in range(20):
                pga.pga_gen_evaluate(ctx)
                pga.pga_gen_breed(ctx)
            gens += 20
            if after is None and pga.pga_cache_stats(ctx)["clears"] >= 1:
                after = gens
        pga.pga_gen_evaluate(ctx)
        pop, L, top = pga.pga_get_population(ctx, with_top=True)
        cache = pga.pga_cache_stats(ctx)
        blocks, _ = pga.pga_profile_sparse(ctx)
        st = pga.pga_get_state(ctx)
        pga.pga_gen_breed(ctx)
        nxt = pga.pga_get_population(ctx)[0]
    finally:
        pga.pga_destroy(ctx)
    assert st["generation"] == gens
    assert cache["slots"] > 0 and cache["clears"] >= 1, cache
    assert blocks > 0
    idx = np.concatenate([np.random.default_rng(3).choice(P, 1024, replace=False), [0, 1, P - 2, P - 1]])
    Lo, to = orc.evaluate(C, pop[idx] - 1, nthreads=NT)
    _assert_L(L[idx], Lo)
    assert np.all(np.isfinite(L)) and L.min() > 0.0
    op = orc.default_params(pop=P, max_gens=4000, tol=-1.0, p_m=2.0 / N, seed=12)
    assert np.array_equal(nxt - 1, orc.step(op, pop - 1, L, top, gen=gens))


# ---------------------------------------------------------------------------
# replicated master-slave at the default label-sparse threshold
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("cfg,P,W,gens", [("C4", 2048, 2, 6), ("C3", 1024, 3, 8)])
def test_replicated_default_theta_lockstep(pga, orc, cfg, P, W, gens):
    """Replicas with the library's automatic threshold (the label-sparse
    pass on for N >= 64, as bench --mode replicated runs it), stepped in
    sequence on one GPU: every generation the gathered L matches the
    oracle, every replica holds the same population, and it equals orc_step
    on the gathered L and top."""
    import torch
    from paper_1403_4099_b200.replicated import GpuReplica, shard
    C, _ = _corr(orc, workloads.CONFIGS[cfg])
    N = C.shape[0]
    pm = 2.0 / N
    params = pga.pga_params_default(pop_size=P, p_mutation=pm, max_gens=gens + 2, tol=-1.0, seed=8)
    op = orc.default_params(pop=P, max_gens=gens + 2, tol=-1.0, p_m=pm, seed=8)
    reps = [GpuReplica(C, params) for _ in range(W)]
    try:
        for r in reps:
            r.init(8)
        pop = pga.pga_get_population(reps[0].ctx)[0] - 1
        S = shard(P, W, 0)[2]
        L_all = torch.zeros(S * W, dtype=torch.float64, device="cuda")
        t_all = torch.zeros(S * W, dtype=torch.int16, device="cuda")
        sparse_seen = 0
        for g in range(gens):
            for k, r in enumerate(reps):
                b, e, _ = shard(P, W, k)
                if e > b:
                    with torch.cuda.stream(r.stream):
                        r.rep_evaluate(b, e, L_all[k * S:k * S + (e - b)], t_all[k * S:k * S + (e - b)])
                    r.stream.synchronize()
            L = L_all[:P].cpu().numpy()
            top = t_all[:P].cpu().numpy().astype(np.int32) & 0xFFFF
            top = np.where(top == 0xFFFF, -1, top)
            _assert_L(L, orc.evaluate(C, pop, nthreads=NT)[0])
            for r in reps:
                r.rep_commit(L_all[:P], t_all[:P])
                r.gen_breed()
                r.stream.synchronize()
            want = orc.step(op, pop, L, top, gen=g)
            for r in reps:
                assert np.array_equal(pga.pga_get_population(r.ctx)[0] - 1, want), g
            pop = want
        for r in reps:
            sparse_seen += pga.pga_profile_sparse(r.ctx)[0]
    finally:
        for r in reps:
            r.close()
    if N >= 64:
        assert sparse_seen > 0


# ---------------------------------------------------------------------------
# C2: the exhaustive set (50 matrices, n in {6, 8, 10}, seeds 2000..2049)
# ---------------------------------------------------------------------------
def test_C2_set_matches_brute_force(pga, orc):
    """SPEC S:536 acceptance 2 / SURVEY §8(d) C2 on the GPU: pga_run with
    P = 1024 and Table 3 termination never exceeds the exhaustive maximum
    over all set partitions (Bell(n) of them) and reaches it in >= 90% of
    the 50 matrices; where it reaches it, L agrees within the tolerance."""
    hits = 0
    bell = {6: 203, 8: 4140, 10: 115975}
    for k in range(workloads.C2_SET["count"]):
        X, _ = workloads.noh_returns(workloads.c2_set_spec(k))
        C = orc.pearson(X)
        best, Lb, count = orc.brute_force(C)
        assert count == bell[C.shape[0]]
        seed = workloads.C2_SET["seed0"] + k
        ctx = pga.pga_create(C, _par(pga, 1024, seed=seed))
        try:
            r = pga.pga_run(ctx, 0, seed)
        finally:
            pga.pga_destroy(ctx)
        assert r["best_L"] <= Lb + TOL * max(1.0, Lb), k
        if abs(r["best_L"] - Lb) <= TOL * max(1.0, Lb):
            hits += 1
            Lc, _ = orc.log_likelihood(C, r["best_labels"] - 1)
            assert abs(Lc - Lb) <= TOL * max(1.0, Lb)
    assert hits >= 45, hits


# ---------------------------------------------------------------------------
# C5: fitness-only at full size, 1024-row sample
# ---------------------------------------------------------------------------
def test_C5_fitness_full_size_1024_sample(pga, orc):
    """C5 as BASELINE configs[4] states it: N = 2000, P = 262144, one
    fitness-only evaluate launch over the whole population (the bench's
    fitness sweep), L checked on a 1024-chromosome sample by the oracle.
    The population is an 8192-row equal-thirds mix repeated
    32 times under per-copy label permutations (distinct rows as data)."""
    import torch
    C, planted = _corr(orc, workloads.CONFIGS["C5"])
    N = C.shape[0]
    base_P, reps = 8192, 32
    P = base_P * reps
    base = workloads.population_mix(321, planted, base_P)
    rng = np.random.default_rng(29)
    perms = np.stack([rng.permutation(N) for _ in range(reps)]).astype(np.int64)
    ctx = pga.pga_create(C, _par(pga, P))
    try:
        db = torch.from_numpy(base.astype(np.int64)).cuda()
        dp = torch.from_numpy(perms).cuda()
        dl = torch.empty((P, N), dtype=torch.int16, device="cuda")
        for t in range(reps):
            dl[t * base_P:(t + 1) * base_P] = torch.gather(dp[t].expand(base_P, N), 1, db).to(torch.int16)
        del db
        L = torch.zeros(P, dtype=torch.float64, device="cuda")
        pga.pga_evaluate_device(ctx, dl, L)
        torch.cuda.synchronize()
        Lg = L.cpu().numpy()
    finally:
        pga.pga_destroy(ctx)
    idx = np.concatenate([rng.choice(P, 1024, replace=False), [0, 1, base_P - 1, base_P, P - 1]])
    rows = np.stack([perms[i // base_P][base[i % base_P]] for i in idx]).astype(np.int32)
    Lo, _ = orc.evaluate(C, rows, nthreads=NT)
    _assert_L(Lg[idx], Lo)
    assert np.all(np.isfinite(Lg))


# ---------------------------------------------------------------------------
# ABI hardening
# ---------------------------------------------------------------------------
def test_evaluate_device_on_a_foreign_stream_is_serialised(pga, orc):
    """pga_evaluate_device on a caller stream joins the ctx's stream both
    ways: back-to-back calls on two different streams, each with its own
    population, give each its own correct L."""
    import torch
    C, planted = _corr(orc, workloads.CONFIGS["C3"])
    N, P = C.shape[0], 4096
    ctx = pga.pga_create(C, _par(pga, P))
    try:
        labs = [workloads.population_mix(s, planted, P) for s in (1, 2, 3)]
        dls = [torch.from_numpy(l.astype(np.int16)).cuda() for l in labs]
        outs = [torch.zeros(P, dtype=torch.float64, device="cuda") for _ in labs]
        streams = [torch.cuda.Stream() for _ in labs]
        torch.cuda.synchronize()
        for _ in range(3):
            for dl, o, s in zip(dls, outs, streams):
                pga.pga_evaluate_device(ctx, dl, o, stream=s.cuda_stream)
        torch.cuda.synchronize()
        for l, o in zip(labs, outs):
            _assert_L(o.cpu().numpy(), orc.evaluate(C, l, nthreads=NT)[0])
        with pytest.raises(ValueError):           # wrong width
            pga.pga_evaluate_device(ctx, dls[0][:, :N - 1].contiguous(), outs[0])
        with pytest.raises(ValueError):           # float32 L
            pga.pga_evaluate_device(ctx, dls[0], outs[0].float())
        with pytest.raises(ValueError):           # population shape mismatch
            pga.pga_get_population(ctx, P + 1, N)
    finally:
        pga.pga_destroy(ctx)
