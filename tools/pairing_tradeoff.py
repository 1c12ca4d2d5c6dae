"""Mate pairing trade-off (Q10): planted recovery on C1 at the
config's 100 generations with the shipped keyed-Feistel pairing vs the
survey's sort-by-Philox-key pairing, over many GA seeds.

Both are uniform random pairings of the offspring slots; only the random
stream differs.  The GA loop here composes the oracle's own operators
(orc_order / orc_select / orc_breed) and swaps only sigma; with the Feistel
sigma it reproduces orc_run exactly (checked on the first seeds).

    python tools/pairing_tradeoff.py [--seeds 200] [--gens 100]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import oracle as orc  # noqa: E402
import workloads  # noqa: E402

TAG_PERM = 3


def sort_sigma(M, seed, gen, island=0):
    """sigma = slots sorted by (key, slot), key_m = Philox(PERM; m >> 2, 0, gen,
    PERM | island << 8)[m & 3]."""
    keys = np.zeros(M, np.uint64)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for b in range((M + 3) // 4):
        u = orc.philox([b, 0, gen, TAG_PERM | (island << 8)], key)
        for j in range(4):
            if 4 * b + j < M:
                keys[4 * b + j] = int(u[j])
    return np.lexsort((np.arange(M), keys)).astype(np.int32)


def ga(C, P, gens, seed, pairing):
    N = C.shape[0]
    p = orc.default_params(pop=P, max_gens=gens, tol=-1.0, seed=seed)
    pop = orc.init_population(seed, N, P)
    best_L, best = -1.0, None
    for g in range(gens):
        L, top = orc.evaluate(C, pop)
        b = int(np.argmax(L))
        if L[b] > best_L:
            best_L, best = float(L[b]), pop[b].copy()
        if g + 1 == gens:
            break
        order, sel = orc.select(L, p.elite, seed=seed, gen=g)
        M = orc.num_offspring(P, p.elite)
        sigma = orc.mates(M, seed=seed, gen=g) if pairing == "feistel" else sort_sigma(M, seed, g)
        pop = orc.breed(pop, top, order, p.elite, sel, sigma, p.p_c, p.p_m, p.p_kb, seed=seed, gen=g)
    return best, best_L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=200)
    ap.add_argument("--gens", type=int, default=100)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    X, planted = workloads.noh_returns(workloads.CONFIGS["C1"])
    C = orc.pearson(X)
    # the loop is the oracle GA: with Feistel sigma it equals orc_run
    for s in (1, 2, 3):
        r = orc.run(C, orc.default_params(pop=128, max_gens=a.gens, tol=-1.0, seed=s))
        lab, L = ga(C, 128, a.gens, s, "feistel")
        assert np.array_equal(lab, r["best_labels"]) and L == r["best_L"], s
    res = {}
    for pairing in ("feistel", "sort"):
        hits = [bool(np.array_equal(ga(C, 128, a.gens, s, pairing)[0], planted))
                for s in range(1, a.seeds + 1)]
        k = sum(hits)
        p = k / a.seeds
        res[pairing] = {"recovered": k, "seeds": a.seeds, "rate": p,
                        "stderr": math.sqrt(p * (1 - p) / a.seeds),
                        "first20": sum(hits[:20])}
    d = res["feistel"]["rate"] - res["sort"]["rate"]
    se = math.sqrt(res["feistel"]["stderr"] ** 2 + res["sort"]["stderr"] ** 2)
    res["difference"] = {"feistel_minus_sort": d, "z": d / se if se else 0.0}
    res["workload"] = "C1 (N=18, P=128, Table 3 operators), %d generations, GA seeds 1..%d" % (a.gens, a.seeds)
    print(json.dumps(res, indent=1))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
