"""Label-sparse pass time against P around one island of an 8-GPU C4 split:
P = 148 * 32 * k fills every SM with k 32-chromosome blocks; P = 8192 leaves
the busiest SMs with 2 blocks (64 chromosomes) against a mean of 55.
python tools/sparse_balance.py"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import workloads  # noqa: E402
import paper_1403_4099_b200 as pga  # noqa: E402


def main():
    X, _ = workloads.noh_returns(workloads.CONFIGS["C4"])
    C = pga.pga_correlation(X)
    N = C.shape[0]
    for P in (4736, 7104, 8192, 9472, 11840, 14208, 16384):
        ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, elite=10, p_mutation=2.0 / N, tol=-1.0,
                                                        max_gens=400, seed=1))
        try:
            pga.pga_init(ctx, 1)
            for _ in range(30):
                pga.pga_gen_evaluate(ctx)
                pga.pga_gen_breed(ctx)
            pga.pga_profile_enable(ctx, 1)
            for _ in range(100):
                pga.pga_gen_evaluate(ctx)
                pga.pga_gen_breed(ctx)
            r = pga.pga_profile_read(ctx)
            n = max(1, r["count"])
            sp, gen = r["fold_ms"] / n, r["gen_ms"] / n   # fold_ms: the label-sparse pass (binding naming)
            print("P %6d  blocks/SM %.2f  sparse pass %.4f ms  (%.2f us per 1000 chromosomes)  generation %.4f ms"
                  % (P, P / 32.0 / 148, sp, 1e3 * sp / (P / 1000.0), gen), flush=True)
        finally:
            pga.pga_destroy(ctx)


if __name__ == "__main__":
    main()
