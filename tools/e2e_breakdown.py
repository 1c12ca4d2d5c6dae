"""Where the C4 e2e time goes (host clock): pga_create from pinned host C,
pga_init, the first generation (graph captures), the next K generations with
the per-step state read, the final gather.  python tools/e2e_breakdown.py [K]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
import workloads  # noqa: E402
import paper_1403_4099_b200 as pga  # noqa: E402
from paper_1403_4099_b200.islands import GpuIsland, IslandRunner  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
    C = pga.pga_correlation(X)
    N = C.shape[0]
    params = pga.pga_params_default(pop_size=65536, elite=10, p_mutation=2.0 / N, tol=-1.0, max_gens=K + 300,
                                    migrate_every=10, migrants=10, seed=1)
    Cp = torch.from_numpy(np.ascontiguousarray(C)).pin_memory()
    for rep in range(2):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        eng = GpuIsland(Cp.numpy(), params)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        runner = IslandRunner(eng)
        eng.init(1)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        runner.step(); eng.state()
        t.append(time.perf_counter())
        for _ in range(K - 1):
            runner.step()
            eng.state()
        t.append(time.perf_counter())
        runner.global_best()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        eng.close()
        d = np.diff(t) * 1e3
        print("rep %d: create %.2f ms, init %.2f, first generation %.2f, next %d generations %.2f (%.3f each), "
              "gather %.2f; total %.2f ms" % (rep, d[0], d[1], d[2], K - 1, d[3], d[3] / (K - 1), d[4], sum(d)))


if __name__ == "__main__":
    main()
