"""C4 generation time: pga_run (one CUDA graph per generation, no profiling)
vs the eager pga_gen_evaluate/pga_gen_breed loop the bench times."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_1403_4099_b200 as pga
X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N, P = 500, 65536
for mode in ("eager", "graph", "eager", "graph"):
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=1100, seed=5))
    pga.pga_init(ctx, 5)
    s = torch.cuda.ExternalStream(pga.pga_get_stream(ctx))
    for _ in range(5):
        pga.pga_gen_evaluate(ctx); pga.pga_gen_breed(ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    if mode == "eager":
        for _ in range(1000):
            pga.pga_gen_evaluate(ctx); pga.pga_gen_breed(ctx)
    else:
        pga.pga_run(ctx, 1000, 5, N)
    e1.record(s)
    torch.cuda.synchronize()
    print(mode, "%.4f ms/gen" % (e0.elapsed_time(e1) / 1000), flush=True)
    pga.pga_destroy(ctx)
