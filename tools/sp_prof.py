"""Label-sparse pass on a realistic C4 population, for ncu.
  python tools/sp_prof.py save G   -- run G GA generations, save the population to gpurun_out/pop_G.npy
  python tools/sp_prof.py load G   -- evaluate that population twice (2nd launch: cache hits as in a GA)
Profile with --kernel-name regex:k_fitness_sparse --launch-skip 1 --launch-count 1."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_1403_4099_b200 as pga

X, planted = workloads.noh_returns(workloads.CONFIGS["C4"])
C = pga.pga_correlation(X)
N, P = 500, 65536
mode, G = sys.argv[1], int(sys.argv[2])
path = "/tmp/pop_%d.npy" % G
if mode == "save":
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P, p_mutation=2.0 / N, tol=-1.0, max_gens=G + 5, seed=5))
    pga.pga_init(ctx, 5)
    for _ in range(G):
        pga.pga_gen_evaluate(ctx)
        pga.pga_gen_breed(ctx)
    pop, _ = pga.pga_get_population(ctx, P, N)
    np.save(path, (pop - 1).astype(np.int16))
    pga.pga_destroy(ctx)
else:
    lab = torch.from_numpy(np.load(path)).cuda()
    ctx = pga.pga_create(C, pga.pga_params_default(pop_size=P))
    pga.pga_set_sparse_threshold(ctx, 1.0)
    pga.pga_set_cluster_cache(ctx, len(sys.argv) < 4 or sys.argv[3] != "nocache")
    L = torch.zeros(P, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    for r in range(2):
        pga.pga_evaluate_device(ctx, lab, L, stream=s.cuda_stream)
    s.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(s):
        ev[0].record(s)
        for r in range(10):
            pga.pga_evaluate_device(ctx, lab, L, stream=s.cuda_stream)
        ev[1].record(s)
    s.synchronize()
    print("G=%d cache=%s: %.3f ms per evaluate (pack + sparse pass)" % (G, sys.argv[3:] or "on", ev[0].elapsed_time(ev[1]) / 10))
    pga.pga_destroy(ctx)
