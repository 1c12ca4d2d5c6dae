"""Time the correlation stream (pga_corr_stream_device) on the F1 shape."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_1403_4099_b200 as pga
B, N, T, stride = 1760, 18, 160, 10
Xs, _ = workloads.stream_returns(T + (B - 1) * stride, N, seed=1760000)
dX = torch.from_numpy(Xs).cuda()
dC = torch.zeros((B, N, N), dtype=torch.float64, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
for q in (-1.0, 0.0, -1.0, 0.0, 0.0):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    pga.pga_corr_stream_device(dX, dC, st, warm=T, stride=stride, q=q, stream=s.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    print("q=%g: events %.3f ms, wall %.3f ms" % (q, e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)))
