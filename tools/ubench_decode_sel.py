"""Per-call GPU time of the decode selection pieces, each captured 20x in a CUDA graph (dev tool):
threshold (warp-per-row kernel) on a contiguous 16384-sample row vs the long-row selector's own
strided threshold, and misa_select_dense_long end to end, at T = 1 and 64, L = 1M."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_07363_b200 import _lib

_lib.load()
st = lambda: torch.cuda.current_stream().cuda_stream


def gtime(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1000  # us per call


L, k = 1 << 20, 2048
for T in (1, 64):
    rows = torch.randn(T, L, device="cuda")
    pl = torch.full((T,), L, dtype=torch.int32, device="cuda")
    m = L // 64
    samp = rows[:, ::64].contiguous()
    tau = torch.empty(T, device="cuda")
    t_warp = gtime(lambda: _lib.call("misa_select_threshold", samp.data_ptr(), m, pl.data_ptr(), T, 64, k, 2.0,
                                     4096, tau.data_ptr(), st()))
    cap = 8192
    n_seg = L // 4096
    seg = torch.empty(T, n_seg, dtype=torch.int32, device="cuda")
    cs = torch.empty(T, cap, device="cuda")
    ci = torch.empty(T, cap, dtype=torch.int32, device="cuda")
    cc = torch.empty(T, dtype=torch.int32, device="cuda")
    out = torch.empty(T, k, dtype=torch.int32, device="cuda")
    t_long = gtime(lambda: _lib.call("misa_select_dense_long", rows.data_ptr(), L, pl.data_ptr(), T, k, L, 2.0,
                                     tau.data_ptr(), seg.data_ptr(), cs.data_ptr(), ci.data_ptr(), cc.data_ptr(), cap,
                                     out.data_ptr(), k, None, st()))
    print(f"T={T}: threshold_warp on contiguous sample {t_warp:.1f} us; misa_select_dense_long {t_long:.1f} us",
          flush=True)
