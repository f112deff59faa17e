"""Sample stride / beta sweep of the fused top-k (dev tool): MISA layer time, stage split and
fallback rows at C4 (L = T = 131072) and C2 (32768), H = 64, h = 8, k = 2048."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_07363_b200 import IndexerEngine, prepare_inputs

combos = [(32, 2.0), (32, 1.6), (16, 1.5), (16, 1.35), (8, 1.3), (8, 1.2)]
for L in (131072, 32768):
    g = torch.Generator(device="cuda").manual_seed(0)
    K = torch.randn(L, 128, device="cuda", generator=g).bfloat16()
    Q = torch.randn(L, 64, 128, device="cuda", generator=g).bfloat16()
    W = torch.softmax(torch.randn(L, 64, device="cuda", generator=g), -1).float()
    x = prepare_inputs(K, Q, W)
    for s, b in combos:
        eng = IndexerEngine("misa", sample_stride=s, beta=b)
        for _ in range(2):
            eng.run_prepared(x)
        st, tot = {}, 0.0
        for _ in range(3):
            eng.stage_events = []
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.run_prepared(x)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1) / 3
            ev = eng.stage_events
            for (n0, a), (_, c) in zip(ev, ev[1:]):
                st[n0] = st.get(n0, 0.0) + a.elapsed_time(c) / 3
        print(f"L={L} stride={s} beta={b} cap={eng.selector_params(2048, L)[2]}: {tot:.3f} ms, fallback rows "
              f"{eng.last_fallback_rows}", {k: round(v, 3) for k, v in st.items() if k.startswith("sel")}, flush=True)
        del eng
