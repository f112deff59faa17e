"""Decode step timing: T query rows at prefix L (all rows see the whole cache)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_07363_b200 import IndexerEngine

def bench(method, L, T, steps=20, warm=3):
    g = torch.Generator(device="cuda").manual_seed(0)
    K = torch.randn(L, 128, device="cuda", generator=g).bfloat16()
    Q = torch.randn(T, 64, 128, device="cuda", generator=g).bfloat16()
    W = torch.softmax(torch.randn(T, 64, device="cuda", generator=g), -1).float()
    eng = IndexerEngine(method, budget_k=2048, active_heads_h=8, block_size=1024)
    for _ in range(warm):
        eng.decode(K, Q, W)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        eng.decode(K, Q, W)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    eng.stage_events = []
    eng.decode(K, Q, W); torch.cuda.synchronize()
    ev = eng.stage_events
    st = {n0: round(a.elapsed_time(b), 4) for (n0, a), (_, b) in zip(ev, ev[1:])}
    return ms, st

for L in (131072, 1048576):
    for T in (1, 64):
        for m in ("misa", "dsa"):
            ms, st = bench(m, L, T)
            print(json.dumps({"method": m, "L": L, "T": T, "ms": round(ms, 4), "stages": st}))
