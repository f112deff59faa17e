"""One eager decode step per (method, T) at L = 1M for an ncu launch list (dev tool):
    ncu --metrics gpu__time_duration.sum --csv python tools/decode_prof.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_07363_b200 import IndexerEngine
from paper_2605_07363_b200.pooling import PooledKeyCache

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
g = torch.Generator(device="cuda").manual_seed(0)
K = torch.randn(L, 128, device="cuda", generator=g).bfloat16()
cache = PooledKeyCache(128, 1024, capacity=L)
cache.append(K)
for T in (1, 64):
    Q = torch.randn(T, 64, 128, device="cuda", generator=g).bfloat16()
    W = torch.softmax(torch.randn(T, 64, device="cuda", generator=g), -1).float()
    for m in ("misa", "dsa"):
        eng = IndexerEngine(m, budget_k=2048, active_heads_h=8, block_size=1024)
        eng.decode(queries=Q, weights=W, cache=cache)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push(f"{m}_T{T}")
        eng.decode(queries=Q, weights=W, cache=cache)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        print("marker", m, T, flush=True)
