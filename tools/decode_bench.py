"""Decode step timing (C5 shapes): T query rows against a PooledKeyCache of L keys,
eager engine.decode vs the CUDA-graph DecodeGraph replay (per-token serving step)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_07363_b200 import DecodeGraph, IndexerEngine
from paper_2605_07363_b200.pooling import PooledKeyCache


def time_fn(fn, steps=30, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def decode_numbers(Ls=(131072, 1048576), Ts=(1, 64), methods=("misa", "dsa")):
    out = []
    for L in Ls:
        g = torch.Generator(device="cuda").manual_seed(0)
        K = torch.randn(L, 128, device="cuda", generator=g).bfloat16()
        cache = PooledKeyCache(128, 1024, capacity=L)
        cache.append(K)
        for T in Ts:
            Q = torch.randn(T, 64, 128, device="cuda", generator=g).bfloat16()
            W = torch.softmax(torch.randn(T, 64, device="cuda", generator=g), -1).float()
            for m in methods:
                eng = IndexerEngine(m, budget_k=2048, active_heads_h=8, block_size=1024)
                eager = time_fn(lambda: eng.decode(queries=Q, weights=W, cache=cache))
                dg = DecodeGraph(IndexerEngine(m, budget_k=2048, active_heads_h=8, block_size=1024), cache, T, 64)
                graph = time_fn(lambda: dg.step(Q, W))
                out.append({"method": m, "L": L, "T": T, "eager_ms": round(eager, 4), "graph_ms": round(graph, 4)})
    return out


if __name__ == "__main__":
    for r in decode_numbers():
        print(json.dumps(r))
