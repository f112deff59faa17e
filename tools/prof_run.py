"""Run one indexer layer (for ncu captures): python tools/prof_run.py --method misa --L 131072 [--reps 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_07363_b200 import IndexerEngine, prepare_inputs  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--method", default="misa")
p.add_argument("--L", type=int, default=131072)
p.add_argument("--H", type=int, default=64)
p.add_argument("--h", type=int, default=8)
p.add_argument("--d", type=int, default=128)
p.add_argument("--B", type=int, default=1024)
p.add_argument("--k", type=int, default=2048)
p.add_argument("--kprime", type=int, default=8192)
p.add_argument("--reps", type=int, default=1)
a = p.parse_args()
gen = torch.Generator(device="cuda").manual_seed(0)
K = torch.randn(a.L, a.d, device="cuda", generator=gen).bfloat16()
Q = torch.randn(a.L, a.H, a.d, device="cuda", generator=gen).bfloat16()
W = torch.softmax(torch.randn(a.L, a.H, device="cuda", generator=gen), -1).float()
x = prepare_inputs(K, Q, W)
eng = IndexerEngine(a.method, budget_k=a.k, active_heads_h=a.h, block_size=a.B, candidate_kprime=a.kprime)
for _ in range(a.reps):
    eng.run_prepared(x)
torch.cuda.synchronize()
print("done", a)
