"""Sparse attention over an indexer selection at C4 scale (dev tool): T = 131072 query rows,
H = 128 heads, d = 128 (MQA latent rows), k = 2048 selected tokens per row."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_07363_b200 import _lib
if len(sys.argv) > 1:
    _lib.load(sys.argv[1])  # a variant library (tools/variant_lib.py)
from paper_2605_07363_b200.sparse_attention import sparse_attention

T = int(os.environ.get("SATTN_T", 131072))
L, H, d, k = 131072, 128, 128, 2048
g = torch.Generator(device="cuda").manual_seed(0)
kv = torch.randn(L, d, device="cuda", generator=g).bfloat16()
q = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
# causal-like selection: row t takes min(t+1, k) tokens of its prefix (ascending, -1 padded)
t = torch.arange(T, device="cuda")[:, None]
j = torch.arange(k, device="cuda")[None, :]
n = torch.clamp(t + 1, max=k)
stride = torch.clamp((t + 1) // k, min=1)
topk = torch.where(j < n, j * stride, -1).to(torch.int32)
sparse_attention(q, kv, topk, d)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    sparse_attention(q, kv, topk, d)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
sel = n.sum().item()
flops = 2 * 2 * H * d * sel  # QK + PV
print(sys.argv[1:], f"sparse attention T={T} H={H} d={d} k={k}: {ms:.2f} ms, {flops / ms / 1e9:.1f} TFLOP/s")
