"""Diagnose fallback rows of the 1M causal prefill (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_07363_b200 import IndexerEngine, prepare_inputs
L = T = 1 << 20
g = torch.Generator(device="cuda").manual_seed(0)
K = torch.randn(L, 128, device="cuda", generator=g).bfloat16()
Q = torch.randn(T, 64, 128, device="cuda", generator=g).bfloat16()
W = torch.softmax(torch.randn(T, 64, device="cuda", generator=g), -1).float()
x = prepare_inputs(K, Q, W)
eng = IndexerEngine("misa", budget_k=2048, active_heads_h=8, block_size=1024, check_overflow=False)
span = eng.row_chunk(x)
print("span", span, "selector", eng.selector_params(2048, L))
for a in range(0, T, span):
    b = min(T, a + span)
    out = torch.empty(b - a, 2048, dtype=torch.int32, device="cuda")
    eng._run_rows(x.rows(a, b), False, out)
    torch.cuda.synchronize()
    f = eng.last_flags[: b - a].cpu().numpy()
    bad = np.nonzero(f)[0]
    cnt = eng._ws["sel_cnt"][: (b - a) * 4].view(b - a, 4).cpu().numpy()
    tau = eng._ws["sel_tau"][: b - a].cpu().numpy()
    print(f"pass [{a},{b}) flagged {bad.size} flags {np.unique(f[bad]) if bad.size else []}")
    if bad.size:
        print("  rows", (bad[:8] + a).tolist(), "...", (bad[-4:] + a).tolist())
        print("  counts", cnt[bad[:4]].tolist(), "tau", tau[bad[:4]].tolist())
        ok = np.nonzero(f == 0)[0]
        print("  ok counts", cnt[ok[-4:]].tolist(), "tau", tau[ok[-4:]].tolist())
