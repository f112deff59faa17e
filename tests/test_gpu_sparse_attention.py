"""Sparse attention over the indexer's selection (Eq. 3, MQA mode) against an fp32
torch restatement on the same gathered rows."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _reference(q, kv, topk, dv, scale):
    T, H, d = q.shape
    out = torch.zeros(T, H, dv, dtype=torch.float32, device=q.device)
    for t in range(T):
        sel = topk[t][topk[t] >= 0].long()
        if sel.numel() == 0:
            continue
        c = kv[sel].float()
        s = scale * (q[t].float() @ c.T)
        p = torch.softmax(s, dim=-1)
        out[t] = p @ c[:, :dv]
    return out


@pytest.mark.parametrize("H,d,dv,k", [(128, 128, 128, 512), (16, 128, 64, 300), (64, 256, 256, 260),
                                      (128, 256, 128, 128)])
def test_sparse_attention_matches_fp32(H, d, dv, k):
    from paper_2605_07363_b200 import IndexerEngine
    from paper_2605_07363_b200.sparse_attention import sparse_attention
    g = torch.Generator(device="cuda").manual_seed(d + k)
    L, T = 3000, 40
    kv = torch.randn(L, d, device="cuda", generator=g).bfloat16()
    q = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
    # a real selection: the MISA indexer's top-k of these rows (short prefixes give -1 padding)
    Qi = torch.randn(T, 8, 128, device="cuda", generator=g).bfloat16()
    Wi = torch.softmax(torch.randn(T, 8, device="cuda", generator=g), -1)
    Ki = torch.randn(L, 128, device="cuda", generator=g).bfloat16()
    pl = np.linspace(1, L, T).astype(np.int64)
    topk = IndexerEngine("misa", budget_k=k, active_heads_h=2, block_size=128).run(Ki, Qi, Wi, prefix_len=pl).topk
    scale = 1.0 / math.sqrt(d)
    got = sparse_attention(q, kv, topk, dv, scale)
    exp = _reference(q, kv, topk, dv, scale)
    torch.cuda.synchronize()
    err = (got - exp).abs().max().item()
    assert err <= 2e-2 * exp.abs().max().item() + 1e-3, err


def test_sparse_attention_empty_and_single_token_rows():
    from paper_2605_07363_b200.sparse_attention import sparse_attention
    g = torch.Generator(device="cuda").manual_seed(1)
    kv = torch.randn(500, 128, device="cuda", generator=g).bfloat16()
    q = torch.randn(3, 8, 128, device="cuda", generator=g).bfloat16()
    topk = torch.full((3, 256), -1, dtype=torch.int32, device="cuda")
    topk[1, 0] = 7                       # one token: the output is that token's value row
    topk[2, :200] = torch.arange(0, 400, 2, device="cuda")
    got = sparse_attention(q, kv, topk, 128)
    torch.cuda.synchronize()
    assert torch.count_nonzero(got[0]) == 0
    assert torch.allclose(got[1], kv[7].float().expand(8, 128), atol=1e-2)
    exp = _reference(q, kv, topk, 128, 1 / math.sqrt(128))
    assert (got[2] - exp[2]).abs().max().item() <= 2e-2 * exp[2].abs().max().item() + 1e-3
