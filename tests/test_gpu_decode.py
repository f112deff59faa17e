"""Decode path: few query rows against long prefixes (C5 decode), key-axis split scoring,
long-row exact selection, and the incrementally maintained PooledKeyCache."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _inputs(L, T, H=64, d=128, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    K = torch.randn(L, d, device="cuda", generator=g).bfloat16()
    Q = torch.randn(T, H, d, device="cuda", generator=g).bfloat16()
    W = torch.softmax(torch.randn(T, H, device="cuda", generator=g), -1).float()
    return K, Q, W


@pytest.mark.parametrize("method", ["dsa", "misa", "misa_hier"])
def test_decode_rows_equal_prefill_rows(method):
    """decode() on explicit prefixes == the engine's causal-prefill rows with the same prefixes."""
    from paper_2605_07363_b200 import IndexerEngine
    L, T, k = 40000, 24, 256
    K, Q, W = _inputs(L, T, seed=3)
    rng = np.random.default_rng(0)
    pl = np.sort(rng.integers(300, L + 1, T))
    pl[-1] = L
    kw = dict(budget_k=k, active_heads_h=8, block_size=1024, candidate_kprime=1024)
    ref = IndexerEngine(method, **kw).run(K, Q, W, prefix_len=pl)
    got = IndexerEngine(method, **kw).decode(K, Q, W, prefix_len=pl)
    torch.cuda.synchronize()
    assert torch.equal(got.topk, ref.topk)
    if method != "dsa":
        assert torch.equal(got.heads, ref.heads)


def test_decode_long_prefix_matches_oracle_rows():
    """One decode row at a 200K prefix (the long-row selector path) against the CPU oracle."""
    from oracle import misa_oracle as O
    from paper_2605_07363_b200 import IndexerEngine
    L, T, k = 200000, 2, 512
    K, Q, W = _inputs(L, T, seed=5)
    out = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=1024).decode(K, Q, W)
    torch.cuda.synchronize()
    Kn = K.double().cpu().numpy()
    for t in range(T):
        ref = O.misa_select(Kn, Q[t].double().cpu().numpy(), W[t].double().cpu().numpy(), k, 8, 1024,
                            precision="fast32")
        assert out.heads[t].cpu().tolist() == ref["heads"].tolist()
        got = set(out.topk[t].cpu().tolist())
        assert len(got ^ set(ref["selection"].tolist())) <= 2


def test_pooled_key_cache_decode_equals_full_recompute():
    """Appending keys to a PooledKeyCache and decoding == decode over the full key set."""
    from paper_2605_07363_b200 import IndexerEngine
    from paper_2605_07363_b200.pooling import PooledKeyCache
    L, T, k, B = 9000, 16, 256, 512
    K, Q, W = _inputs(L, T, seed=7)
    cache = PooledKeyCache(128, B, capacity=16384)
    cache.append(K[:6000])
    eng = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=B)
    a = eng.decode(queries=Q[:8], weights=W[:8], cache=cache)
    b = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=B).decode(K[:6000], Q[:8], W[:8])
    torch.cuda.synchronize()
    assert torch.equal(a.heads, b.heads) and torch.equal(a.topk, b.topk)
    for i in range(6000, L, 1000):  # token-by-token growth in chunks
        cache.append(K[i:i + 1000])
    a = eng.decode(queries=Q[8:], weights=W[8:], cache=cache)
    b = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=B).decode(K, Q[8:], W[8:])
    torch.cuda.synchronize()
    assert cache.length == L
    assert torch.equal(a.heads, b.heads) and torch.equal(a.topk, b.topk)
