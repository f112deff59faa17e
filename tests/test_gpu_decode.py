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


@pytest.mark.parametrize("quantize,T,L", [(False, 6, 50000), (True, 6, 50000), (False, 40, 600000)])
def test_dense_long_selector_matches_sort(quantize, T, L):
    """misa_select_dense_long on long rows (incl. heavy ties -> on-device exact re-selection)
    equals a (score desc, index asc) sort.  The 40 x 600K case runs ~6000 look-back segments."""
    from paper_2605_07363_b200 import _lib
    torch.manual_seed(11)
    k = 700
    s = torch.randn(T, L, device="cuda")
    if quantize:
        s = (s * 2).round() / 2  # few distinct values: ties at the cut, candidate overflow
    n = torch.tensor(([L, L - 1, 4000, 701, 700, 30000] * T)[:T], dtype=torch.int32, device="cuda")
    n[6:] = torch.randint(1, L + 1, (max(T - 6, 0),), dtype=torch.int32)
    cap = 2048
    n_seg = -(-L // 4096)
    bufs = dict(tau=torch.empty(T, device="cuda"), seg=torch.empty(T * n_seg + 1, dtype=torch.int32, device="cuda"),
                cs=torch.empty(T, cap, device="cuda"), ci=torch.empty(T, cap, dtype=torch.int32, device="cuda"),
                cc=torch.empty(T, dtype=torch.int32, device="cuda"))
    out = torch.empty(T, k, dtype=torch.int32, device="cuda")
    outs = torch.empty(T, k, device="cuda")
    _lib.call("misa_select_dense_long", s.data_ptr(), L, n.data_ptr(), T, k, L, 2.0, bufs["tau"].data_ptr(),
              bufs["seg"].data_ptr(), bufs["cs"].data_ptr(), bufs["ci"].data_ptr(), bufs["cc"].data_ptr(), cap,
              out.data_ptr(), k, outs.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    sc = s.cpu().numpy()
    for r in range(T):
        m = int(n[r])
        order = np.argsort(-sc[r, :m], kind="stable")[: min(k, m)]  # ties -> smaller index
        exp = np.sort(order)
        got = out[r].cpu().numpy()
        assert got[: len(exp)].tolist() == exp.tolist(), r
        assert (got[len(exp):] == -1).all()
        np.testing.assert_array_equal(outs[r, : len(exp)].cpu().numpy(), sc[r, exp])


@pytest.mark.parametrize("method", ["misa", "dsa"])
def test_decode_graph_replay_matches_eager(method):
    """DecodeGraph (CUDA-graph replay, bucketed work lists, device prefix length) == eager
    decode, token after token, across a bucket boundary (re-capture)."""
    from paper_2605_07363_b200 import DecodeGraph, IndexerEngine
    from paper_2605_07363_b200.pooling import PooledKeyCache
    L0, T, k, B = 20000, 4, 256, 1024
    K, Q, W = _inputs(L0 + 600, T * 3, seed=13)
    cache = PooledKeyCache(128, B, capacity=32768)
    cache.append(K[:L0])
    eng_g = IndexerEngine(method, budget_k=k, active_heads_h=8, block_size=B)
    dg = DecodeGraph(eng_g, cache, T, 64, bucket=4096)
    for step, L in enumerate((L0, L0 + 300, L0 + 600)):  # 20000 -> bucket 20480; 20600 -> 24576
        if cache.length < L:
            cache.append(K[cache.length:L])
        q, w = Q[step * T:(step + 1) * T], W[step * T:(step + 1) * T]
        got = dg.step(q, w)
        ref = IndexerEngine(method, budget_k=k, active_heads_h=8, block_size=B).decode(queries=q, weights=w,
                                                                                       cache=cache)
        torch.cuda.synchronize()
        assert torch.equal(got.topk, ref.topk), (method, L)
        if method != "dsa":
            assert torch.equal(got.heads, ref.heads)


def test_decode_graph_misa_hier_short_cache_signed_gates():
    """MISA-dagger under DecodeGraph with a cache shorter than k' and not a bucket multiple:
    the candidate count comes from the device prefix (not the bucket length), so padded
    candidate slots never compete in the re-rank, even with signed gates (negative scores)."""
    from paper_2605_07363_b200 import DecodeGraph, IndexerEngine
    from paper_2605_07363_b200.pooling import PooledKeyCache
    T, k, B, kp = 3, 256, 512, 4096
    g = torch.Generator(device="cuda").manual_seed(41)
    K = torch.randn(3000, 128, device="cuda", generator=g).bfloat16()
    Q = torch.randn(3 * T, 16, 128, device="cuda", generator=g).bfloat16()
    W = torch.randn(3 * T, 16, device="cuda", generator=g)  # signed gates: most scores negative
    cache = PooledKeyCache(128, B, capacity=8192)
    cache.append(K[:1500])
    kw = dict(budget_k=k, active_heads_h=4, block_size=B, candidate_kprime=kp)
    dg = DecodeGraph(IndexerEngine("misa_hier", **kw), cache, T, 16, bucket=1024)
    for step, L in enumerate((1500, 2100, 3000)):
        if cache.length < L:
            cache.append(K[cache.length:L])
        q, w = Q[step * T:(step + 1) * T], W[step * T:(step + 1) * T]
        got = dg.step(q, w)
        ref = IndexerEngine("misa_hier", **kw).decode(queries=q, weights=w, cache=cache)
        torch.cuda.synchronize()
        assert torch.equal(got.topk, ref.topk), L
        assert (got.topk >= 0).all() and (got.topk < L).all()


def test_decode_graph_survives_engine_reuse():
    """Eager calls with larger shapes on the graph's engine (new workspace, work-list cache
    churn) must not invalidate the captured graph: it keeps its buffers alive."""
    from paper_2605_07363_b200 import DecodeGraph, IndexerEngine
    from paper_2605_07363_b200.pooling import PooledKeyCache
    T, k, B = 4, 256, 1024
    K, Q, W = _inputs(12000, 80, seed=43)
    cache = PooledKeyCache(128, B, capacity=16384)
    cache.append(K[:9000])
    eng = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=B)
    dg = DecodeGraph(eng, cache, T, 64)
    first = dg.step(Q[:T], W[:T]).topk.clone()
    for n in range(70):  # > 64 distinct work lists: the engine clears its cache
        eng.decode(K[:12000], Q[:8], W[:8], prefix_len=np.full(8, 3000 + 100 * n))
    eng.run(K, Q[:80], W[:80], prefix_len=np.arange(11921, 12001))  # larger workspace
    torch.cuda.synchronize()
    again = dg.step(Q[:T], W[:T]).topk
    ref = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=B).decode(queries=Q[:T], weights=W[:T],
                                                                                   cache=cache)
    torch.cuda.synchronize()
    assert torch.equal(again, first) and torch.equal(again, ref.topk)


@pytest.mark.parametrize("method,G", [("misa", 2), ("misa", 8), ("dsa", 4)])
def test_virtual_key_shards_decode_merge_to_single_gpu(method, G):
    """G key shards on one GPU: per-shard decode top-k with scores -> global index map ->
    merge == the unsharded decode (the ShardedIndexer.decode pipeline minus NCCL)."""
    from paper_2605_07363_b200 import IndexerEngine, _lib, prepare_inputs
    from paper_2605_07363_b200.engine import PreparedInputs
    from paper_2605_07363_b200.sharded import KeyShardLayout
    L, T, k, B = 70000, 6, 512, 1024
    K, Q, W = _inputs(L, T, seed=17)
    eng = IndexerEngine(method, budget_k=k, active_heads_h=8, block_size=B)
    ref = eng.decode(K, Q, W)
    x = prepare_inputs(K, Q, W, np.full(T, L))
    heads, hq = (None, x.Hp)
    if method == "misa":
        heads, hq, _ = eng.route(x)
        heads = heads.clone()
    parts_i = torch.full((G, T, k), -1, dtype=torch.int32, device="cuda")
    parts_s = torch.full((G, T, k), float("-inf"), device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for r in range(G):
        lay = KeyShardLayout(G, r, B)
        loc = torch.from_numpy(lay.local_keys(L)).cuda()
        n_loc = lay.local_count(x.prefix_host)
        Kl = x.keys.index_select(0, loc).contiguous()
        xl = PreparedInputs(Kl, x.queries, x.weights, torch.from_numpy(n_loc.astype(np.int32)).cuda(), n_loc,
                            Kl.shape[0], x.T, x.H, x.Hp, x.d, x.D, None)
        IndexerEngine(method, budget_k=k, active_heads_h=8, block_size=B).dense_select(
            xl, heads, hq, k, parts_i[r], scores=parts_s[r])
        _lib.call("misa_shard_map_indices", parts_i[r].data_ptr(), parts_i[r].numel(), B, G, r, stream)
    out = torch.empty(T, k, dtype=torch.int32, device="cuda")
    _lib.call("misa_merge_topk", parts_s.data_ptr(), parts_i.data_ptr(), G, T * k, T, k, k, out.data_ptr(), k, None,
              stream)
    torch.cuda.synchronize()
    assert torch.equal(out, ref.topk)


@pytest.mark.parametrize("method", ["misa", "dsa"])
def test_paged_key_cache_decode_equals_contiguous(method):
    """Keys in shuffled pages of a PagedKeyCache (bulk and per-token appends, partial last
    page) decode exactly like the contiguous cache: heads and top-k bit-identical."""
    from paper_2605_07363_b200 import DecodeGraph, IndexerEngine, PagedKeyCache
    from paper_2605_07363_b200.pooling import PooledKeyCache
    L, T, k, B = 9000, 6, 256, 1024
    K, Q, W = _inputs(L + 3, T, seed=21)
    rng = np.random.default_rng(0)
    paged = PagedKeyCache(128, B, n_pages=16, page_order=rng.permutation(16))
    flat = PooledKeyCache(128, B, capacity=16 * B)
    for c in (paged, flat):
        c.append(K[:5000])
        c.append(K[5000:L])
    kw = dict(budget_k=k, active_heads_h=8, block_size=B)
    a = IndexerEngine(method, **kw).decode(queries=Q, weights=W, cache=paged)
    b = IndexerEngine(method, **kw).decode(queries=Q, weights=W, cache=flat)
    torch.cuda.synchronize()
    assert torch.equal(a.topk, b.topk)
    if method != "dsa":
        assert torch.equal(a.heads, b.heads)
    for i in range(L, L + 3):  # token-by-token appends
        paged.append(K[i:i + 1])
        flat.append(K[i:i + 1])
    a = IndexerEngine(method, **kw).decode(queries=Q, weights=W, cache=paged)
    b = IndexerEngine(method, **kw).decode(queries=Q, weights=W, cache=flat)
    torch.cuda.synchronize()
    assert torch.equal(a.topk, b.topk)


def test_decode_graph_over_paged_cache():
    """DecodeGraph replay over a PagedKeyCache (page-bucketed capture) == eager paged decode."""
    from paper_2605_07363_b200 import DecodeGraph, IndexerEngine, PagedKeyCache
    L0, T, k, B = 5000, 2, 256, 1024
    K, Q, W = _inputs(L0 + 1100, T * 3, seed=23)
    rng = np.random.default_rng(1)
    cache = PagedKeyCache(128, B, n_pages=8, page_order=rng.permutation(8))
    cache.append(K[:L0])
    dg = DecodeGraph(IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=B), cache, T, 64)
    for step, L in enumerate((L0, L0 + 500, L0 + 1100)):  # crosses a page boundary (re-capture)
        if cache.length < L:
            cache.append(K[cache.length:L])
        q, w = Q[step * T:(step + 1) * T], W[step * T:(step + 1) * T]
        got = dg.step(q, w)
        ref = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=B).decode(queries=q, weights=w,
                                                                                       cache=cache)
        torch.cuda.synchronize()
        assert torch.equal(got.topk, ref.topk) and torch.equal(got.heads, ref.heads), L


@pytest.mark.parametrize("method,L,T", [("misa", 300000, 16), ("dsa", 70000, 8), ("misa_hier", 50000, 12),
                                        ("misa", 5000, 9)])
def test_decode_fused_filter_equals_dense_path(method, L, T):
    """Decode rows through the fused filter (sample -> tau -> key-split filter with atomic slot
    reservation -> unordered cut -> row sort) == the materialised dense path, bit for bit;
    L > 262144 exercises the unordered selector past topk5's chunk-scan range."""
    from paper_2605_07363_b200 import IndexerEngine
    K, Q, W = _inputs(L, T, seed=11)
    rng = np.random.default_rng(1)
    pl = rng.integers(max(1, L // 3), L + 1, T)
    pl[0], pl[-1] = L, min(L, 700)
    kw = dict(budget_k=512, active_heads_h=8, block_size=1024, candidate_kprime=2048)
    fused = IndexerEngine(method, **kw)
    fused.decode_filter_min_rows, fused.decode_filter_min_keys = 1, 1
    dense = IndexerEngine(method, **kw)
    dense.decode_filter_min_rows = 1 << 30
    a = fused.decode(K, Q, W, prefix_len=pl)
    assert fused.last_decode_flags is not None
    b = dense.decode(K, Q, W, prefix_len=pl)
    torch.cuda.synchronize()
    assert torch.equal(a.topk, b.topk)
    if method == "misa_hier":
        assert torch.equal(a.candidates, b.candidates)


def test_decode_fused_filter_flagged_rows_are_exact():
    """All-equal keys: every score ties, every key passes tau, the candidate lists overflow and
    the rows are flagged; eager decode and DecodeGraph re-select them exactly (ties -> smaller
    index: the first k keys)."""
    from paper_2605_07363_b200 import DecodeGraph, IndexerEngine
    from paper_2605_07363_b200.pooling import PooledKeyCache
    L, T, k = 40000, 8, 256
    _, Q, W = _inputs(L, T, seed=13)
    K = torch.ones(L, 128, device="cuda").bfloat16()
    eng = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=1024)
    eng.decode_filter_min_rows, eng.decode_filter_min_keys = 1, 1
    out = eng.decode(K, Q, W)
    torch.cuda.synchronize()
    assert eng.last_fallback_rows > 0
    exp = torch.arange(k, dtype=torch.int32, device="cuda").expand(T, k)
    assert torch.equal(out.topk, exp)
    cache = PooledKeyCache(128, 1024, capacity=L)
    cache.append(K)
    eg = IndexerEngine("misa", budget_k=k, active_heads_h=8, block_size=1024)
    eg.decode_filter_min_rows, eg.decode_filter_min_keys = 1, 1
    dg = DecodeGraph(eg, cache, T, 64)
    r = dg.step(Q, W)
    torch.cuda.synchronize()
    assert torch.equal(r.topk, exp)
