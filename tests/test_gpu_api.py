"""Reference-facing API on the GPU: estimators, registry, pure functions, ledgers, decode pooling."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import misa_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def _bf16_workload(seed, L, H, d, raw=False):
    from paper_2605_07363_b200 import IndexerWorkload
    K, Q, W = O.synthetic_prefill(seed, L, H, d, T=1, raw_gates=raw)
    return IndexerWorkload(K, Q[0], W[0], seed)


def test_estimators_select_and_ledger():
    from paper_2605_07363_b200 import make_indexer, METHODS, cost_ratio
    w = _bf16_workload(0, 4096, 64, 128)
    res = {m: make_indexer(m, budget_k=256, **({} if m == "dsa" else {"block_size": 64})).select(w) for m in METHODS}
    assert res["dsa"].ledger.total() == 64 * 4096
    assert res["misa"].ledger.token_dot_products == 8 * 4096
    assert res["misa"].ledger.block_dot_products == 64 * 64
    assert res["misa_hier"].ledger.stage_labels == ("router", "token_scan", "refine")
    assert res["misa_hier"].ledger.refine_dot_products == 64 * min(8192, 4096)
    for m in METHODS:
        sel = res[m].selection
        assert len(sel) == 256 and sel.prefix_len == 4096
        assert np.all(np.diff(sel.indices) > 0)
    exp = O.dsa_select(w.keys, w.queries, w.gate_weights, 256, "fast32")["selection"]
    assert res["dsa"].selection.indices.tolist() == exp.tolist()
    assert cost_ratio(res["misa"].ledger, res["dsa"].ledger) > 1


def test_reference_scale_ledger_ratios():
    """Acceptance criterion 4 constants: H=64, h=8, B=1024, L=131072, k'=8192 -> 7.94x / 5.31x."""
    from paper_2605_07363_b200 import DSAIndexer, MISAIndexer, HierarchicalMISAIndexer, cost_ratio
    w = _bf16_workload(424242, 131072, 64, 64)
    d = DSAIndexer().select(w)
    m = MISAIndexer().select(w)
    h = HierarchicalMISAIndexer().select(w)
    assert d.ledger.total() == 8388608 and m.ledger.total() == 1056768 and h.ledger.total() == 1581056
    assert abs(cost_ratio(m.ledger, d.ledger) - 7.94) <= 0.01
    assert abs(cost_ratio(h.ledger, d.ledger) - 5.31) <= 0.01
    exp = O.misa_select(w.keys, w.queries, w.gate_weights, 2048, 8, 1024, precision="fast32")
    assert m.heads.head_indices.tolist() == exp["heads"].tolist()
    inter = len(set(m.selection.indices.tolist()) & set(exp["selection"].tolist()))
    assert inter >= 0.999 * 2048


def test_router_kinds_and_transform():
    from paper_2605_07363_b200 import MISAIndexer, build_block_summary, route_head_importance, route_topk_heads
    w = _bf16_workload(5, 3000, 16, 64, raw=True)
    s = build_block_summary(w.keys, 256)
    for kind in ("block_attention", "gate_only", "query_norm"):
        E = route_head_importance(w, s, kind).values
        _, pooled = O.block_pool(w.keys, 256)
        ref = O.route_head_importance(w.queries, w.gate_weights, pooled, kind, "fast32")
        np.testing.assert_allclose(E, ref, rtol=2e-5, atol=1e-9)
        assert route_topk_heads(E, 4).head_indices.tolist() == O.route_topk_heads(ref, 4).tolist()
        r = MISAIndexer(budget_k=64, active_heads_h=4, block_size=256, router_score=kind).select(w)
        assert r.ledger.block_dot_products == (16 * 12 if kind == "block_attention" else 0)
    est = MISAIndexer(budget_k=64, active_heads_h=4, block_size=256)
    assert est.transform(w).tolist() == est.select(w).selection.indices.tolist()


def test_pooling_and_incremental_append():
    from paper_2605_07363_b200 import build_block_summary, incremental_append, PooledKeyCache
    rng = np.random.default_rng(9)
    keys = O.bf16_round(rng.standard_normal((37, 5)))
    for B in (1, 4, 8, 64):
        s = build_block_summary(keys, B)
        b, p = O.block_pool(keys, B)
        assert s.boundaries.tolist() == b.tolist()
        np.testing.assert_allclose(s.pooled_keys, p, rtol=1e-6, atol=1e-6)
    s = build_block_summary(np.empty((0, 5)), 4)
    for row in keys:
        s = incremental_append(s, row)
    b, p = O.block_pool(keys, 4)
    assert s.boundaries.tolist() == b.tolist()
    np.testing.assert_allclose(s.pooled_keys, p, rtol=1e-6, atol=1e-6)
    cache = PooledKeyCache(5, 4, 64)
    cache.append(keys[:20])
    cache.append(keys[20:])
    cs = cache.summary()
    np.testing.assert_allclose(cs.pooled_keys, p, rtol=1e-6, atol=1e-6)


def test_topk_primitives():
    from paper_2605_07363_b200 import topk_tokens, topk_within
    assert topk_tokens(np.array([5.0, 5.0, 1.0]), 1).indices.tolist() == [0]
    assert topk_tokens(np.array([0.3, 0.1, 0.2]), 2048).indices.tolist() == [0, 1, 2]
    rng = np.random.default_rng(1)
    for _ in range(20):
        s = np.round(rng.standard_normal(300), 1)
        k = int(rng.integers(1, 300))
        assert topk_tokens(s, k).indices.tolist() == O.topk_tokens(s, k).tolist()
        cand = np.sort(rng.choice(1000, 300, replace=False))
        assert topk_within(s, cand, k, 1000).indices.tolist() == O.topk_within(s, cand, k).tolist()


def test_errors_follow_reference_convention():
    from paper_2605_07363_b200 import DSAIndexer, MISAIndexer, HierarchicalMISAIndexer, make_indexer
    w = _bf16_workload(1, 64, 8, 8)
    with pytest.raises(ValueError):
        DSAIndexer(budget_k=0).select(w)
    with pytest.raises(ValueError):
        MISAIndexer(router_score="entropy").select(w)
    with pytest.raises(ValueError):
        HierarchicalMISAIndexer(budget_k=32, candidate_kprime=16).select(w)
    with pytest.raises(ValueError):
        make_indexer("dense")
    assert len(MISAIndexer(budget_k=8, active_heads_h=32, block_size=8).select(w).heads) == 8


def test_select_batch_host_pipeline_equals_device_path():
    """Pinned host inputs take the copy-overlapped row-chunk pipeline; same top-k as on device."""
    import torch
    from paper_2605_07363_b200 import MISAIndexer
    g = torch.Generator().manual_seed(4)
    L, H, d = 12000, 64, 128
    K = torch.randn(L, d, generator=g).bfloat16()
    Q = torch.randn(L, H, d, generator=g).bfloat16()
    W = torch.softmax(torch.randn(L, H, generator=g), -1).float()
    est = MISAIndexer(budget_k=512, active_heads_h=8, block_size=1024)
    host = est.select_batch(K.pin_memory(), Q.pin_memory(), W.pin_memory()).topk
    torch.cuda.synchronize()
    dev = est.select_batch(K.cuda(), Q.cuda(), W.cuda()).topk
    torch.cuda.synchronize()
    assert not host.is_cuda and torch.equal(host, dev.cpu())


def test_host_pipeline_ragged_prefixes_and_chunk_counts():
    """The host pipeline (row chunks processed last rows first, the first chunk split again,
    a ring of device buffers) returns the device path's top-k for arbitrary prefix lengths and
    every chunk count, including more chunks than rows fit evenly."""
    import numpy as np
    import torch
    from paper_2605_07363_b200 import IndexerEngine
    g = torch.Generator().manual_seed(5)
    L, T, H, d = 9000, 3001, 32, 128
    K = torch.randn(L, d, generator=g).bfloat16()
    Q = torch.randn(T, H, d, generator=g).bfloat16()
    W = torch.softmax(torch.randn(T, H, generator=g), -1).float()
    pl = np.random.default_rng(5).integers(1, L + 1, T)
    eng = IndexerEngine("misa", budget_k=256, active_heads_h=4, block_size=256)
    dev = eng.run(K.cuda(), Q.cuda(), W.cuda(), prefix_len=pl).topk.cpu()
    for chunks in (1, 3, 8, 13):
        host = eng.run_host(K.pin_memory(), Q.pin_memory(), W.pin_memory(), pl, chunks=chunks)
        assert torch.equal(host, dev), chunks


def test_constructive_needle_retrieval():
    """Acceptance criterion 5 (``test_acceptance.py:203-243``) through the GPU registry:
    margin-10, 32-token needles aligned with the top-gate head are fully retrieved by the
    dense, routed and hierarchical indexers at every length and depth of the reference grid."""
    from paper_2605_07363_b200 import IndexerConfig, gen_needle_workload, make_indexer, needle_recall
    cfg = IndexerConfig()
    misses = []
    for li, L in enumerate((1024, 2048, 4096, 8192)):
        k = min(cfg.budget_k, L // 4)
        idx = {m: make_indexer(m, budget_k=k) for m in ("dsa", "misa", "misa_hier")}
        for di in range(11):
            for rep in range(2):
                w = gen_needle_workload(1000 * li + 10 * di + rep, L, di / 10, 32, 10.0, cfg, noise_scale=0.01)
                for m, ix in idx.items():
                    if needle_recall(ix.select(w).selection, w.label.interval) < 1.0:
                        misses.append((m, L, di, rep))
    assert not misses, misses[:5]
