"""The reference's invariants (pkg/tests/test_routing.py, test_dsa.py) on the device path, plus a
hypothesis sweep of small random workloads against the oracle."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

from oracle import misa_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

TAU_S = 1e-5  # score tolerance relative to sum |w| |q.k| (bf16 operands, f32 accumulation)


def _workload(seed, L, H, d, raw=False, scale=1.0):
    from paper_2605_07363_b200 import IndexerWorkload
    K, Q, W = O.synthetic_prefill(seed, L, H, d, T=1, raw_gates=raw)
    return IndexerWorkload(K, Q[0] * scale, W[0].astype(np.float32).astype(np.float64))  # f32 gates: exact on device


def _near_tie_ok(got, exp, scores, mag, k):
    """got / exp index sets differ only in elements tied with the k-th score within tolerance."""
    if got == exp:
        return True
    kth = np.sort(scores)[::-1][min(k, scores.shape[0]) - 1]
    return all(abs(scores[i] - kth) <= TAU_S * (mag[i] + abs(kth)) + 1e-12 for i in set(got) ^ set(exp))


def test_all_heads_routed_score_is_the_dense_score():
    """misa_score over every head == dsa_score bit for bit (test_routing.py:108-111)."""
    from paper_2605_07363_b200 import HeadSet, dsa_score, misa_score
    for H, d, L in ((8, 64, 777), (16, 128, 2000), (64, 128, 3000)):
        w = _workload(1, L, H, d)
        a = misa_score(w, HeadSet(np.arange(H), H)).values
        b = dsa_score(w).values
        assert np.array_equal(a, b), (H, d, L)


def test_routed_score_bounded_by_dense_score():
    """I-hat <= I for non-negative gates (test_routing.py:221-228)."""
    from paper_2605_07363_b200 import HeadSet, dsa_score, misa_score
    w = _workload(2, 4000, 64, 128)
    dense = dsa_score(w).values
    for heads in (np.arange(8), np.arange(0, 64, 8), np.array([3, 17, 40, 63])):
        routed = misa_score(w, HeadSet(heads, 64)).values
        assert np.all(routed <= dense * (1 + 1e-6) + 1e-7)


def test_selection_scale_invariance():
    """Scaling queries (x2, exact in bf16) or gates (x0.5) leaves every selection unchanged
    (test_routing.py:231-240, test_dsa.py:83-93)."""
    from paper_2605_07363_b200 import IndexerWorkload, make_indexer
    w = _workload(3, 3000, 32, 64)
    variants = [IndexerWorkload(w.keys, w.queries * 2.0, w.gate_weights),
                IndexerWorkload(w.keys, w.queries, w.gate_weights * 0.5)]
    for m, kw in (("dsa", {}), ("misa", dict(block_size=256)), ("misa_hier", dict(block_size=256,
                                                                                    candidate_kprime=1024))):
        ind = make_indexer(m, budget_k=200, **kw)
        base = ind.select(w)
        for v in variants:
            r = ind.select(v)
            assert r.selection.indices.tolist() == base.selection.indices.tolist(), m
            if base.heads is not None:
                assert r.heads.head_indices.tolist() == base.heads.head_indices.tolist(), m


def test_dense_selection_head_permutation_invariance():
    """Permuting the indexer heads (queries and gates together) does not change the dense
    selection beyond score ties (test_dsa.py:96-105)."""
    from paper_2605_07363_b200 import IndexerWorkload, dsa_select
    w = _workload(4, 3500, 64, 128)
    perm = np.random.default_rng(0).permutation(64)
    p = IndexerWorkload(w.keys, w.queries[perm], w.gate_weights[perm])
    a = dsa_select(w, 300).selection.indices.tolist()
    b = dsa_select(p, 300).selection.indices.tolist()
    scores = O.gated_relu_scores(w.keys, w.queries, w.gate_weights, "fast32")
    mag = np.abs(w.gate_weights) @ np.abs(w.queries @ w.keys.T)
    assert _near_tie_ok(a, b, scores, mag, 300)


# MISA_HYPOTHESIS_EXAMPLES / MISA_HYPOTHESIS_SEED widen the sweep (default: 30 fixed examples)
@settings(max_examples=int(os.environ.get("MISA_HYPOTHESIS_EXAMPLES", 30)), deadline=None,
          derandomize="MISA_HYPOTHESIS_SEED" not in os.environ)
@given(L=st.integers(1, 700), H=st.sampled_from([4, 8, 16]), d=st.sampled_from([16, 32, 64]),
       k=st.integers(1, 260), h=st.integers(1, 8), B=st.sampled_from([1, 7, 64, 128]),
       raw=st.booleans(), seed=st.integers(0, 10_000))
def test_random_workloads_match_oracle(L, H, d, k, h, B, raw, seed):
    """Random small workloads (any L, k >= L, B > L, signed gates, h > H clamped) through the
    estimators == the oracle at fast32 on the same bf16 data, heads exact up to ties."""
    from paper_2605_07363_b200 import make_indexer
    w = _workload(seed, L, H, d, raw=raw)
    K, q, g = w.keys, w.queries, w.gate_weights
    hh = min(h, H)
    kp = max(k, 2 * k)
    dense = O.gated_relu_scores(K, q, g, "fast32")
    mag = np.abs(g) @ np.abs(q @ K.T)
    r = make_indexer("dsa", budget_k=k).select(w)
    exp = O.dsa_select(K, q, g, k, "fast32")["selection"].tolist()
    assert _near_tie_ok(r.selection.indices.tolist(), exp, dense, mag, k)
    rm = make_indexer("misa", budget_k=k, active_heads_h=h, block_size=B).select(w)
    om = O.misa_select(K, q, g, k, hh, B, precision="fast32")
    heads = rm.heads.head_indices
    if heads.tolist() == om["heads"].tolist():
        ms = O.misa_score(K, q, g, heads, "fast32")
        hm = np.abs(g[heads]) @ np.abs(q[heads] @ K.T)
        assert _near_tie_ok(rm.selection.indices.tolist(), om["selection"].tolist(), ms, hm, k)
    else:  # a router tie: the reference's h-th and (h+1)-th importances agree within 1e-5
        E = O.route_head_importance(q, g, O.block_pool(K, B)[1], precision="fast32")
        hth = np.sort(E)[::-1][hh - 1]
        for j in set(heads.tolist()) ^ set(om["heads"].tolist()):
            assert abs(E[j] - hth) <= 1e-5 * abs(hth) + 1e-12
    rh = make_indexer("misa_hier", budget_k=k, active_heads_h=h, block_size=B, candidate_kprime=kp).select(w)
    assert len(rh.selection) == min(k, L) and len(rh.candidates) == min(kp, L)
    assert set(rh.selection.indices.tolist()) <= set(rh.candidates.indices.tolist())
