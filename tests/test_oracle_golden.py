"""Pin the numpy oracle against the reference's own golden vectors (CPU only).

Fixtures in tests/golden were produced by running the reference package
(oracle/make_golden.py).  The hand-derived known-answer vectors below are the
ones the reference's unit tests assert (file:line cited per test).
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import misa_oracle as O

CASES = ["tiny_softmax", "tiny_signed", "small_h64", "glm_h32", "c1_sampled"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _load(golden_dir, name):
    return dict(np.load(os.path.join(golden_dir, f"{name}.npz")))


def _inputs(g):
    seed, L, H, d, h, B, k, kp, raw = (int(x) for x in g["meta"])
    if "K" in g:
        K, Q, W = g["K"], g["Q"], g["W"]
    else:
        K, Q, W = O.synthetic_prefill(seed, L, H, d, raw_gates=bool(raw))
    assert _sha(K) == str(g["sha_K"]) and _sha(Q) == str(g["sha_Q"]) and _sha(W) == str(g["sha_W"])
    return (K, Q, W), (seed, L, H, d, h, B, k, kp, raw)


# ---------------------------------------------------------- known answers --
def test_known_answer_scores():
    # test_dsa.py:14-17: one head, dots [2,-1,3] -> [2,0,3]
    np.testing.assert_array_equal(O.gated_relu_scores([[2.0], [-1.0], [3.0]], [[1.0]], [1.0]), [2, 0, 3])
    # test_dsa.py:20-23: zero gates -> zeros
    np.testing.assert_array_equal(
        O.gated_relu_scores([[1.0, 2.0], [3.0, 4.0]], [[1.0, 0.0], [0.0, 1.0]], [0.0, 0.0]), [0, 0])
    # test_dsa.py:26-28 / support.py:23-29: per-head dots [[4,-2],[0,6]], w=[.5,.5] -> [2,3]
    keys, qs, ws = [[4.0, 0.0], [-2.0, 6.0]], [[1.0, 0.0], [0.0, 1.0]], [0.5, 0.5]
    np.testing.assert_array_equal(O.gated_relu_scores(keys, qs, ws), [2.0, 3.0])
    # test_routing.py:121-125: head {0} -> [2, 0]
    np.testing.assert_array_equal(O.misa_score(keys, qs, ws, [0]), [2.0, 0.0])


def test_known_answer_topk_and_route():
    assert O.topk_tokens(np.array([5.0, 5.0, 1.0]), 1).tolist() == [0]           # test_dsa.py:45-47
    assert O.topk_tokens(np.array([0.3, 0.1, 0.2]), 2048).tolist() == [0, 1, 2]  # test_dsa.py:38-42
    assert O.route_topk_heads(np.array([0.0, 5.0, 5.0, 1.0]), 2).tolist() == [1, 2]  # test_routing.py:95-97
    assert O.route_topk_heads(np.array([0.1, 0.4, 0.2]), 3).tolist() == [0, 1, 2]    # test_routing.py:90-92


def test_known_answer_router():
    # test_routing.py:37-45: aligned block -> E = [4, 0, 0]
    queries = [[2.0, 0, 0, 0], [0, 3.0, 0, 0], [0, 0, 1.0, 0]]
    keys = np.tile([2.0, 0, 0, 0], (4, 1))
    _, pooled = O.block_pool(keys, 8)
    np.testing.assert_allclose(O.route_head_importance(queries, [1.0] * 3, pooled), [4, 0, 0], atol=1e-12)
    # test_routing.py:243-252: signed gates -> |.| matters, E=[2.0, 0.5]
    keys = np.tile([1.0, 0.0], (4, 1))
    _, pooled = O.block_pool(keys, 4)
    E = O.route_head_importance([[1.0, 0.0], [0.5, 0.0]], [-2.0, 1.0], pooled)
    np.testing.assert_allclose(E, [2.0, 0.5], atol=1e-12)
    assert O.route_topk_heads(E, 1).tolist() == [0]


def test_known_answer_ledgers():
    # test_dsa.py:59-65: H=64, L=4096 -> 262144 token products
    rng = np.random.default_rng(0)
    K, Q, W = rng.standard_normal((4096, 8)), rng.standard_normal((64, 8)), np.full(64, 1 / 64)
    assert O.dsa_select(K, Q, W, 64)["ledger"] == (("token_scan", "token", 262144),)
    # test_routing.py:209-218 shape: router H*M, token h*L, refine H*min(k',L)
    K, Q, W = rng.standard_normal((64, 8)), rng.standard_normal((8, 8)), np.full(8, 1 / 8)
    r = O.misa_hier_select(K, Q, W, 8, 2, 16, 24)
    assert [e[2] for e in r["ledger"]] == [8 * 4, 2 * 64, 8 * 24]


# ---------------------------------------------------------- pooling goldens --
def test_pooling_golden(golden_dir):
    g = _load(golden_dir, "pooling")
    for B in (1, 4, 8, 64):
        bounds, pooled = O.block_pool(g["keys"], B)
        assert bounds.tolist() == g[f"bounds_{B}"].tolist()
        np.testing.assert_allclose(pooled, g[f"pooled_{B}"], atol=1e-12)
    bounds, pooled = np.empty((0, 2), np.int64), np.empty((0, 5))
    for row in g["keys"]:
        bounds, pooled = O.incremental_append(bounds, pooled, row, 4)
    assert bounds.tolist() == g["incr_bounds_4"].tolist()
    np.testing.assert_allclose(pooled, g["incr_pooled_4"], atol=1e-12)


# ------------------------------------------------------- batched goldens ----
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("prec", ["fast32", "reference64"])
def test_batched_selections_match_reference(golden_dir, name, prec):
    g = _load(golden_dir, name)
    (K, Q, W), (seed, L, H, d, h, B, k, kp, raw) = _inputs(g)
    rows = g["rows"].tolist()
    if name == "c1_sampled" and prec == "reference64":
        rows = rows[:6] + rows[-2:]
    for i, t in enumerate(g["rows"].tolist()):
        if t not in rows:
            continue
        kw = dict(k=k, h=h, block_size=B, kprime=kp, precision=prec)
        r_d = O.row_select("dsa", K, Q, W, t + 1, t, **kw)
        r_m = O.row_select("misa", K, Q, W, t + 1, t, **kw)
        r_h = O.row_select("misa_hier", K, Q, W, t + 1, t, **kw)
        exp = lambda key: g[f"{prec}_{key}"][i][g[f"{prec}_{key}"][i] >= 0].tolist()  # noqa: E731
        assert r_d["selection"].tolist() == exp("dsa"), (name, t)
        assert r_m["selection"].tolist() == exp("misa"), (name, t)
        assert r_m["heads"].tolist() == exp("heads"), (name, t)
        assert r_h["selection"].tolist() == exp("hier"), (name, t)
        assert r_h["candidates"].tolist() == exp("hier_cand"), (name, t)
        np.testing.assert_allclose(r_m["importance"], g[f"{prec}_importance"][i], rtol=1e-12, atol=1e-15)
        ledg = [sum(e[2] for e in r["ledger"] if e[1] == kind)
                for r in (r_d, r_m, r_h) for kind in ("token", "block", "refine")]
        assert ledg == g[f"{prec}_ledger"][i].reshape(-1).tolist()


def test_last_row_scores(golden_dir):
    for name in ("tiny_softmax", "tiny_signed", "small_h64", "glm_h32"):
        g = _load(golden_dir, name)
        (K, Q, W), (seed, L, H, d, h, B, k, kp, raw) = _inputs(g)
        t = int(g["rows"][-1])
        np.testing.assert_array_equal(O.gated_relu_scores(K[: t + 1], Q[t], W[t], "fast32"),
                                      g["fast32_last_dsa_scores"])
        heads = g["fast32_heads"][-1]
        np.testing.assert_array_equal(O.misa_score(K[: t + 1], Q[t], W[t], heads[heads >= 0], "fast32"),
                                      g["fast32_last_misa_scores"])


def test_needle_goldens(golden_dir):
    g = _load(golden_dir, "needles")
    for i in range(3):
        seed, L, depth, align = g[f"spec{i}"].tolist()
        K, Q, W, label = O.needle_workload(int(seed), int(L), depth, 32, 10.0, 64, 64,
                                           align_head=None if align < 0 else int(align))
        assert _sha(K) + _sha(Q) + _sha(W) == str(g[f"sha{i}"])
        assert list(label) == g[f"label{i}"].tolist()
        k = int(g[f"k{i}"])
        for prec in ("reference64", "fast32"):
            assert O.dsa_select(K, Q, W, k, prec)["selection"].tolist() == g[f"{prec}_dsa{i}"].tolist()
            r = O.misa_select(K, Q, W, k, 8, 1024, precision=prec)
            assert r["selection"].tolist() == g[f"{prec}_misa{i}"].tolist()
            assert r["heads"].tolist() == g[f"{prec}_heads{i}"].tolist()
