"""CPU oracle for the MISA / DSA indexer hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's indexer
algorithm (``/root/reference/pkg/src/misa``).  It exists to check the CUDA
path; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
package (``paper_2605_07363_b200``) never imports, calls or links anything
here, and has no CPU fallback.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function below
against golden vectors produced by running the reference itself
(``oracle/make_golden.py`` imports ``/root/reference/pkg/src``; the vectors are
committed under ``tests/golden/``) and against the hand-derived known-answer
vectors of the reference's own unit tests.

Every function cites the reference file:line it restates.  Precision modes:
``reference64`` computes f64 dot products; ``fast32`` rounds operands to f32
and returns the correctly rounded f32 value of each (f64-accumulated) dot
(``dsa.py:18-34``).  The gating epilogue is always f64 (``dsa.py:53``).
"""

from __future__ import annotations

import numpy as np

REFERENCE64 = "reference64"
FAST32 = "fast32"
BLOCK_ATTENTION = "block_attention"
GATE_ONLY = "gate_only"
QUERY_NORM = "query_norm"


# ---------------------------------------------------------------- dsa.py ----
def relevance_dots(keys: np.ndarray, queries: np.ndarray, precision: str = REFERENCE64) -> np.ndarray:
    """(R, d) x (N, d) -> (N, R) dots.  Restates ``dsa.py:18-34``."""
    if precision == FAST32:
        q = np.asarray(queries, dtype=np.float32).astype(np.float64)
        k = np.asarray(keys, dtype=np.float32).astype(np.float64)
        return (q @ k.T).astype(np.float32).astype(np.float64)
    return np.asarray(queries, dtype=np.float64) @ np.asarray(keys, dtype=np.float64).T


def gated_relu_scores(keys, queries, gates, precision: str = REFERENCE64) -> np.ndarray:
    """sum_j w_j * ReLU(q_j . k_s) per key row.  Restates ``dsa.py:37-53``."""
    dots = relevance_dots(keys, queries, precision)
    np.maximum(dots, 0, out=dots)
    return np.asarray(gates, dtype=np.float64) @ dots


def topk_tokens(values: np.ndarray, k: int) -> np.ndarray:
    """min(k, L) largest, ties -> smaller index, ascending output.  ``dsa.py:64-76``."""
    values = np.asarray(values)
    keep = min(int(k), int(values.shape[0]))
    order = np.argsort(-values, kind="stable")
    return np.sort(order[:keep])


def topk_within(scores: np.ndarray, candidates: np.ndarray, k: int) -> np.ndarray:
    """Top-k inside an ascending candidate list, ties -> smaller global index.  ``dsa.py:79-92``."""
    keep = min(int(k), int(candidates.shape[0]))
    order = np.argsort(-np.asarray(scores), kind="stable")
    return np.sort(np.asarray(candidates)[order[:keep]])


# ------------------------------------------------------------ pooling.py ----
def block_pool(keys: np.ndarray, block_size: int) -> tuple[np.ndarray, np.ndarray]:
    """Contiguous blocks + mean pooling (partial last block over its real length).

    Restates ``pooling.py:57-84``.  Returns (boundaries (M,2) int64, pooled (M,d) f64).
    """
    keys = np.asarray(keys, dtype=np.float64)
    L = keys.shape[0]
    if L == 0:
        return np.empty((0, 2), np.int64), np.empty((0, keys.shape[1]))
    m = -(-L // block_size)
    starts = np.arange(m, dtype=np.int64) * block_size
    ends = np.minimum(starts + block_size, L)
    sums = np.add.reduceat(keys, starts, axis=0)
    return np.stack([starts, ends], axis=1), sums / (ends - starts)[:, None]


def incremental_append(bounds: np.ndarray, pooled: np.ndarray, new_key: np.ndarray, block_size: int):
    """Running-mean decode update.  Restates ``pooling.py:87-115``."""
    new_key = np.asarray(new_key, dtype=np.float64).reshape(-1)
    if bounds.shape[0] == 0:
        return np.array([[0, 1]], np.int64), new_key[None, :].copy()
    start, end = bounds[-1]
    length = int(end - start)
    if length < block_size:
        pooled = pooled.copy()
        pooled[-1] = pooled[-1] + (new_key - pooled[-1]) / (length + 1)
        bounds = bounds.copy()
        bounds[-1, 1] = end + 1
        return bounds, pooled
    return np.vstack([bounds, [[end, end + 1]]]), np.vstack([pooled, new_key[None, :]])


# ------------------------------------------------------------ routing.py ----
def route_head_importance(queries, gates, pooled, kind: str = BLOCK_ATTENTION,
                          precision: str = REFERENCE64) -> np.ndarray:
    """Per-head importance E_j.  Restates ``routing.py:38-64``.

    block_attention: mean_b |w_j ReLU(q_j . pooled_b)|; gate_only: w_j;
    query_norm: ||q_j||_2.
    """
    gates = np.asarray(gates, dtype=np.float64)
    if kind == GATE_ONLY:
        return gates.copy()
    if kind == QUERY_NORM:
        return np.linalg.norm(np.asarray(queries, dtype=np.float64), axis=1)
    aff = relevance_dots(pooled, queries, precision)
    np.maximum(aff, 0, out=aff)
    aff *= gates[:, None]
    np.abs(aff, out=aff)
    return aff.mean(axis=1)


def route_topk_heads(importance: np.ndarray, h: int) -> np.ndarray:
    """min(h, H) most important heads, ties -> smaller head, ascending.  ``routing.py:67-75``."""
    order = np.argsort(-np.asarray(importance), kind="stable")
    return np.sort(order[: min(int(h), importance.shape[0])])


def misa_score(keys, queries, gates, heads, precision: str = REFERENCE64) -> np.ndarray:
    """Routed-head token scores.  Restates ``routing.py:78-99``."""
    heads = np.asarray(heads)
    return gated_relu_scores(keys, np.asarray(queries)[heads], np.asarray(gates)[heads], precision)


# ------------------------------------------------------- selectors (one query)
def dsa_select(keys, queries, gates, k, precision=REFERENCE64) -> dict:
    """Dense selection + ledger.  Restates ``dsa.py:118-132``."""
    scores = gated_relu_scores(keys, queries, gates, precision)
    H, L = np.asarray(queries).shape[0], np.asarray(keys).shape[0]
    return {"selection": topk_tokens(scores, k), "scores": scores,
            "ledger": (("token_scan", "token", H * L),)}


def _route(keys, queries, gates, block_size, h, kind, precision):
    """Router + ledger bookkeeping.  Restates ``routing.py:102-120``."""
    bounds, pooled = block_pool(keys, block_size)
    E = route_head_importance(queries, gates, pooled, kind, precision)
    heads = route_topk_heads(E, h)
    H = np.asarray(queries).shape[0]
    entries = (("router", "block", H * bounds.shape[0]),) if kind == BLOCK_ATTENTION else ()
    return heads, E, entries


def misa_select(keys, queries, gates, k, h, block_size, kind=BLOCK_ATTENTION, precision=REFERENCE64) -> dict:
    """Single-stage routed selection.  Restates ``routing.py:123-141`` (+ ``estimators.py:185-188``)."""
    H = np.asarray(queries).shape[0]
    heads, E, entries = _route(keys, queries, gates, block_size, min(h, H), kind, precision)
    scores = misa_score(keys, queries, gates, heads, precision)
    L = np.asarray(keys).shape[0]
    return {"selection": topk_tokens(scores, k), "heads": heads, "importance": E, "scores": scores,
            "ledger": entries + (("token_scan", "token", len(heads) * L),)}


def misa_hier_select(keys, queries, gates, k, h, block_size, kprime, kind=BLOCK_ATTENTION,
                     precision=REFERENCE64) -> dict:
    """Two-stage routed selection (MISA-dagger).  Restates ``routing.py:144-174`` and ``dsa.py:95-115``."""
    H = np.asarray(queries).shape[0]
    heads, E, entries = _route(keys, queries, gates, block_size, min(h, H), kind, precision)
    coarse = misa_score(keys, queries, gates, heads, precision)
    cand = topk_tokens(coarse, kprime)
    fine = gated_relu_scores(np.asarray(keys)[cand], queries, gates, precision)
    sel = topk_within(fine, cand, k)
    L = np.asarray(keys).shape[0]
    return {"selection": sel, "heads": heads, "importance": E, "candidates": cand,
            "scores": coarse, "refine_scores": fine,
            "ledger": entries + (("token_scan", "token", len(heads) * L),
                                 ("refine", "refine", H * cand.shape[0]))}


# --------------------------------------------------- batched causal driver --
def row_select(method: str, K, Q, W, n: int, t: int, *, k: int, h: int = 8, block_size: int = 1024,
               kprime: int = 8192, kind: str = BLOCK_ATTENTION, precision: str = FAST32) -> dict:
    """Row t of a batched call == the reference on ``IndexerWorkload(K[:n], Q[t], W[t])``.

    This is exactly ``IndexerWorkload.truncated(n)`` semantics (``workload.py:91-110``) with the
    SPEC prefix convention that the query's own token is in the prefix (``SPEC.md:79``).
    """
    keys, queries, gates = K[:n], Q[t], W[t]
    if method == "dsa":
        return dsa_select(keys, queries, gates, k, precision)
    if method == "misa":
        return misa_select(keys, queries, gates, k, h, block_size, kind, precision)
    if method == "misa_hier":
        return misa_hier_select(keys, queries, gates, k, h, block_size, max(kprime, k), kind, precision)
    raise ValueError(f"unknown method {method!r}")


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (exactly representable)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    u = ((u + rounding) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def softmax_rows(x: np.ndarray) -> np.ndarray:
    """Row-wise stable softmax, as ``workload.py:113-117`` applied per query row."""
    z = x - x.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def synthetic_prefill(seed: int, L: int, H: int, d: int, T: int | None = None, *, raw_gates: bool = False):
    """Batched synthetic inputs: K ~ N(0,1) (L,d), Q ~ N(0,1) (T,H,d),
    W = softmax over heads of N(0,1) per row (``workload.py:135-139``); K and Q bf16-rounded.
    Returned as float64 arrays holding bf16-exact (K, Q) and f32-exact (W) values."""
    T = L if T is None else T
    rng = np.random.default_rng(seed)
    K = bf16_round(rng.standard_normal((L, d), dtype=np.float32))
    Q = bf16_round(rng.standard_normal((T, H, d), dtype=np.float32))
    g = rng.standard_normal((T, H), dtype=np.float32).astype(np.float64)
    W = g if raw_gates else softmax_rows(g)
    W = W.astype(np.float32).astype(np.float64)
    return K, Q, W


def needle_workload(seed: int, L: int, depth_fraction: float, needle_len: int, margin: float,
                    H: int, d: int, *, noise_scale: float = 0.01, align_head: int | None = None,
                    raw_gates: bool = False):
    """Planted-needle single-query workload.  Restates ``workload.py:143-199`` (same RNG order,
    so it is bit-identical to the reference generator).  Returns (keys, queries, gates, (start, len, head))."""
    rng = np.random.default_rng(seed)
    keys = rng.standard_normal((L, d))
    queries = rng.standard_normal((H, d))
    gates = rng.standard_normal(H)
    if not raw_gates:
        z = gates - gates.max()
        e = np.exp(z)
        gates = e / e.sum()
    target = int(np.argmax(gates)) if align_head is None else int(align_head)
    start = int(np.floor(depth_fraction * (L - needle_len)))
    direction = queries[target] / np.linalg.norm(queries[target])
    noise = noise_scale * rng.standard_normal((needle_len, d))
    keys[start:start + needle_len] = margin * direction + noise
    return keys, queries, gates, (start, needle_len, target)
