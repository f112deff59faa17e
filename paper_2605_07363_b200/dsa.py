"""Dense DSA indexer, single-query API (``dsa.py:18-132``) on the device.

Each function takes the reference's numpy-level arguments, runs the sm_100a
kernels (scores: tcgen05 scorer in materialize mode; top-k: radix selector)
and returns the reference's result types.  Operands are rounded to bf16 on
upload and dot products accumulate in f32 — the reference's ``fast32``
contract on bf16-representable inputs.  The batched path is ``engine``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .config import REFERENCE64, dtype_for, warn_if_rounded
from .engine import head_dim_pad, heads_pad, heads_per_query, prepare_inputs, shared_engine
from .types import CostEntry, CostLedger, ScoreVector, SelectionResult, TokenSelection
from .validation import check_positive_int
from .workload import IndexerWorkload


def _stream():
    return torch.cuda.current_stream().cuda_stream


def device_scores(keys, queries, gates, heads=None) -> np.ndarray:
    """sum_j w_j ReLU(q_j . k_s) over the given query rows (all of them, or the `heads` subset)."""
    keys = np.asarray(keys, dtype=np.float64)
    queries = np.asarray(queries, dtype=np.float64)
    gates = np.asarray(gates, dtype=np.float64)
    x = prepare_inputs(torch.tensor(keys), torch.tensor(queries)[None], torch.tensor(gates)[None],
                       [keys.shape[0]])
    L = x.L
    if heads is None:
        hq, hd = x.Hp, None
    else:
        heads = np.asarray(heads, dtype=np.int64)
        hq = heads_per_query(max(1, heads.shape[0]))
        row = np.full(hq, -1, np.int32)
        row[: heads.shape[0]] = heads
        hd = torch.from_numpy(row[None]).cuda()
    out = torch.empty(1, L, dtype=torch.float32, device="cuda")
    items = torch.zeros(1, dtype=torch.int32, device="cuda")
    tiles = torch.full((1,), (L + 127) // 128, dtype=torch.int32, device="cuda")
    _lib.call("misa_score_materialize", x.keys.data_ptr(), L, 1, x.D, x.queries.data_ptr(), x.weights.data_ptr(),
              x.H, x.Hp, None if hd is None else hd.data_ptr(), hq, x.prefix.data_ptr(), 1, items.data_ptr(),
              tiles.data_ptr(), 1, out.data_ptr(), L, _stream())
    return out[0].double().cpu().numpy()


def relevance_dots(keys, queries, dtype=np.float32) -> np.ndarray:
    """(N, R) query-key dots on bf16 operands with f32 accumulation (``dsa.py:18-34``).

    ``misa_relevance_dots``: the tcgen05 contraction of the refine kernel over contiguous key
    tiles, 128 query rows per launch, the raw accumulator stored."""
    keys = np.asarray(keys, dtype=np.float64)
    queries = np.asarray(queries, dtype=np.float64)
    if keys.ndim != 2 or queries.ndim != 2 or keys.shape[1] != queries.shape[1]:
        raise ValueError("keys must be (R, d) and queries (N, d) with the same d")
    R, d = keys.shape
    N = queries.shape[0]
    if R == 0 or N == 0:
        return np.zeros((N, R))
    D = head_dim_pad(d)
    K = torch.zeros(R, D, dtype=torch.bfloat16, device="cuda")
    K[:, :d] = torch.from_numpy(keys).cuda().to(torch.bfloat16)
    out = np.empty((N, R))
    for a in range(0, N, 128):
        n = min(128, N - a)
        npad = heads_pad(n)
        Qc = torch.zeros(npad, D, dtype=torch.bfloat16, device="cuda")
        Qc[:n, :d] = torch.from_numpy(queries[a:a + n]).cuda().to(torch.bfloat16)
        o = torch.empty(R, n, dtype=torch.float32, device="cuda")
        _lib.call("misa_relevance_dots", K.data_ptr(), R, D, Qc.data_ptr(), n, npad, o.data_ptr(), n, _stream())
        out[a:a + n] = o.double().cpu().numpy().T
    return out


def gated_relu_scores(keys, queries, gate_weights, dtype=np.float32) -> np.ndarray:
    """Sum over heads of gate * ReLU(query . key) per key row (``dsa.py:37-53``)."""
    return device_scores(keys, queries, gate_weights)


def dsa_score(workload: IndexerWorkload, *, precision: str = REFERENCE64) -> ScoreVector:
    dtype_for(precision)
    warn_if_rounded(workload, precision)
    return ScoreVector(device_scores(workload.keys, workload.queries, workload.gate_weights), "token")


def _select_dense_row(values: np.ndarray, k: int, idx: np.ndarray | None = None) -> np.ndarray:
    """Top-min(k, n) of one score row on the device; ties -> smaller position (the stable
    argsort of ``dsa.py:74,90``); returns the positions, or ``idx`` at those positions,
    ascending.

    The register selector orders f32 keys.  Float64 scores that f32 does not represent
    exactly are resolved exactly: f32 rounding is monotone, so every score whose f32 value
    exceeds the k-th largest f32 value is selected and every one below it is not; only the
    scores tied with it in f32 are re-ranked by their f64 values."""
    v64 = np.ascontiguousarray(values, dtype=np.float64)
    n = v64.shape[0]
    if n == 0:
        return np.empty(0, np.int64)
    vals = torch.as_tensor(v64.astype(np.float32), device="cuda")[None]
    lens = torch.tensor([n], dtype=torch.int32, device="cuda")
    out = torch.empty(1, k, dtype=torch.int32, device="cuda")
    _lib.call("misa_select_dense", vals.data_ptr(), n, None, n, lens.data_ptr(), None, 1, k, out.data_ptr(), k, None,
              _stream())
    sel = out[0]
    sel = sel[sel >= 0].long()
    if not np.array_equal(v64.astype(np.float32).astype(np.float64), v64):
        v32 = vals[0]
        thr = v32[sel].min()
        above = torch.nonzero(v32 > thr).flatten()
        tied = torch.nonzero(v32 == thr).flatten()
        need = int(sel.numel()) - int(above.numel())
        if need < tied.numel():
            vd = torch.as_tensor(v64, device="cuda")
            tied = tied[torch.sort(vd[tied], descending=True, stable=True).indices[:need]]
        sel = torch.sort(torch.cat([above, tied])).values
    if idx is not None:
        sel = torch.sort(torch.as_tensor(np.asarray(idx, dtype=np.int64), device="cuda")[sel]).values
    return sel.cpu().numpy().astype(np.int64)


def topk_tokens(scores, k: int) -> TokenSelection:
    """The min(k, L) highest scores, ties to the smaller index, ascending (``dsa.py:64-76``)."""
    check_positive_int(k, "k")
    values = scores.values if isinstance(scores, ScoreVector) else np.asarray(scores)
    L = int(values.shape[0])
    return TokenSelection(indices=_select_dense_row(values, k), budget=k, prefix_len=L)


def topk_within(scores, candidates, k: int, prefix_len: int) -> TokenSelection:
    """Top-k inside an ascending candidate set, ties to the smaller token index (``dsa.py:79-92``)."""
    check_positive_int(k, "k")
    cand = np.asarray(candidates, dtype=np.int64)
    return TokenSelection(indices=_select_dense_row(np.asarray(scores), k, cand), budget=k, prefix_len=prefix_len)


def dsa_rescore(workload: IndexerWorkload, candidates, k: int, *, precision: str = REFERENCE64):
    """All-head re-score of a candidate set + top-k (``dsa.py:95-115``) via the gather kernel."""
    dtype_for(precision)
    warn_if_rounded(workload, precision)
    cand = np.asarray(candidates, dtype=np.int64)
    x = prepare_inputs(torch.tensor(workload.keys), torch.tensor(workload.queries)[None],
                       torch.tensor(workload.gate_weights)[None], [workload.prefix_len])
    n = cand.shape[0]
    if n == 0:
        return TokenSelection(np.empty(0, np.int64), k, workload.prefix_len), 0
    c = torch.from_numpy(cand.astype(np.int32)).cuda()[None].contiguous()
    ncand = torch.tensor([n], dtype=torch.int32, device="cuda")
    rows = torch.zeros(1, dtype=torch.int32, device="cuda")
    rs = torch.empty(1, n, dtype=torch.float32, device="cuda")
    _lib.call("misa_refine_scores", x.keys.data_ptr(), x.L, x.D, x.queries.data_ptr(), x.weights.data_ptr(), x.H,
              x.Hp, c.data_ptr(), n, ncand.data_ptr(), rows.data_ptr(), 1, 1, None, rs.data_ptr(), n, _stream())
    out = torch.empty(1, k, dtype=torch.int32, device="cuda")
    _lib.call("misa_select_dense", rs.data_ptr(), n, c.data_ptr(), n, ncand.data_ptr(), None, 1, k, out.data_ptr(), k,
              None, _stream())
    o = out[0].cpu().numpy()
    sel = TokenSelection(o[o >= 0].astype(np.int64), k, workload.prefix_len)
    return sel, workload.n_heads * n


def dsa_select(workload: IndexerWorkload, k: int, *, precision: str = REFERENCE64) -> SelectionResult:
    """Dense selection: all heads score all prefix tokens, top-k (``dsa.py:118-132``)."""
    check_positive_int(k, "k")
    dtype_for(precision)
    warn_if_rounded(workload, precision)
    eng = shared_engine("dsa", budget_k=k)
    res = eng.run(torch.tensor(workload.keys), torch.tensor(workload.queries)[None],
                  torch.tensor(workload.gate_weights)[None], [workload.prefix_len])
    o = res.topk[0].cpu().numpy()
    sel = TokenSelection(o[o >= 0].astype(np.int64), k, workload.prefix_len)
    ledger = CostLedger((CostEntry("token_scan", "token", workload.n_heads * workload.prefix_len),))
    return SelectionResult(selection=sel, ledger=ledger)


__all__ = ["device_scores", "relevance_dots", "gated_relu_scores", "dsa_score", "topk_tokens", "topk_within",
           "dsa_rescore", "dsa_select", "head_dim_pad", "heads_pad"]
