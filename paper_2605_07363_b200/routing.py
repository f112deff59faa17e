"""Head routing and the routed selectors, single-query API (``routing.py:38-174``).

``route_head_importance`` runs the tcgen05 router (K2) for one query row;
``misa_select`` / ``misa_hier_select`` run the batched engine with T = 1 and
attach the reference's closed-form cost ledger (``SPEC.md:302``).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .config import BLOCK_ATTENTION, REFERENCE64, ROUTER_SCORE_KINDS, IndexerConfig, dtype_for, warn_if_rounded
from .dsa import _select_dense_row, device_scores
from .engine import prepare_inputs, shared_engine
from .pooling import BlockSummary
from .types import CostEntry, CostLedger, HeadSet, ScoreVector, SelectionResult, TokenSelection
from .validation import check_choice
from .workload import IndexerWorkload


def _check_router_inputs(workload: IndexerWorkload, summary: BlockSummary) -> None:
    if summary.prefix_len != workload.prefix_len:
        raise ValueError(f"summary covers {summary.prefix_len} keys but workload has {workload.prefix_len}")
    if summary.n_blocks and summary.pooled_keys.shape[1] != workload.head_dim:
        raise ValueError("summary key dimension does not match workload")


def _one(workload: IndexerWorkload):
    return (torch.tensor(workload.keys), torch.tensor(workload.queries)[None],
            torch.tensor(workload.gate_weights)[None], [workload.prefix_len])


def route_head_importance(workload: IndexerWorkload, summary: BlockSummary, kind: str = BLOCK_ATTENTION, *,
                          precision: str = REFERENCE64) -> ScoreVector:
    """Per-head importance: block_attention mean_b |w ReLU(q . kbar_b)|, gate_only w, query_norm ||q||."""
    check_choice(kind, ROUTER_SCORE_KINDS, "kind")
    dtype_for(precision)
    warn_if_rounded(workload, precision)
    if kind == BLOCK_ATTENTION:
        _check_router_inputs(workload, summary)
    eng = shared_engine("misa", active_heads_h=1, block_size=summary.block_size, router_score=kind)
    x = prepare_inputs(*_one(workload))
    _, _, imp = eng.route(x, need_importance=True)
    return ScoreVector(imp[0, : workload.n_heads].double().cpu().numpy(), "head")


def route_topk_heads(importance, h: int) -> HeadSet:
    """The min(h, H) most important heads, ties to the smaller index, ascending (``routing.py:67-75``)."""
    if h < 1:
        raise ValueError(f"h must be positive, got {h}")
    values = importance.values if isinstance(importance, ScoreVector) else np.asarray(importance)
    H = int(values.shape[0])
    return HeadSet(head_indices=_select_dense_row(values, min(h, H)), n_heads=H)


def misa_score(workload: IndexerWorkload, heads: HeadSet, *, precision: str = REFERENCE64) -> ScoreVector:
    """Per-token scores over the active heads only (``routing.py:78-99``)."""
    dtype_for(precision)
    warn_if_rounded(workload, precision)
    if len(heads) == 0:
        raise ValueError("head set must contain at least one active head")
    if heads.n_heads != workload.n_heads:
        raise ValueError(f"head set is over {heads.n_heads} heads but workload has {workload.n_heads}")
    if len(heads) > 128:
        return ScoreVector(device_scores(workload.keys, workload.queries[heads.head_indices],
                                         workload.gate_weights[heads.head_indices]), "token")
    return ScoreVector(device_scores(workload.keys, workload.queries, workload.gate_weights,
                                     heads.head_indices), "token")


def _ledger(workload, summary_blocks, n_heads_used, kind, refine=None):
    entries = ()
    if kind == BLOCK_ATTENTION:
        entries = (CostEntry("router", "block", workload.n_heads * summary_blocks),)
    entries += (CostEntry("token_scan", "token", n_heads_used * workload.prefix_len),)
    if refine is not None:
        entries += (CostEntry("refine", "refine", refine),)
    return CostLedger(entries)


def _run(workload, summary, cfg: IndexerConfig, kind, method):
    check_choice(kind, ROUTER_SCORE_KINDS, "kind")
    warn_if_rounded(workload, cfg.precision_mode)
    if kind == BLOCK_ATTENTION:
        _check_router_inputs(workload, summary)
    eng = shared_engine(method, budget_k=cfg.budget_k, active_heads_h=cfg.active_heads_h,
                        block_size=summary.block_size, candidate_kprime=cfg.candidate_kprime, router_score=kind)
    return eng.run(*_one(workload))


def misa_select(workload: IndexerWorkload, summary: BlockSummary, cfg: IndexerConfig,
                kind: str = BLOCK_ATTENTION) -> SelectionResult:
    """Single-stage routed selection (``routing.py:123-141``)."""
    res = _run(workload, summary, cfg, kind, "misa")
    heads = res.heads[0].cpu().numpy()
    hs = HeadSet(heads[heads >= 0].astype(np.int64), workload.n_heads)
    o = res.topk[0].cpu().numpy()
    sel = TokenSelection(o[o >= 0].astype(np.int64), cfg.budget_k, workload.prefix_len)
    return SelectionResult(selection=sel, ledger=_ledger(workload, summary.n_blocks, len(hs), kind), heads=hs)


def misa_hier_select(workload: IndexerWorkload, summary: BlockSummary, cfg: IndexerConfig,
                     kind: str = BLOCK_ATTENTION) -> SelectionResult:
    """Two-stage routed selection: routed top-k' candidates, all-head re-rank (``routing.py:144-174``)."""
    res = _run(workload, summary, cfg, kind, "misa_hier")
    heads = res.heads[0].cpu().numpy()
    hs = HeadSet(heads[heads >= 0].astype(np.int64), workload.n_heads)
    c = res.candidates[0].cpu().numpy()
    cand = TokenSelection(np.sort(c[c >= 0]).astype(np.int64), cfg.candidate_kprime, workload.prefix_len)
    o = res.topk[0].cpu().numpy()
    sel = TokenSelection(o[o >= 0].astype(np.int64), cfg.budget_k, workload.prefix_len)
    ledger = _ledger(workload, summary.n_blocks, len(hs), kind, refine=workload.n_heads * len(cand))
    return SelectionResult(selection=sel, ledger=ledger, heads=hs, candidates=cand)


__all__ = ["route_head_importance", "route_topk_heads", "misa_score", "misa_select", "misa_hier_select"]
