"""B200-native (sm_100a) MISA / DSA indexer.

Drop-in for the indexer path of the reference ``misa`` package: the same
estimators (``DSAIndexer``, ``MISAIndexer``, ``HierarchicalMISAIndexer``,
``INDEXER_REGISTRY``, ``make_indexer``), pure functions and result types, with
every score, pooling, routing and top-k computed by hand-written sm_100a CUDA
kernels behind the C ABI in ``include/misa_b200.h``.  There is no CPU
fallback: importing works anywhere, calling requires the built extension and
a CUDA device.  The batched performance path is ``IndexerEngine`` /
``estimator.select_batch``.
"""

from .config import (BASELINE_BLOCK_SIZE, BLOCK_ATTENTION, FAST32, GATE_ONLY, PRECISION_MODES, QUERY_NORM,
                     REFERENCE64, ROUTER_BLOCK_SIZE, ROUTER_SCORE_KINDS, IndexerConfig, PrecisionWarning, dtype_for)
from .types import CostEntry, CostLedger, HeadSet, ScoreVector, SelectionResult, TokenSelection
from .workload import (IndexerWorkload, NeedleLabel, gen_needle_workload, gen_random_workload, load_workload,
                       save_workload, softmax)
from .metrics import candidate_recall, cost_ratio, iou, needle_recall
from .engine import DecodeGraph, IndexerEngine, IndexerOutput, prepare_inputs
from .pooling import BlockSummary, PagedKeyCache, PooledKeyCache, build_block_summary, incremental_append
from .dsa import dsa_rescore, dsa_score, dsa_select, gated_relu_scores, relevance_dots, topk_tokens, topk_within
from .routing import misa_hier_select, misa_score, misa_select, route_head_importance, route_topk_heads
from .corpus import Corpus, read_header, save_corpus, select_corpus
from .sparse_attention import sparse_attention
from .projections import IndexerProjections, quantize_rows_fp8
from .estimators import (INDEXER_REGISTRY, METHODS, BaseTokenIndexer, DSAIndexer, HierarchicalMISAIndexer,
                         MISAIndexer, make_indexer)

__version__ = "0.1.0"

__all__ = [
    "Corpus", "sparse_attention", "IndexerProjections", "quantize_rows_fp8", "DecodeGraph", "PagedKeyCache", "PrecisionWarning", "read_header", "save_corpus", "select_corpus",
    "BASELINE_BLOCK_SIZE", "BLOCK_ATTENTION", "BaseTokenIndexer", "BlockSummary", "CostEntry", "CostLedger",
    "DSAIndexer", "FAST32", "GATE_ONLY", "HeadSet", "HierarchicalMISAIndexer", "INDEXER_REGISTRY", "IndexerConfig",
    "IndexerEngine", "IndexerOutput", "IndexerWorkload", "METHODS", "MISAIndexer", "NeedleLabel", "PRECISION_MODES",
    "PooledKeyCache", "QUERY_NORM", "REFERENCE64", "ROUTER_BLOCK_SIZE", "ROUTER_SCORE_KINDS", "ScoreVector",
    "SelectionResult", "TokenSelection", "build_block_summary", "candidate_recall", "cost_ratio", "dsa_rescore",
    "dsa_score", "dsa_select", "dtype_for", "gated_relu_scores", "gen_needle_workload", "gen_random_workload",
    "incremental_append", "iou", "load_workload", "make_indexer", "misa_hier_select", "misa_score", "misa_select",
    "needle_recall", "prepare_inputs", "relevance_dots", "route_head_importance", "route_topk_heads",
    "save_workload", "softmax", "topk_tokens", "topk_within",
]
