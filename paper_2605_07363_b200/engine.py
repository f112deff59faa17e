"""Batched device engine: the performance path of the indexer.

One call scores T query rows against a key cache on the GPU and returns the
top-k token indices per row (ascending, -1 padded), the routed heads and,
optionally, the router importances.  Row t is exactly the reference run on
``IndexerWorkload(keys=K[:n_t], queries=Q[t], gate_weights=W[t])``
(``workload.py:91-110``); the default ``prefix_len`` is causal prefill,
n_t = L - T + t + 1 (``SPEC.md:79``: the query's own token is in the prefix).

Pipeline per method (all kernels in ``csrc/``; every launch goes through the
C ABI in ``include/misa_b200.h``):

  dsa        score_materialize(sampled keys) -> select_threshold -> score_filter
             (all H heads) -> select_topk                      (dsa.py:56-76,118-132)
  misa       pool_keys -> route_scores -> route_select -> the same selector with
             the h routed heads                                 (routing.py:102-141)
  misa_hier  misa with k' -> refine_scores (all heads on the k' candidates)
             -> select_dense within candidates                  (routing.py:144-174)

The fused selector is exact: tau_t is the j-th largest score on a 1/stride key
sample (j = ceil(beta*k*m/n)), every key with score >= tau_t is kept as a
candidate, and when the candidate count is >= min(k, n_t) the exact top-k
(score desc, index asc) provably lies among them.  Rows whose sample threshold
was too high (underflow) or whose candidates overflow the buffer are re-done
densely, so the result never depends on the estimate.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import BLOCK_ATTENTION, ROUTER_KIND_CODE, ROUTER_SCORE_KINDS
from .validation import check_choice, check_positive_int

METHODS = ("dsa", "misa", "misa_hier")
V5_CAPS = (512, 1024, 1536, 2048, 3072, 4096)  # per-quadrant capacities of select.cu launch_topk5


def _ptr(t):
    return None if t is None else t.data_ptr()


def _pow2(x: int) -> int:
    return 1 << max(0, (int(x) - 1).bit_length())


def head_dim_pad(d: int) -> int:
    if d <= 64:
        return 64
    if d <= 128:
        return 128
    raise ValueError(f"head_dim {d} > 128 is not supported by the sm_100a kernels")


def heads_pad(H: int) -> int:
    if H > 128:
        raise ValueError(f"n_heads {H} > 128 is not supported by the sm_100a kernels")
    return max(8, _pow2(H))


def heads_per_query(h: int) -> int:
    return max(8, _pow2(h))


@dataclass
class IndexerOutput:
    topk: torch.Tensor                  # (T, k) int32, ascending, -1 padded
    heads: torch.Tensor | None = None   # (T, h) int32 ascending (misa / misa_hier)
    importance: torch.Tensor | None = None  # (T, H) f32 router importance
    candidates: torch.Tensor | None = None  # (T, k') int32 coarse candidates (misa_hier), -1 padded
    n_fallback_rows: int = 0
    # (T, 4) int32: when set, row t of `candidates` is 4 consecutive ascending runs of these
    # lengths (the coarse selector's unordered output); None: each row is ascending
    candidate_runs: torch.Tensor | None = None

    def sorted_candidates(self) -> torch.Tensor | None:
        """The coarse candidates ascending per row (-1 padding last), as ``topk_tokens``
        returns them (``routing.py:157-159``)."""
        if self.candidates is None or self.candidate_runs is None:
            return self.candidates
        c = self.candidates.long()
        c = torch.where(c < 0, torch.iinfo(torch.int64).max, c)
        c = torch.sort(c, dim=1).values
        return torch.where(c == torch.iinfo(torch.int64).max, -1, c).to(torch.int32)


@dataclass
class SeqLayout:
    """Several independent key sequences packed in one key buffer, each starting at a
    multiple of ``align`` key rows (``align`` is a multiple of the pooling block and of
    the 128-key tile): row t's keys are key rows key0[t] .. key0[t] + n_t - 1, and the
    indices it returns are relative to its own sequence.  Rows of one sequence are
    consecutive.  This batches the reference's independent workloads
    (``IndexerWorkload`` per query, ``workload.py:40-110``) into one device call."""

    key0: torch.Tensor        # (T,) int32 device
    key0_host: np.ndarray     # (T,) int64
    align: int
    block: int                # pooling block the alignment was made for (router)

    def rows(self, a: int, b: int) -> "SeqLayout":
        return SeqLayout(self.key0[a:b], self.key0_host[a:b], self.align, self.block)

    @property
    def boff(self) -> torch.Tensor:
        return torch.div(self.key0, self.block, rounding_mode="floor").to(torch.int32)


@dataclass
class PreparedInputs:
    keys: torch.Tensor      # (L, D) bf16
    queries: torch.Tensor   # (T, Hp, D) bf16
    weights: torch.Tensor   # (T, Hp) f32
    prefix: torch.Tensor    # (T,) int32 device
    prefix_host: np.ndarray  # (T,) int64
    L: int
    T: int
    H: int
    Hp: int
    d: int
    D: int
    causal_key: tuple | None
    pages: tuple | None = None  # paged key cache: (page_table (n_pages,) int32 device, page_size)
    seq: SeqLayout | None = None  # several key sequences (L = the longest one)

    def rows(self, a: int, b: int) -> "PreparedInputs":
        """Rows [a, b) against the same key set (views, no copies)."""
        ck = None if self.causal_key is None else self.causal_key + ("rows", a, b)
        return PreparedInputs(self.keys, self.queries[a:b], self.weights[a:b], self.prefix[a:b],
                              self.prefix_host[a:b], self.L, b - a, self.H, self.Hp, self.d, self.D, ck, self.pages,
                              None if self.seq is None else self.seq.rows(a, b))

    @property
    def n_keys(self) -> int:
        """Key rows of the key buffer (all sequences, with alignment padding)."""
        return int(self.keys.shape[0]) if self.seq is not None else self.L

    def list_key(self):
        """Cache key of the host work lists derived from the row lengths (and sequences)."""
        if self.causal_key is not None:
            return self.causal_key
        return self.prefix_host.tobytes() + (b"" if self.seq is None else self.seq.key0_host.tobytes())


def prepare_inputs(keys, queries, weights, prefix_len=None, device=None, prefix_dev=None) -> PreparedInputs:
    """Move/convert/pad inputs to the kernel layouts (no copy when already conforming).

    ``prefix_dev``: the prefix lengths already on the device (int32, same values as
    ``prefix_len``), so that no host->device copy is issued here."""
    dev = torch.device(device) if device is not None else (
        keys.device if isinstance(keys, torch.Tensor) and keys.is_cuda else torch.device("cuda"))
    K = torch.as_tensor(keys, device=dev)
    Q = torch.as_tensor(queries, device=dev)
    W = torch.as_tensor(weights, device=dev)
    if K.ndim != 2 or Q.ndim != 3 or W.ndim != 2:
        raise ValueError("keys must be (L, d), queries (T, H, d), weights (T, H)")
    L, d = K.shape
    T, H, dq = Q.shape
    if dq != d:
        raise ValueError(f"queries have dim {dq} but keys have dim {d}")
    if tuple(W.shape) != (T, H):
        raise ValueError(f"weights must be ({T}, {H}), got {tuple(W.shape)}")
    if L < 1 or T < 1:
        raise ValueError("need at least one key and one query row")
    D, Hp = head_dim_pad(d), heads_pad(H)
    K = K.to(torch.bfloat16)
    if d != D:
        K = torch.nn.functional.pad(K, (0, D - d))
    K = K.contiguous()
    Q = Q.to(torch.bfloat16)
    if d != D or H != Hp:
        Q = torch.nn.functional.pad(Q, (0, D - d, 0, Hp - H))
    Q = Q.contiguous()
    W = W.to(torch.float32)
    if H != Hp:
        W = torch.nn.functional.pad(W, (0, Hp - H))
    W = W.contiguous()
    causal_key = None
    if prefix_len is None:
        if T > L:
            raise ValueError(f"causal prefill needs T <= L, got T={T}, L={L}")
        host = np.arange(L - T + 1, L + 1, dtype=np.int64)
        causal_key = (L, T)
    else:
        host = np.asarray(prefix_len.cpu() if isinstance(prefix_len, torch.Tensor) else prefix_len,
                          dtype=np.int64).reshape(-1)
        if host.shape[0] != T:
            raise ValueError(f"prefix_len must have {T} entries")
        if host.min() < 1 or host.max() > L:
            raise ValueError("prefix lengths must lie in [1, L]")
    if prefix_dev is not None:
        if tuple(prefix_dev.shape) != (T,) or prefix_dev.dtype != torch.int32 or prefix_dev.device != K.device:
            raise ValueError("prefix_dev must be a (T,) int32 tensor on the keys' device")
        prefix = prefix_dev
    else:
        prefix = torch.from_numpy(host.astype(np.int32)).to(dev)
    return PreparedInputs(K, Q, W, prefix, host, L, T, H, Hp, d, D, causal_key)


def paged_inputs(cache, queries, weights, prefix_len=None) -> PreparedInputs:
    """Decode inputs over a ``PagedKeyCache``: keys stay in the page pool (the scorer
    translates logical tiles through the page table); every row sees the whole cache."""
    dev = cache.pool_keys.device
    Q = torch.as_tensor(queries, device=dev)
    W = torch.as_tensor(weights, device=dev)
    if Q.ndim != 3 or W.ndim != 2 or tuple(W.shape) != tuple(Q.shape[:2]):
        raise ValueError("queries must be (T, H, d) and weights (T, H)")
    T, H, d = Q.shape
    if d != cache.d:
        raise ValueError(f"queries have dim {d}, the cache holds dim {cache.d}")
    D, Hp, L = cache.D, heads_pad(H), cache.length
    if L < 1:
        raise ValueError("empty cache")
    Q = Q.to(torch.bfloat16)
    if d != D or H != Hp:
        Q = torch.nn.functional.pad(Q, (0, D - d, 0, Hp - H))
    W = W.to(torch.float32)
    if H != Hp:
        W = torch.nn.functional.pad(W, (0, Hp - H))
    host = np.full(T, L, dtype=np.int64) if prefix_len is None else np.asarray(
        prefix_len.cpu() if isinstance(prefix_len, torch.Tensor) else prefix_len, dtype=np.int64).reshape(-1)
    if host.shape[0] != T or np.any(host != L):
        raise ValueError("paged decode scores every row against the whole cache (prefix_len == cache.length)")
    prefix = torch.from_numpy(host.astype(np.int32)).to(dev)
    return PreparedInputs(cache.pool_keys, Q.contiguous(), W.contiguous(), prefix, host, L, T, H, Hp, d, D,
                          ("paged", L, T), pages=(cache.page_table, cache.B))


def prepare_varlen(keys, cu_seqlens_k, queries, weights, cu_seqlens_q, prefix_len=None, *, block_size: int = 1024,
                   device=None) -> PreparedInputs:
    """Inputs of several independent sequences for one batched call.

    ``keys``: (sum L_s, d) packed keys with ``cu_seqlens_k`` (S+1,) offsets; ``queries`` /
    ``weights``: (sum T_s, H, d) / (sum T_s, H) rows of every sequence, consecutive, with
    ``cu_seqlens_q`` (S+1,).  Row i of sequence s sees the first n keys of s: ``prefix_len``
    per row, default causal within the sequence (n = L_s - T_s + i + 1).  A corpus of
    single-query workloads is S sequences of T_s = 1 row with n = L_s.  The keys are copied
    once into a buffer where every sequence starts at a multiple of lcm(block, 128) rows."""
    ck = np.asarray(cu_seqlens_k.cpu() if isinstance(cu_seqlens_k, torch.Tensor) else cu_seqlens_k, np.int64)
    cq = np.asarray(cu_seqlens_q.cpu() if isinstance(cu_seqlens_q, torch.Tensor) else cu_seqlens_q, np.int64)
    if ck.ndim != 1 or cq.shape != ck.shape or ck.shape[0] < 2 or ck[0] != 0 or cq[0] != 0:
        raise ValueError("cu_seqlens_k / cu_seqlens_q must be (S+1,) offsets starting at 0")
    lk, lq = np.diff(ck), np.diff(cq)
    if np.any(lk < 1) or np.any(lq < 0):
        raise ValueError("every sequence needs >= 1 key and >= 0 query rows")
    dev = torch.device(device) if device is not None else (
        keys.device if isinstance(keys, torch.Tensor) and keys.is_cuda else torch.device("cuda"))
    K = torch.as_tensor(keys, device=dev)
    if K.ndim != 2 or K.shape[0] != ck[-1]:
        raise ValueError(f"keys must be ({ck[-1]}, d)")
    T = int(cq[-1])
    if T < 1:
        raise ValueError("need at least one query row")
    seq_of_row = np.repeat(np.arange(lk.shape[0]), lq)
    pos = np.arange(T) - cq[:-1][seq_of_row]
    if prefix_len is None:
        if np.any(lq > lk):
            raise ValueError("causal prefill needs T_s <= L_s for every sequence")
        host = (lk - lq)[seq_of_row] + pos + 1
    else:
        host = np.asarray(prefix_len.cpu() if isinstance(prefix_len, torch.Tensor) else prefix_len,
                          np.int64).reshape(-1)
        if host.shape[0] != T:
            raise ValueError(f"prefix_len must have {T} entries")
        if np.any(host < 1) or np.any(host > lk[seq_of_row]):
            raise ValueError("prefix lengths must lie in [1, L_s] of each row's sequence")
    align = math.lcm(int(block_size), 128)
    padded = -(-lk // align) * align
    off = np.concatenate([[0], np.cumsum(padded)[:-1]])
    x = prepare_inputs(torch.zeros(1, K.shape[1], dtype=K.dtype, device=dev), queries, weights, [1] * T,
                       device=dev)
    Kp = torch.zeros(int(padded.sum()), x.D, dtype=torch.bfloat16, device=dev)
    dst = torch.from_numpy(np.concatenate([np.arange(o, o + n) for o, n in zip(off, lk)])).to(dev)
    Kp[dst, : K.shape[1]] = K.to(torch.bfloat16)
    key0 = off[seq_of_row]
    prefix = torch.from_numpy(host.astype(np.int32)).to(dev)
    seq = SeqLayout(torch.from_numpy(key0.astype(np.int32)).to(dev), key0, align, int(block_size))
    return PreparedInputs(Kp, x.queries, x.weights, prefix, host, int(lk.max()), T, x.H, x.Hp, x.d, x.D, None,
                          None, seq)


def varlen_groups(lens: np.ndarray, key0: np.ndarray, G: int, stride: int, min_len: int):
    """Work items of a several-sequence call: runs of rows with the same key offset split into
    groups of <= G rows; (row0, nrows, key0 / stride, tiles) for groups with a row longer
    than min_len, longest first."""
    T = lens.shape[0]
    if np.any(key0 % stride):
        raise ValueError(f"sequence offsets must be multiples of the sample stride {stride}")
    run_start = np.r_[True, key0[1:] != key0[:-1]]
    run_id = np.cumsum(run_start) - 1
    pos = np.arange(T) - np.flatnonzero(run_start)[run_id]
    grp = pos // G
    g_start = np.flatnonzero(np.r_[True, (run_id[1:] != run_id[:-1]) | (grp[1:] != grp[:-1])])
    nrows = np.diff(np.r_[g_start, T])
    gmax = np.maximum.reduceat(lens, g_start)
    keep = np.nonzero(gmax > min_len)[0]
    tiles = ((gmax[keep] + stride - 1) // stride + 127) // 128
    order = np.argsort(-tiles, kind="stable")
    sel = keep[order]
    return (g_start[sel].astype(np.int32), nrows[sel].astype(np.int32), (key0[g_start[sel]] // stride).astype(np.int32),
            tiles[order].astype(np.int32))


class IndexerEngine:
    """Device indexer for one method/config; caches work lists and workspace per shape."""

    def __init__(self, method: str = "misa", *, budget_k: int = 2048, active_heads_h: int = 8,
                 block_size: int = 1024, candidate_kprime: int = 8192, router_score: str = BLOCK_ATTENTION,
                 sample_stride: int = 32, beta: float | None = None, workspace_bytes: int = 32 << 30,
                 check_overflow: bool = True):
        check_choice(method, METHODS, "method")
        self.method = method
        self.k = check_positive_int(budget_k, "budget_k")
        self.h = check_positive_int(active_heads_h, "active_heads_h")
        self.B = check_positive_int(block_size, "block_size")
        self.kprime = check_positive_int(candidate_kprime, "candidate_kprime")
        if method == "misa_hier" and self.kprime < self.k:
            raise ValueError(f"candidate_kprime ({self.kprime}) must be >= budget_k ({self.k})")
        self.router_score = check_choice(router_score, ROUTER_SCORE_KINDS, "router_score")
        self.stride = check_positive_int(sample_stride, "sample_stride")
        self.beta = beta
        self.workspace_bytes = workspace_bytes
        self.check_overflow = check_overflow
        self._ws: dict = {}
        self._lists: dict = {}
        self.last_fallback_rows = 0
        # decode steps with at least this many rows and keys score through the fused filter (no
        # T x L score rows in HBM); others take the materialised key-split path.  Measured on a
        # B200 (graph replay, no flag check): 1M keys x 64 rows 0.26 vs 0.31 ms, but 128K x 64
        # 0.135 vs 0.092 and 1M x 16 0.17 vs 0.14 — the sample / tau / select / sort chain costs
        # more than the score rows it saves below that size
        self.decode_filter_min_rows = 32
        self.decode_filter_min_keys = 1 << 19
        self.last_decode_flags = None  # (T,) flags of the last fused-filter decode step (None: dense path)
        self.stage_events: list | None = None  # set to [] to record (stage, cuda event) pairs
        _lib.load()

    def _mark(self, name: str) -> None:
        if self.stage_events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.stage_events.append((name, ev))

    # ----------------------------------------------------------- workspace
    def _buf(self, name, shape, dtype, device):
        n = int(np.prod(shape))
        cur = self._ws.get(name)
        if cur is None or cur.numel() < n or cur.dtype != dtype or cur.device != device:
            cur = torch.empty(max(n, 1), dtype=dtype, device=device)
            self._ws[name] = cur
        return cur[:n].view(*shape)

    def _cached(self, key, fn):
        v = self._lists.get(key)
        if v is None:
            v = fn()
            if len(self._lists) > 64:
                self._lists.clear()
            self._lists[key] = v
        return v

    @staticmethod
    def _stream():
        return torch.cuda.current_stream().cuda_stream

    # ----------------------------------------------------------- work lists
    @staticmethod
    def group_items(lens: np.ndarray, G: int, stride: int, min_len: int) -> tuple[np.ndarray, np.ndarray]:
        """Groups of G rows (group id, 128-key tiles) with some row longer than min_len, longest first."""
        T = lens.shape[0]
        ng = (T + G - 1) // G
        pad = np.zeros(ng * G, dtype=np.int64)
        pad[:T] = lens
        mx = pad.reshape(ng, G).max(1)
        keep = np.nonzero(mx > min_len)[0]
        tiles = ((mx[keep] + stride - 1) // stride + 127) // 128
        order = np.argsort(-tiles, kind="stable")
        return keep[order].astype(np.int32), tiles[order].astype(np.int32)

    def _route_items(self, lens: np.ndarray, Hp: int, n_chunks: int):
        T = lens.shape[0]
        rpt = 128 // Hp
        ntiles = (T * Hp + 127) // 128
        pad = np.zeros(ntiles * rpt, dtype=np.int64)
        pad[:T] = lens // self.B
        nf = pad.reshape(ntiles, rpt).max(1)
        tl, ch, cols = [], [], []
        for c in range(n_chunks):
            cc = np.clip(nf - 128 * c, 0, 128)
            cc = (cc + 15) // 16 * 16
            sel = np.arange(ntiles) if c == 0 else np.nonzero(cc > 0)[0]
            order = sel[np.argsort(-cc[sel], kind="stable")]
            tl.append(order)
            ch.append(np.full(order.shape[0], c))
            cols.append(cc[order])
        return tuple(np.concatenate(x).astype(np.int32) for x in (tl, ch, cols))

    def _route_items_varlen(self, lens: np.ndarray, boff: np.ndarray, Hp: int):
        """Router items of a several-sequence call: one item per (tile, sequence in the tile,
        chunk), the chunk counted from the sequence's first pooled block; every (tile,
        sequence) pair has a chunk-0 item (the partial block)."""
        T = lens.shape[0]
        rpt = 128 // Hp
        tile = np.arange(T) // rpt
        nf = lens // self.B
        # (tile, boff) pairs with the largest full-block count of their rows
        start = np.flatnonzero(np.r_[True, (tile[1:] != tile[:-1]) | (boff[1:] != boff[:-1])])
        p_tile, p_boff = tile[start], boff[start]
        p_nf = np.maximum.reduceat(nf, start)
        nch = np.maximum(1, (p_nf + 127) // 128)
        rep = np.repeat(np.arange(start.shape[0]), nch)
        chunk = np.arange(rep.shape[0]) - np.repeat(np.cumsum(nch) - nch, nch)
        cols = np.clip(p_nf[rep] - 128 * chunk, 0, 128)
        cols = (cols + 15) // 16 * 16
        order = np.lexsort((-cols, p_boff[rep], chunk))  # chunk-major, then sequence
        return tuple(a[order].astype(np.int32) for a in (p_tile[rep], chunk, cols, p_boff[rep]))

    def _dev_list(self, key, fn, device):
        def make():
            arrs = fn()
            return tuple(torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in arrs)
        return self._cached(key, make)

    # ----------------------------------------------------------- stages
    def selector_params(self, k: int, L: int) -> tuple[int, float, int]:
        """(sample stride, beta, per-quadrant candidate capacity) of the fused top-k.

        tau is the j-th largest score on a 1/stride key sample, j = beta*k/stride, so about
        beta*k keys pass; its relative spread is ~1/sqrt(j).  Capacity is (1 + 5.5/sqrt(j))x
        the expected per-quadrant count (5.5 sigma: 1.49x at j = 128, the C4 shape; 1.69x at
        j = 64, where 1M-key rows sample every 64th key), and rows with n <= 4*cap keep
        every key.
        """
        if k < 4096:
            stride, beta = self.stride, (self.beta or 2.0)
        else:  # j >= 600 samples: a 4 % spread, so beta = 1.2 is still > 5 sigma from underflow
            stride, beta = max(1, self.stride // 2), (self.beta or 1.2)
        stride = max(stride, -(-L // 16384))  # <= 16384 samples per row bounds the (T, L/stride) sample buffer
        j = max(1.0, beta * k / stride)
        cap = int(math.ceil((1.0 + 5.5 / math.sqrt(j)) * beta * k / 4 / 32)) * 32
        # round up to a capacity the merge-free selector (select.cu topk5) is compiled for
        for c in V5_CAPS:
            if c >= cap:
                return stride, beta, c
        return stride, beta, cap

    def pool(self, x: PreparedInputs):
        """K1: in-block prefix sums + pooled planes."""
        nk = x.n_keys
        nf = nk // self.B
        n_chunks = max(1, (nf + 127) // 128)
        rows = n_chunks * 128
        P = self._buf("prefix", (nk, x.D), torch.float32, x.keys.device)
        planes = self._buf("planes", (3, rows, x.D), torch.bfloat16, x.keys.device)
        self._mark("pool")
        _lib.call("misa_pool_keys", _ptr(x.keys), nk, x.D, self.B, _ptr(P), None, _ptr(planes), rows, self._stream())
        if x.seq is not None:  # chunks of the router partials count from each row's first block
            n_chunks = max(1, (int(x.prefix_host.max()) // self.B + 127) // 128)
        return P, planes, n_chunks, rows

    def route(self, x: PreparedInputs, need_importance: bool = False, cache=None):
        """K2: heads (T, hq) int32 ascending, -1 padded; importance (T, Hp) f32 or None.

        With a ``PooledKeyCache`` the router reads its incrementally maintained prefix sums
        and pooled planes (``pooling.py:87-115``) instead of re-pooling the prefix."""
        h = min(self.h, x.H)
        hq = heads_per_query(h)
        dev = x.keys.device
        kind = ROUTER_KIND_CODE[self.router_score]
        heads = self._buf("heads", (x.T, hq), torch.int32, dev)
        imp = self._buf("importance", (x.T, x.Hp), torch.float32, dev) if need_importance else None
        partial, n_chunks = None, 1
        if self.router_score == BLOCK_ATTENTION:
            if cache is not None:
                if cache.B != self.B:
                    raise ValueError(f"cache block size {cache.B} != engine block_size {self.B}")
                # a paged cache hands out the address that maps its shared partial block
                P = cache.prefix_base(x.L) if getattr(cache, "paged", False) else cache.prefix
                planes, rows = cache.planes, cache.rows
                n_chunks = max(1, (x.L // self.B + 127) // 128)
            else:
                P, planes, n_chunks, rows = self.pool(x)
            key = ("route", x.list_key(), x.Hp, self.B, n_chunks)
            partial = self._buf("partial", (n_chunks, x.T, x.Hp), torch.float32, dev)
            if x.seq is None:
                it_tile, it_chunk, it_cols = self._dev_list(
                    key, lambda: self._route_items(x.prefix_host, x.Hp, n_chunks), dev)
                self._mark("route_scores")
                _lib.call("misa_route_scores", _ptr(x.queries), x.T, x.Hp, x.D, _ptr(planes), rows,
                          P if isinstance(P, int) else _ptr(P),
                          _ptr(x.prefix), self.B, _ptr(it_tile), _ptr(it_chunk), _ptr(it_cols), it_tile.numel(),
                          _ptr(partial), self._stream())
            else:
                if x.seq.block != self.B:
                    raise ValueError(f"sequences were aligned for block size {x.seq.block}, engine uses {self.B}")
                it_tile, it_chunk, it_cols, it_boff = self._dev_list(
                    key, lambda: self._route_items_varlen(x.prefix_host, x.seq.key0_host // self.B, x.Hp), dev)
                row_boff = x.seq.boff
                self._mark("route_scores")
                _lib.call("misa_route_scores_varlen", _ptr(x.queries), x.T, x.Hp, x.D, _ptr(planes), rows, _ptr(P),
                          _ptr(x.prefix), self.B, _ptr(it_tile), _ptr(it_chunk), _ptr(it_cols), _ptr(it_boff),
                          _ptr(row_boff), it_tile.numel(), _ptr(partial), self._stream())
        self._mark("route_select")
        _lib.call("misa_route_select", _ptr(partial), n_chunks, _ptr(x.weights), _ptr(x.queries), _ptr(x.prefix),
                  x.T, x.H, x.Hp, x.D, self.B, h, kind, _ptr(heads), hq, _ptr(imp), self._stream())
        return heads, hq, imp

    def select(self, x: PreparedInputs, heads: torch.Tensor | None, hq: int, k: int, out: torch.Tensor,
               tag: str = "sel", scores: torch.Tensor | None = None, runs: torch.Tensor | None = None) -> int:
        """Fused streaming top-k over the given head set (None = all heads). Returns #fallback rows.

        With ``scores`` (T, k) f32 the selected scores are returned too (aligned with ``out``)
        and short rows are scored rather than short-cut — what a key shard's local top-k needs.
        With ``runs`` (T, 4) int32 the rows are left unordered: 4 ascending runs of these
        lengths (``misa_select_topk_runs``)."""
        dev = x.keys.device
        stride, beta, cap = self.selector_params(k, x.L)
        append_all = 4 * cap
        G = 256 // hq
        stream = self._stream()
        ckey = x.list_key()
        min_len = 0 if scores is not None else k
        if x.seq is None:
            s_items, s_tiles = self._dev_list(("samp", ckey, G, stride, append_all),
                                              lambda: self.group_items(x.prefix_host, G, stride, append_all), dev)
            f_items, f_tiles = self._dev_list(("filt", ckey, G, min_len),
                                              lambda: self.group_items(x.prefix_host, G, 1, min_len), dev)
        else:
            s_items, s_rows, s_key0, s_tiles = self._dev_list(
                ("vsamp", ckey, G, stride, append_all),
                lambda: varlen_groups(x.prefix_host, x.seq.key0_host, G, stride, append_all), dev)
            f_items, f_rows, f_key0, f_tiles = self._dev_list(
                ("vfilt", ckey, G, min_len), lambda: varlen_groups(x.prefix_host, x.seq.key0_host, G, 1, min_len), dev)
        Ls = (x.L + stride - 1) // stride
        tau = self._buf(tag + "_tau", (x.T,), torch.float32, dev)
        if s_items.numel():
            samp = self._buf(tag + "_samp", (x.T, Ls), torch.float32, dev)
            self._mark(tag + ":sample")
            if x.seq is None:
                _lib.call("misa_score_materialize", _ptr(x.keys), x.L, stride, x.D, _ptr(x.queries),
                          _ptr(x.weights), x.H, x.Hp, _ptr(heads), hq, _ptr(x.prefix), x.T, _ptr(s_items),
                          _ptr(s_tiles), s_items.numel(), _ptr(samp), Ls, stream)
            else:
                _lib.call("misa_score_materialize_varlen", _ptr(x.keys), x.n_keys, stride, x.D, _ptr(x.queries),
                          _ptr(x.weights), x.H, x.Hp, _ptr(heads), hq, _ptr(x.prefix), x.T, _ptr(s_items),
                          _ptr(s_rows), _ptr(s_key0), _ptr(s_tiles), s_items.numel(), _ptr(samp), Ls, stream)
        else:
            samp = self._buf(tag + "_samp", (1, 1), torch.float32, dev)
        self._mark(tag + ":threshold")
        _lib.call("misa_select_threshold", _ptr(samp), Ls, _ptr(x.prefix), x.T, stride, k, float(beta),
                  append_all, _ptr(tau), stream)
        cand = self._buf(tag + "_cand", (x.T * 4 * cap,), torch.int64, dev)
        cnt = self._buf(tag + "_cnt", (x.T * 4,), torch.int32, dev)
        cnt.zero_()  # rows without a filter item (n <= k) keep defined counts (the selector prefetches them)
        if f_items.numel():
            self._mark(tag + ":filter")
            if x.seq is None:
                _lib.call("misa_score_filter", _ptr(x.keys), x.L, x.D, _ptr(x.queries), _ptr(x.weights), x.H, x.Hp,
                          _ptr(heads), hq, _ptr(x.prefix), x.T, _ptr(f_items), _ptr(f_tiles), f_items.numel(),
                          _ptr(tau), _ptr(cand), cap, _ptr(cnt), stream)
            else:
                _lib.call("misa_score_filter_varlen", _ptr(x.keys), x.n_keys, x.D, _ptr(x.queries), _ptr(x.weights),
                          x.H, x.Hp, _ptr(heads), hq, _ptr(x.prefix), x.T, _ptr(f_items), _ptr(f_rows), _ptr(f_key0),
                          _ptr(f_tiles), f_items.numel(), _ptr(tau), _ptr(cand), cap, _ptr(cnt), stream)
        flags = self._buf(tag + "_flags", (x.T,), torch.int32, dev)
        self.last_flags = flags
        self._mark(tag + ":select")
        if runs is not None and scores is None:
            _lib.call("misa_select_topk_runs", _ptr(cand), _ptr(cnt), cap, _ptr(x.prefix), x.T, k, x.L, _ptr(out),
                      out.stride(0), _ptr(runs), _ptr(flags), stream)
        else:
            runs = None
            _lib.call("misa_select_topk", _ptr(cand), _ptr(cnt), cap, _ptr(x.prefix), x.T, k, x.L, _ptr(out),
                      out.stride(0), _ptr(scores), _ptr(flags), stream)
        self._mark(tag + ":end")
        if not self.check_overflow:
            return 0
        # one reduction + one 4-byte read on the common (no flagged row) path; the row list
        # (a device-wide select + size sync) only when some row was flagged
        if int(flags.amax().item()) == 0:
            return 0
        bad = torch.nonzero(flags).flatten()
        self._dense_rows(x, heads, hq, k, out, bad.cpu().numpy(), scores)
        if runs is not None:  # re-selected rows are ascending: one run
            runs[bad] = 0
            runs[bad, 0] = torch.clamp_max(x.prefix[bad], k)
        return int(bad.numel())

    def _dense_rows(self, x: PreparedInputs, heads, hq, k, out, rows: np.ndarray, scores=None):
        """Exact fallback for flagged rows: the decode machinery on just those rows (their
        queries / gates / heads gathered), i.e. key-split dense scores on every SM and the
        long-row exact selector — one pass for all flagged rows, whatever their number."""
        dev = x.keys.device
        if heads is not None and heads.dim() == 1:  # a raw workspace buffer
            heads = heads[: x.T * hq].view(x.T, hq)
        if x.seq is not None:  # one pass per sequence: the decode machinery scores one key set
            k0 = x.seq.key0_host[rows]
            for key0 in np.unique(k0):
                rs = rows[k0 == key0]
                n = int(x.prefix_host[rs].max())
                xs = PreparedInputs(x.keys[key0: key0 + n], x.queries, x.weights, x.prefix, x.prefix_host, n, x.T,
                                    x.H, x.Hp, x.d, x.D, None)
                self._dense_rows(xs, heads, hq, k, out, rs, scores)
            return
        sel = torch.from_numpy(rows.astype(np.int64)).to(dev)
        xr = PreparedInputs(x.keys, x.queries.index_select(0, sel).contiguous(),
                            x.weights.index_select(0, sel).contiguous(), x.prefix.index_select(0, sel).contiguous(),
                            x.prefix_host[rows], x.L, int(rows.shape[0]), x.H, x.Hp, x.d, x.D, None, x.pages)
        hr = None if heads is None else heads.index_select(0, sel).contiguous()
        o = torch.empty((xr.T, k), dtype=torch.int32, device=dev)
        so = None if scores is None else torch.empty((xr.T, k), dtype=torch.float32, device=dev)
        self.dense_select(xr, hr, hq, k, o, scores=so)
        out[sel] = o
        if scores is not None:
            scores[sel] = so

    def refine(self, x: PreparedInputs, cand: torch.Tensor, k: int, out: torch.Tensor,
               runs: torch.Tensor | None = None):
        """K5 + dense select within candidates (MISA-dagger fine stage); ``runs``: the
        candidates are the coarse selector's 4 ascending runs per row."""
        dev = x.keys.device
        kp = cand.shape[1]
        ckey = x.list_key()
        # the candidate count of row t is min(n_t, k'), taken from the device prefix lengths:
        # under a CUDA graph (DecodeGraph) the host lengths are the bucket's, not the cache's
        ncand = self._buf("refine_ncand", (x.T,), torch.int32, dev)
        torch.clamp_max(x.prefix, kp, out=ncand)
        (rows,) = self._dev_list(("refine_rows", ckey, kp),  # schedule only: longest rows first
                                 lambda: (np.argsort(-np.minimum(x.prefix_host, kp), kind="stable").astype(np.int32),),
                                 dev)
        stream = self._stream()
        lc = kp // 4
        if kp % 4 == 0 and lc in V5_CAPS and x.L <= 32 * 8192:  # topk5's chunk scan covers <= 8192 chunks
            # scores packed as the fused selector's 4 candidate lists: the re-rank's top-k is then
            # misa_select_topk (chunk-scan ordering), not a per-row CTA over a dense score row
            lists = self._buf("refine_lists", (x.T, 4, lc), torch.int64, dev)
            lcnt = self._buf("refine_lcnt", (x.T, 4), torch.int32, dev)
            flags = self._buf("refine_flags", (x.T,), torch.int32, dev)
            self._mark("refine")
            _lib.call("misa_refine_candidates", _ptr(x.keys), x.n_keys, x.D, _ptr(x.queries), _ptr(x.weights), x.H,
                      x.Hp, _ptr(cand), cand.stride(0), _ptr(ncand), _ptr(rows), rows.numel(), x.T,
                      None if x.seq is None else _ptr(x.seq.key0), _ptr(lists), lc, _ptr(lcnt), stream)
            self._mark("refine_select")
            _lib.call("misa_select_topk", _ptr(lists), _ptr(lcnt), lc, _ptr(x.prefix), x.T, k, x.L, _ptr(out),
                      out.stride(0), None, _ptr(flags), stream)
        else:
            rs = self._buf("refine_scores", (x.T, kp), torch.float32, dev)
            self._mark("refine")
            _lib.call("misa_refine_scores", _ptr(x.keys), x.n_keys, x.D, _ptr(x.queries), _ptr(x.weights), x.H,
                      x.Hp, _ptr(cand), cand.stride(0), _ptr(ncand), _ptr(rows), rows.numel(), x.T,
                      None if x.seq is None else _ptr(x.seq.key0), _ptr(rs), kp, stream)
            self._mark("refine_select")
            if runs is not None:
                _lib.call("misa_select_dense_runs", _ptr(rs), kp, _ptr(cand), cand.stride(0), _ptr(ncand),
                          _ptr(runs), x.T, k, _ptr(out), out.stride(0), stream)
            else:
                _lib.call("misa_select_dense", _ptr(rs), kp, _ptr(cand), cand.stride(0), _ptr(ncand), None, x.T, k,
                          _ptr(out), out.stride(0), None, stream)
        self._mark("refine:end")

    # ----------------------------------------------------------- decode
    @staticmethod
    def split_items(lens: np.ndarray, G: int, target_items: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Groups of G rows, each group's 128-key tiles split into chunks so that about
        ``target_items`` work items exist (key-axis split for few rows x long prefixes)."""
        T = lens.shape[0]
        ng = (T + G - 1) // G
        pad = np.zeros(ng * G, dtype=np.int64)
        pad[:T] = lens
        tiles = (pad.reshape(ng, G).max(1) + 127) // 128
        total = int(tiles.sum())
        chunk = max(4, -(-total // max(1, target_items)))
        it_g, it_n, it_0 = [], [], []
        for g in range(ng):
            for t0 in range(0, int(tiles[g]), chunk):
                it_g.append(g)
                it_0.append(t0)
                it_n.append(min(chunk, int(tiles[g]) - t0))
        order = np.argsort(-np.asarray(it_n), kind="stable")
        return (np.asarray(it_g, np.int32)[order], np.asarray(it_n, np.int32)[order],
                np.asarray(it_0, np.int32)[order])

    def dense_scores(self, x: PreparedInputs, heads, hq: int) -> torch.Tensor:
        """(T, L) f32 score rows (valid up to each prefix), key-axis split across the SMs."""
        dev = x.keys.device
        G = 256 // hq
        ckey = x.list_key()
        target = 4 * _lib.load().misa_sm_count()
        items, tiles, tile0 = self._dev_list(("split", ckey, G, target),
                                             lambda: self.split_items(x.prefix_host, G, target), dev)
        rows = self._buf("dense_rows", (x.T, x.L), torch.float32, dev)
        self._mark("decode:score")
        if x.pages is not None:
            table, page = x.pages
            _lib.call("misa_score_materialize_paged", _ptr(x.keys), x.keys.shape[0], x.D, _ptr(x.queries),
                      _ptr(x.weights), x.H, x.Hp, _ptr(heads), hq, _ptr(x.prefix), x.T, _ptr(items), _ptr(tiles),
                      _ptr(tile0), items.numel(), _ptr(table), page, _ptr(rows), x.L, self._stream())
        else:
            _lib.call("misa_score_materialize_split", _ptr(x.keys), x.L, 1, x.D, _ptr(x.queries), _ptr(x.weights),
                      x.H, x.Hp, _ptr(heads), hq, _ptr(x.prefix), x.T, _ptr(items), _ptr(tiles), _ptr(tile0),
                      items.numel(), _ptr(rows), x.L, self._stream())
        return rows

    def dense_select(self, x: PreparedInputs, heads, hq: int, k: int, out: torch.Tensor,
                     scores: torch.Tensor | None = None) -> None:
        """Key-split dense scoring + exact per-row top-k (decode rows); ``scores`` (T, k)
        receives the selected scores (a key shard's local top-k)."""
        dev = x.keys.device
        rows = self.dense_scores(x, heads, hq)
        self._mark("decode:select")
        if x.L <= 16384:  # the whole row fits the register selector
            _lib.call("misa_select_dense", _ptr(rows), x.L, None, 0, _ptr(x.prefix), None, x.T, k, _ptr(out),
                      out.stride(0), _ptr(scores), self._stream())
            return
        beta = 2.0 if k < 4096 else 1.3
        cap = min(16384, max(2 * k, 1 << (int(math.ceil(1.5 * beta * k)) - 1).bit_length()))
        n_seg = -(-x.L // 4096)
        tau = self._buf("long_tau", (x.T,), torch.float32, dev)
        seg = self._buf("long_seg", (x.T, n_seg), torch.int32, dev)
        cs = self._buf("long_cs", (x.T, cap), torch.float32, dev)
        ci = self._buf("long_ci", (x.T, cap), torch.int32, dev)
        cc = self._buf("long_cc", (x.T,), torch.int32, dev)
        _lib.call("misa_select_dense_long", _ptr(rows), x.L, _ptr(x.prefix), x.T, k, int(x.prefix_host.max()),
                  float(beta), _ptr(tau), _ptr(seg), _ptr(cs), _ptr(ci), _ptr(cc), cap, _ptr(out), out.stride(0),
                  _ptr(scores), self._stream())

    def decode_filter_select(self, x: PreparedInputs, heads, hq: int, k: int, out: torch.Tensor):
        """Decode rows through the fused filter: a 1/stride key sample scored on every SM gives
        tau_t (a CTA per row), the key-split filter scorer appends (score, key) >= tau_t to the
        row's four candidate lists (slots reserved per 32-key chunk with one atomic), the
        selector cuts the exact top-k (unordered runs) and a row sort restores topk_tokens'
        ascending order.  No T x L score rows touch HBM.  Returns the (T,) flags of rows whose
        candidates under/overflowed (to be re-selected exactly), or None when the shape falls
        outside the compiled selector (caller takes the dense path)."""
        dev = x.keys.device
        if x.pages is not None or x.seq is not None:
            return None
        stride = max(32, -(-x.L // 16384))
        beta = 2.0 if k < 4096 else 1.2
        j = max(1.0, beta * k / stride)
        cap = int(math.ceil((1.0 + 5.5 / math.sqrt(j)) * beta * k / 4 / 32)) * 32
        cap = next((c for c in V5_CAPS if c >= cap), None)
        if cap is None:
            return None
        G = 256 // hq
        target = 4 * _lib.load().misa_sm_count()
        ckey = x.list_key()
        m = -(-x.L // stride)
        lens_s = -(-x.prefix_host // stride)
        s_items, s_tiles, s_tile0 = self._dev_list(("dsamp", ckey, G, target, stride),
                                                   lambda: self.split_items(lens_s, G, target), dev)
        samp = self._buf("dec_samp", (x.T, m), torch.float32, dev)
        stream = self._stream()
        self._mark("decode:sample")
        _lib.call("misa_score_materialize_split", _ptr(x.keys), x.L, stride, x.D, _ptr(x.queries), _ptr(x.weights),
                  x.H, x.Hp, _ptr(heads), hq, _ptr(x.prefix), x.T, _ptr(s_items), _ptr(s_tiles), _ptr(s_tile0),
                  s_items.numel(), _ptr(samp), m, stream)
        tau = self._buf("dec_tau", (x.T,), torch.float32, dev)
        self._mark("decode:threshold")
        _lib.call("misa_select_threshold", _ptr(samp), m, _ptr(x.prefix), x.T, stride, k, float(beta), 4 * cap,
                  _ptr(tau), stream)
        cand = self._buf("dec_cand", (x.T * 4 * cap,), torch.int64, dev)
        cnt = self._buf("dec_cnt", (x.T * 4,), torch.int32, dev)
        cnt.zero_()
        items, tiles, tile0 = self._dev_list(("split", ckey, G, target),
                                             lambda: self.split_items(x.prefix_host, G, target), dev)
        self._mark("decode:filter")
        _lib.call("misa_score_filter_split", _ptr(x.keys), x.L, x.D, _ptr(x.queries), _ptr(x.weights), x.H, x.Hp,
                  _ptr(heads), hq, _ptr(x.prefix), x.T, _ptr(items), _ptr(tiles), _ptr(tile0), items.numel(),
                  _ptr(tau), _ptr(cand), cap, _ptr(cnt), stream)
        flags = self._buf("dec_flags", (x.T,), torch.int32, dev)
        runs = self._buf("dec_runs", (x.T, 4), torch.int32, dev)
        self._mark("decode:select")
        _lib.call("misa_select_topk_runs", _ptr(cand), _ptr(cnt), cap, _ptr(x.prefix), x.T, k, x.L, _ptr(out),
                  out.stride(0), _ptr(runs), _ptr(flags), stream)
        _lib.call("misa_sort_rows", _ptr(out), out.stride(0), _ptr(x.prefix), x.T, k, stream)
        return flags

    def decode(self, keys=None, queries=None, weights=None, prefix_len=None, *, cache=None,
               need_importance: bool = False, out: torch.Tensor | None = None) -> IndexerOutput:
        """Decode step: a few query rows (T <= a few hundred) against long prefixes.

        Scores are materialised with the key axis split across the SMs (a causal-prefill
        work item is a whole row group, which would leave most SMs idle here) and each row
        takes the exact long-row selector; with ``cache`` (a ``PooledKeyCache``) the keys
        and the router's pooled state come from the incrementally maintained cache.
        Row t equals the reference on ``IndexerWorkload(K[:n_t], Q[t], W[t])``; the
        default prefix is the whole cache / key set for every row."""
        if cache is not None and getattr(cache, "paged", False):
            if self.method == "misa_hier":
                raise ValueError("misa_hier decode needs a contiguous key cache (PooledKeyCache)")
            x = paged_inputs(cache, queries, weights, prefix_len)
            return self.decode_prepared(x, cache=cache, need_importance=need_importance, out=out)
        if cache is not None:
            keys = cache.keys[:cache.length, :cache.d]
        if keys is None or queries is None or weights is None:
            raise ValueError("decode needs keys (or a cache), queries and weights")
        Tq = int(queries.shape[0])
        L = int(keys.shape[0])
        if prefix_len is None:
            prefix_len = np.full(Tq, L, dtype=np.int64)
        x = prepare_inputs(keys, queries, weights, prefix_len)
        return self.decode_prepared(x, cache=cache, need_importance=need_importance, out=out)

    def decode_prepared(self, x: PreparedInputs, *, cache=None, need_importance: bool = False,
                        out: torch.Tensor | None = None) -> IndexerOutput:
        """decode() on prepared inputs: no host synchronisation and no allocation once the
        workspace exists, so it can be captured in a CUDA graph (``DecodeGraph``)."""
        dev = x.keys.device
        k = self.k
        if out is None:
            out = torch.empty(x.T, k, dtype=torch.int32, device=dev)
        heads, hq, imp = None, x.Hp, None
        if self.method != "dsa":
            heads, hq, imp = self.route(x, need_importance, cache=cache)
        kk = k if self.method != "misa_hier" else max(self.kprime, k)
        tgt = out if self.method != "misa_hier" else self._buf("hier_cand", (x.T, kk), torch.int32, dev)
        flags = None
        if x.T >= self.decode_filter_min_rows and x.L >= self.decode_filter_min_keys:
            flags = self.decode_filter_select(x, heads, hq, kk, tgt)
        if flags is None:
            self.dense_select(x, heads, hq, kk, tgt)
        self.last_decode_flags = flags
        self.last_fallback_rows = 0
        if flags is not None and not torch.cuda.is_current_stream_capturing():
            # eager: flagged rows (candidate under/overflow) are re-selected exactly on the
            # dense path; under a CUDA graph DecodeGraph.step checks the flags after replay
            self.last_fallback_rows = self.fix_decode_rows(x, heads, hq, kk, tgt, flags)
        self._mark("decode:end")
        h = min(self.h, x.H)
        if self.method == "dsa":
            return IndexerOutput(topk=out)
        if self.method == "misa":
            return IndexerOutput(topk=out, heads=heads[:, :h], importance=None if imp is None else imp[:, :x.H])
        self.refine(x, tgt, k, out)
        return IndexerOutput(topk=out, heads=heads[:, :h], importance=None if imp is None else imp[:, :x.H],
                             candidates=tgt)

    def fix_decode_rows(self, x: PreparedInputs, heads, hq: int, k: int, out: torch.Tensor, flags) -> int:
        """Exact re-selection of the rows a fused-filter decode step flagged (host check)."""
        if int(flags.amax().item()) == 0:
            return 0
        bad = torch.nonzero(flags).flatten().cpu().numpy()
        self._dense_rows(x, heads, hq, k, out, bad)
        return int(bad.shape[0])

    # ----------------------------------------------------------- host pipeline
    def run_host(self, keys, queries, weights, prefix_len=None, *, chunks: int = 8,
                 out: torch.Tensor | None = None) -> torch.Tensor:
        """Host (ideally pinned) inputs -> host (T, k) top-k, with the copies overlapped.

        Rows are split into ``chunks`` groups of about equal causal work; chunk c+1's
        queries / gates are copied host->device on one stream while chunk c is scored on
        the compute stream, and chunk c's result goes device->host on a third stream.  The
        keys (small: L x d bf16) are uploaded once up front."""
        Kh = torch.as_tensor(keys)
        Qh = torch.as_tensor(queries)
        Wh = torch.as_tensor(weights)
        L, T = int(Kh.shape[0]), int(Qh.shape[0])
        if prefix_len is None:
            if T > L:
                raise ValueError(f"causal prefill needs T <= L, got T={T}, L={L}")
            pl = np.arange(L - T + 1, L + 1, dtype=np.int64)
        else:
            pl = np.asarray(prefix_len.cpu() if isinstance(prefix_len, torch.Tensor) else prefix_len,
                            dtype=np.int64).reshape(-1)
        dev = torch.device("cuda")
        k = self.k
        if out is None:  # a fresh result per call (the caller owns it); pass `out` to reuse a pinned buffer
            out = torch.empty(T, k, dtype=torch.int32, pin_memory=True)
        elif tuple(out.shape) != (T, k) or out.dtype != torch.int32 or out.is_cuda:
            raise ValueError(f"out must be a host (T={T}, k={k}) int32 tensor")
        # chunks of equal row counts (the uploads bound the pipeline and every row is the same
        # number of bytes), processed LAST rows first: the long causal rows' scoring then
        # overlaps the later uploads and the final chunks are the cheap short rows; the first
        # chunk of rows is cut again into 4 so that what runs after the final upload — its
        # scoring and result copy — is short
        fr = [(c + 1) / chunks for c in range(chunks - 1)]
        if chunks >= 4:
            fr = [i / (4 * chunks) for i in (1, 2, 3)] + fr
        cuts = [0] + [int(round(T * f)) for f in fr] + [T]
        cuts = sorted(set(min(max(c, 0), T) for c in cuts))
        spans = [(a, b) for a, b in zip(cuts, cuts[1:]) if b > a][::-1]
        rmax = max(b - a for a, b in spans)
        comp = torch.cuda.current_stream()
        # nothing in the loop below waits on the device: the prefix lengths go up once, and
        # the fused selector's overflow flags are gathered on the device and checked after
        # the last chunk (flagged rows are then re-run exactly from the host inputs)
        pl_dev = torch.from_numpy(pl.astype(np.int32)).pin_memory().to(dev, non_blocking=True)
        flags_all = torch.zeros(T, dtype=torch.int32, device=dev)
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        Kd = torch.empty(Kh.shape, dtype=Kh.dtype, device=dev)
        # a ring of device buffers, as deep as 8 GiB allows: an upload never waits for the
        # scoring of an earlier chunk to free its buffer (with two buffers the uploads stalled
        # behind the longer late chunks: 48.7 -> 42 ms at C4)
        row_bytes = Qh[0].numel() * Qh.element_size() + Wh[0].numel() * Wh.element_size() + k * 4
        NB = int(min(len(spans), max(2, (8 << 30) // max(1, rmax * row_bytes))))
        Qd = [torch.empty((rmax,) + tuple(Qh.shape[1:]), dtype=Qh.dtype, device=dev) for _ in range(NB)]
        Wd = [torch.empty((rmax,) + tuple(Wh.shape[1:]), dtype=Wh.dtype, device=dev) for _ in range(NB)]
        Od = [torch.empty((rmax, k), dtype=torch.int32, device=dev) for _ in range(NB)]
        timed = getattr(self, "time_host_pipeline", False)  # dev: keep timed events for inspection
        ev_in = [torch.cuda.Event(enable_timing=timed) for _ in spans]
        ev_comp = [torch.cuda.Event(enable_timing=timed) for _ in spans]
        ev_out = [torch.cuda.Event(enable_timing=timed) for _ in spans]
        if timed:
            self.host_pipeline_events = (spans, ev_in, ev_comp, ev_out)

        def upload(c):
            a, b = spans[c]
            buf = c % NB
            with torch.cuda.stream(s_in):
                if c >= NB:
                    s_in.wait_event(ev_comp[c - NB])  # buffer reused from chunk c-NB
                if c == 0:
                    Kd.copy_(Kh, non_blocking=True)
                Qd[buf][: b - a].copy_(Qh[a:b], non_blocking=True)
                Wd[buf][: b - a].copy_(Wh[a:b], non_blocking=True)
                ev_in[c].record(s_in)

        upload(0)
        for c, (a, b) in enumerate(spans):
            buf = c % NB
            if c + 1 < len(spans):
                upload(c + 1)  # next chunk's copy overlaps this chunk's scoring
            comp.wait_event(ev_in[c])
            if c >= NB:
                comp.wait_event(ev_out[c - NB])  # result buffer drained
            x = prepare_inputs(Kd, Qd[buf][: b - a], Wd[buf][: b - a], pl[a:b], prefix_dev=pl_dev[a:b])
            check, self.check_overflow = self.check_overflow, False
            try:
                self.run_prepared(x, out=Od[buf][: b - a])
            finally:
                self.check_overflow = check
            if check:
                flags_all[a:b].copy_(self.last_flags[: b - a])
            ev_comp[c].record(comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[c])
                out[a:b].copy_(Od[buf][: b - a], non_blocking=True)
                ev_out[c].record(s_out)
        for e in ev_out:
            comp.wait_event(e)
        ev_out[-1].synchronize()  # the D2H copies are stream-ordered on s_out: the last one covers all
        if self.check_overflow:
            bad = torch.nonzero(flags_all).flatten().cpu().numpy()
            if bad.size:  # exact re-run of just those rows (the device path's own fallback)
                torch.cuda.current_stream().synchronize()
                bi = torch.from_numpy(bad)
                fix = self.run(Kd, Qh[bi].to(dev), Wh[bi].to(dev), prefix_len=pl[bad]).topk
                out[bi] = fix.cpu()
            self.last_fallback_rows = int(bad.size)
        return out

    # ----------------------------------------------------------- entry
    def run(self, keys, queries, weights, prefix_len=None, *, need_importance: bool = False,
            out: torch.Tensor | None = None) -> IndexerOutput:
        x = prepare_inputs(keys, queries, weights, prefix_len)
        return self.run_prepared(x, need_importance=need_importance, out=out)

    def run_varlen(self, keys, cu_seqlens_k, queries, weights, cu_seqlens_q, prefix_len=None, *,
                   need_importance: bool = False, out: torch.Tensor | None = None) -> IndexerOutput:
        """Rows of several independent sequences in one call (see ``prepare_varlen``); the
        returned token indices are relative to each row's own sequence."""
        x = prepare_varlen(keys, cu_seqlens_k, queries, weights, cu_seqlens_q, prefix_len, block_size=self.B)
        return self.run_prepared(x, need_importance=need_importance, out=out)

    def row_chunk(self, x: PreparedInputs) -> int:
        """Rows per pass so that the per-row workspace (sampled scores, candidate lists, router
        partials, MISA-dagger candidates and re-rank scores) stays within ``workspace_bytes``.
        At C4 (128K) every method runs in one pass; at C5 (1M keys) the sample row alone is
        64 KiB and the candidate lists 48 KiB per row, so the rows go in a few passes."""
        kc = self.k if self.method != "misa_hier" else max(self.kprime, self.k)
        stride, _, cap = self.selector_params(kc, x.L)
        per_row = -(-x.L // stride) * 4 + 4 * cap * 8 + 64
        if self.method != "dsa":
            per_row += max(1, (x.L // self.B + 127) // 128) * x.Hp * 4 + x.Hp * 4 + 64
        if self.method == "misa_hier":
            per_row += 2 * kc * 4
        rows = max(256, (self.workspace_bytes // per_row) // 256 * 256)
        return x.T if rows >= x.T else rows

    def run_prepared(self, x: PreparedInputs, *, need_importance: bool = False,
                     out: torch.Tensor | None = None) -> IndexerOutput:
        """All T rows; in row passes of ``row_chunk`` rows when the workspace would exceed
        ``workspace_bytes`` (each pass is an independent batch of rows: same result)."""
        if out is None:
            out = torch.empty(x.T, self.k, dtype=torch.int32, device=x.keys.device)
        span = self.row_chunk(x)
        if span >= x.T:
            return self._run_rows(x, need_importance, out)
        res = IndexerOutput(topk=out)
        flags = torch.empty(x.T, dtype=torch.int32, device=x.keys.device) if not self.check_overflow else None
        nfb = 0
        for a in range(0, x.T, span):
            b = min(x.T, a + span)
            r = self._run_rows(x.rows(a, b), need_importance, out[a:b])
            nfb += r.n_fallback_rows
            if flags is not None:
                flags[a:b].copy_(self.last_flags[: b - a])
            for name in ("heads", "importance", "candidates", "candidate_runs"):
                v = getattr(r, name)
                if v is None:
                    continue
                if getattr(res, name) is None:
                    setattr(res, name, torch.empty((x.T,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device))
                getattr(res, name)[a:b].copy_(v)
        if flags is not None:
            self.last_flags = flags
        res.n_fallback_rows = nfb
        self.last_fallback_rows = nfb
        return res

    def _run_rows(self, x: PreparedInputs, need_importance: bool, out: torch.Tensor) -> IndexerOutput:
        dev = x.keys.device
        k = self.k
        if self.method == "dsa":
            nfb = self.select(x, None, x.Hp, k, out)
            self.last_fallback_rows = nfb
            return IndexerOutput(topk=out, n_fallback_rows=nfb)
        heads, hq, imp = self.route(x, need_importance)
        h = min(self.h, x.H)
        if self.method == "misa":
            nfb = self.select(x, heads, hq, k, out)
            self.last_fallback_rows = nfb
            return IndexerOutput(topk=out, heads=heads[:, :h], importance=None if imp is None else imp[:, :x.H],
                                 n_fallback_rows=nfb)
        kp = max(self.kprime, k)
        cand = self._buf("hier_cand", (x.T, kp), torch.int32, dev)
        runs = self._buf("hier_runs", (x.T, 4), torch.int32, dev)
        nfb = self.select(x, heads, hq, kp, cand, tag="coarse", runs=runs)
        self.refine(x, cand, k, out, runs=runs)
        self.last_fallback_rows = nfb
        return IndexerOutput(topk=out, heads=heads[:, :h], importance=None if imp is None else imp[:, :x.H],
                             candidates=cand, n_fallback_rows=nfb, candidate_runs=runs)


_SHARED = threading.local()


def shared_engine(method: str, **kw) -> IndexerEngine:
    """One engine per (method, parameters) and thread for the single-query API
    (``dsa_select``, ``misa_select``, ...): its workspace and work lists are reused across
    calls instead of being rebuilt per query.  Per-thread small LRU, so concurrent calls from
    several threads stay independent (the reference functions are thread-safe)."""
    cache = getattr(_SHARED, "engines", None)
    if cache is None:
        cache = _SHARED.engines = {}
    key = (method, torch.cuda.current_device(), tuple(sorted(kw.items())))
    eng = cache.pop(key, None)
    if eng is None:
        eng = IndexerEngine(method, **kw)
        while len(cache) >= 8:
            cache.pop(next(iter(cache)))
    cache[key] = eng
    return eng


class DecodeGraph:
    """Per-token decode step replayed from a CUDA graph (serving path for configs C5).

    The step (router on the cache's pooled state, key-split scoring, long-row exact
    selection) is captured once per key bucket: work lists cover the cache length
    rounded up to ``bucket`` keys while the kernels read the true prefix length from a
    device buffer, so a graph serves every length in its bucket (the masked tail costs
    < bucket keys) and is re-captured only when the cache crosses into the next bucket.
    Inputs are copied into static buffers; the result tensor is reused across steps."""

    def __init__(self, engine: "IndexerEngine", cache, n_rows: int, n_heads: int, bucket: int = 4096):
        self.engine, self.cache, self.T, self.H = engine, cache, int(n_rows), int(n_heads)
        self.bucket = check_positive_int(bucket, "bucket")
        self.paged = bool(getattr(cache, "paged", False))
        if self.paged:
            if engine.method == "misa_hier":
                raise ValueError("misa_hier decode needs a contiguous key cache (PooledKeyCache)")
            self.bucket = cache.B  # the router's partial-block address is fixed within one page
        dev = (cache.pool_keys if self.paged else cache.keys).device
        self.Hp = heads_pad(self.H)
        self.q = torch.zeros(self.T, self.Hp, cache.D, dtype=torch.bfloat16, device=dev)
        self.w = torch.zeros(self.T, self.Hp, dtype=torch.float32, device=dev)
        self.prefix = torch.zeros(self.T, dtype=torch.int32, device=dev)
        self.out = torch.empty(self.T, engine.k, dtype=torch.int32, device=dev)
        self.graph = None
        self.Lb = 0
        self.result = None
        self._x = None
        self._flag_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)  # fused-filter steps: max flag
        self._checks = False

    def _capture(self, Lb: int) -> None:
        c = self.cache
        host = np.full(self.T, Lb, dtype=np.int64)
        if self.paged:
            x = PreparedInputs(c.pool_keys, self.q, self.w, self.prefix, host, Lb, self.T, self.H, self.Hp, c.d, c.D,
                               ("decode-paged", Lb, self.T), pages=(c.page_table, c.B))
        else:
            x = PreparedInputs(c.keys[:Lb], self.q, self.w, self.prefix, host, Lb, self.T, self.H, self.Hp, c.d,
                               c.D, ("decode", Lb, self.T))
        eng = self.engine
        self.prefix.fill_(max(1, min(c.length, Lb)))  # warm-up on a valid prefix
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            eng.decode_prepared(x, cache=c, out=self.out)  # warm-up: workspace + work lists
        torch.cuda.current_stream().wait_stream(stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            self.result = eng.decode_prepared(x, cache=c, out=self.out)
            fl = eng.last_decode_flags
            self._checks = fl is not None
            if self._checks:  # the step's flag summary lands in pinned memory inside the graph
                self._flag_host.copy_(fl.amax().view(1), non_blocking=True)
        self._x = x
        # the graph holds raw device pointers into the engine's workspace and cached work
        # lists: keep those tensors alive for the graph's lifetime, even if a later eager call
        # on the same engine swaps in larger buffers or clears the work-list cache
        self._keep = (list(eng._ws.values()), list(eng._lists.values()))
        self.graph, self.Lb = g, Lb

    def step(self, queries, weights) -> IndexerOutput:
        """Top-k of ``queries`` (T, H, d) / ``weights`` (T, H) against the whole cache."""
        L = self.cache.length
        if L < 1:
            raise ValueError("empty cache")
        Lb = min(self.cache.capacity, -(-L // self.bucket) * self.bucket)
        if self.graph is None or Lb != self.Lb:
            self._capture(Lb)
        self.q[:, :self.H, :self.cache.d].copy_(queries, non_blocking=True)
        self.w[:, :self.H].copy_(weights, non_blocking=True)
        self.prefix.fill_(L)
        self.graph.replay()
        if self._checks:
            # a fused-filter step is exact unless a row's candidates under/overflowed: then the
            # whole step is re-run eagerly on the dense path (rare; keeps every step exact)
            torch.cuda.current_stream().synchronize()
            if int(self._flag_host.item()):
                eng = self.engine
                keep, eng.decode_filter_min_rows = eng.decode_filter_min_rows, 1 << 30
                try:
                    self.result = eng.decode_prepared(self._x, cache=self.cache, out=self.out)
                finally:
                    eng.decode_filter_min_rows = keep
        return self.result
