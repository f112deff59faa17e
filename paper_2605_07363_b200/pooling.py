"""Block pooling (``pooling.py:12-115``) on the device.

``build_block_summary`` runs the K1 pooling kernel; ``incremental_append`` runs
the decode-append kernel on the block's running prefix sum.  ``PooledKeyCache``
is the device-resident decode state (keys + in-block prefix sums + pooled
planes) that serving code appends to one key at a time.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import head_dim_pad
from .validation import check_positive_int


@dataclass(frozen=True)
class BlockSummary:
    """Block partition of a prefix plus one mean-pooled key per block (``pooling.py:12-54``)."""

    block_size: int
    boundaries: np.ndarray
    pooled_keys: np.ndarray

    def __post_init__(self) -> None:
        check_positive_int(self.block_size, "block_size")
        bounds = np.array(self.boundaries, dtype=np.int64, copy=True).reshape(-1, 2)
        pooled = np.array(self.pooled_keys, dtype=np.float64, copy=True)
        if pooled.ndim != 2 or pooled.shape[0] != bounds.shape[0]:
            raise ValueError("pooled_keys must hold one row per block")
        if bounds.shape[0]:
            starts, ends = bounds[:, 0], bounds[:, 1]
            if starts[0] != 0 or np.any(starts[1:] != ends[:-1]) or np.any(ends <= starts):
                raise ValueError("blocks must tile the prefix contiguously")
            lengths = ends - starts
            if np.any(lengths[:-1] != self.block_size) or lengths[-1] > self.block_size:
                raise ValueError("all blocks must have block_size keys except a shorter last block")
        bounds.setflags(write=False)
        pooled.setflags(write=False)
        object.__setattr__(self, "boundaries", bounds)
        object.__setattr__(self, "pooled_keys", pooled)

    @property
    def n_blocks(self) -> int:
        return int(self.boundaries.shape[0])

    @property
    def prefix_len(self) -> int:
        return int(self.boundaries[-1, 1]) if self.n_blocks else 0

    def block_tokens(self, block: int) -> np.ndarray:
        start, end = self.boundaries[block]
        return np.arange(start, end, dtype=np.int64)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _bounds(L: int, B: int) -> np.ndarray:
    m = -(-L // B)
    starts = np.arange(m, dtype=np.int64) * B
    return np.stack([starts, np.minimum(starts + B, L)], axis=1)


def build_block_summary(keys, block_size: int) -> BlockSummary:
    """Mean-pool contiguous blocks; the partial last block is pooled over its real length."""
    check_positive_int(block_size, "block_size")
    arr = keys if isinstance(keys, torch.Tensor) else np.asarray(keys, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError("keys must be a 2-D matrix")
    L, d = int(arr.shape[0]), int(arr.shape[1])
    if L == 0:
        return BlockSummary(block_size, np.empty((0, 2), np.int64), np.empty((0, d)))
    D = head_dim_pad(d)
    K = (arr if isinstance(arr, torch.Tensor) else torch.tensor(arr)).to(device="cuda", dtype=torch.bfloat16)
    if D != d:
        K = torch.nn.functional.pad(K, (0, D - d))
    K = K.contiguous()
    nf = L // block_size
    P = torch.empty(L, D, dtype=torch.float32, device="cuda")
    pooled = torch.empty(max(nf, 1), D, dtype=torch.float32, device="cuda")
    _lib.call("misa_pool_keys", K.data_ptr(), L, D, block_size, P.data_ptr(), pooled.data_ptr(), None, 0, _stream())
    out = pooled[:nf, :d].double()
    rem = L - nf * block_size
    if rem:
        out = torch.cat([out, (P[L - 1, :d].double() / rem)[None]], 0)
    return BlockSummary(block_size, _bounds(L, block_size), out.cpu().numpy())


def incremental_append(summary: BlockSummary, new_key) -> BlockSummary:
    """Summary for the prefix grown by one key (running mean / new block), on the device."""
    new_key = np.asarray(new_key, dtype=np.float64).reshape(-1)
    if summary.n_blocks and new_key.shape[0] != summary.pooled_keys.shape[1]:
        raise ValueError(f"new key has dim {new_key.shape[0]}, summary has dim {summary.pooled_keys.shape[1]}")
    B = summary.block_size
    d = new_key.shape[0]
    D = head_dim_pad(d)
    L = summary.prefix_len
    pos = L % B
    open_block = summary.n_blocks > 0 and pos != 0
    # row 0 carries the open block's running sum (zero for a new block), row 1 is the new key;
    # the append kernel at s=1 (block size >= 2, so s is mid-block) writes P[1] = P[0] + key.
    keys = torch.zeros(2, D, dtype=torch.bfloat16, device="cuda")
    keys[1, :d] = torch.as_tensor(new_key, device="cuda").to(torch.bfloat16)
    P = torch.zeros(2, D, dtype=torch.float32, device="cuda")
    if open_block:
        P[0, :d] = torch.as_tensor(summary.pooled_keys[-1] * pos, device="cuda").float()
    _lib.call("misa_pool_append", keys.data_ptr(), 1, D, max(B, 2), P.data_ptr(), None, None, 0, _stream())
    if open_block:
        pooled = summary.pooled_keys.copy()
        pooled[-1] = (P[1, :d].double() / (pos + 1)).cpu().numpy()
        bounds = summary.boundaries.copy()
        bounds[-1, 1] = L + 1
    else:
        pooled = np.vstack([summary.pooled_keys.reshape(-1, d), P[1, :d].double().cpu().numpy()[None]])
        bounds = np.vstack([summary.boundaries.reshape(-1, 2), [[L, L + 1]]])
    return BlockSummary(B, bounds, pooled)


class PooledKeyCache:
    """Device-resident decode state: bf16 keys, in-block prefix sums and pooled planes.

    ``append(key_rows)`` extends the cache and updates the pooling state with the
    decode kernel (one launch per key); the arrays are consumed directly by
    ``IndexerEngine`` (see ``engine.IndexerEngine.route``)."""

    def __init__(self, head_dim: int, block_size: int, capacity: int, device="cuda"):
        self.d = head_dim
        self.D = head_dim_pad(head_dim)
        self.B = check_positive_int(block_size, "block_size")
        self.capacity = check_positive_int(capacity, "capacity")
        self.keys = torch.zeros(capacity, self.D, dtype=torch.bfloat16, device=device)
        self.prefix = torch.zeros(capacity, self.D, dtype=torch.float32, device=device)
        self.rows = max(128, (capacity // self.B + 127) // 128 * 128)
        self.planes = torch.zeros(3, self.rows, self.D, dtype=torch.bfloat16, device=device)
        self.length = 0

    def append(self, key_rows) -> None:
        kr = torch.as_tensor(key_rows, device=self.keys.device).reshape(-1, self.d)
        n = kr.shape[0]
        if self.length + n > self.capacity:
            raise ValueError("PooledKeyCache capacity exceeded")
        self.keys[self.length:self.length + n, :self.d] = kr.to(torch.bfloat16)
        if n <= 8:  # decode: one append launch per key (pooling.py:87-115)
            for i in range(n):
                _lib.call("misa_pool_append", self.keys.data_ptr(), self.length + i, self.D, self.B,
                          self.prefix.data_ptr(), None, self.planes.data_ptr(), self.rows, _stream())
        else:  # bulk (prefill): re-pool the whole prefix in one launch (O(L), ~0.2 ms at 1M keys)
            _lib.call("misa_pool_keys", self.keys.data_ptr(), self.length + n, self.D, self.B,
                      self.prefix.data_ptr(), None, self.planes.data_ptr(), self.rows, _stream())
        self.length += n

    def summary(self) -> BlockSummary:
        L, B, d = self.length, self.B, self.d
        nf = L // B
        full = (self.planes[0, :nf, :d].double() + self.planes[1, :nf, :d].double() + self.planes[2, :nf, :d].double())
        rem = L - nf * B
        out = full if not rem else torch.cat([full, (self.prefix[L - 1, :d].double() / rem)[None]], 0)
        return BlockSummary(B, _bounds(L, B), out.cpu().numpy())


class PagedKeyCache:
    """Paged decode state: keys and in-block prefix sums live in fixed-size pages of one
    pool (page = pooled block, a multiple of 128 keys), reached through a page table;
    the pooled planes of the full blocks stay contiguous (one small row per block).

    Pages are taken from a free list in any order (``page_order`` shuffles it to prove
    the indirection), so a serving system can share the pool across sequences.  The
    scorer translates logical 128-key tiles through the table
    (``misa_score_materialize_paged``); the router needs only the pooled planes and the
    partial block's running sum, whose address ``prefix_base`` hands out."""

    paged = True

    def __init__(self, head_dim: int, block_size: int, n_pages: int, device="cuda", page_order=None):
        self.d = head_dim
        self.D = head_dim_pad(head_dim)
        self.B = check_positive_int(block_size, "block_size")
        if self.B % 128:
            raise ValueError("pages hold whole 128-key tiles: block_size must be a multiple of 128")
        self.n_pages = check_positive_int(n_pages, "n_pages")
        self.capacity = self.n_pages * self.B
        self.pool_keys = torch.zeros(self.capacity, self.D, dtype=torch.bfloat16, device=device)
        self.pool_prefix = torch.zeros(self.capacity, self.D, dtype=torch.float32, device=device)
        self.rows = max(128, (self.n_pages + 127) // 128 * 128)
        self.planes = torch.zeros(3, self.rows, self.D, dtype=torch.bfloat16, device=device)
        self.page_table = torch.full((self.n_pages,), -1, dtype=torch.int32, device=device)
        self._tmp_planes = torch.zeros(3, 1, self.D, dtype=torch.bfloat16, device=device)
        self.free = list(range(self.n_pages)) if page_order is None else [int(p) for p in page_order]
        if sorted(self.free) != list(range(self.n_pages)):
            raise ValueError("page_order must be a permutation of the pool's pages")
        self.pages: list[int] = []
        self.length = 0

    def _phys(self, i: int) -> int:
        return self.pages[i // self.B] * self.B + i % self.B

    def prefix_base(self, L: int) -> int:
        """Address P such that P + (L-1)*D*4 is key L-1's in-block prefix sum (router)."""
        return self.pool_prefix.data_ptr() + (self._phys(L - 1) - (L - 1)) * self.D * 4

    def append(self, key_rows) -> None:
        kr = torch.as_tensor(key_rows, device=self.pool_keys.device).reshape(-1, self.d).to(torch.bfloat16)
        n = kr.shape[0]
        if self.length + n > self.capacity:
            raise ValueError("PagedKeyCache capacity exceeded")
        D, B = self.D, self.B
        pos = 0
        while pos < n:
            L = self.length
            if L % B == 0:  # open a page
                page = self.free.pop(0)
                self.page_table[len(self.pages)] = page
                self.pages.append(page)
            page = self.pages[L // B]
            off = L % B
            m = min(n - pos, B - off)
            base = page * B
            self.pool_keys[base + off:base + off + m, :self.d] = kr[pos:pos + m]
            if m <= 8:
                for i in range(m):  # decode append into the page (logical index via an offset base)
                    _lib.call("misa_pool_append", self.pool_keys.data_ptr() + (base - (L - off)) * D * 2, L + i, D, B,
                              self.pool_prefix.data_ptr() + (base - (L - off)) * D * 4, None,
                              self.planes.data_ptr(), self.rows, _stream())
            else:  # re-pool the page's keys so far: one block, exactly the full-prefix pooling of it
                full = off + m == B
                _lib.call("misa_pool_keys", self.pool_keys.data_ptr() + base * D * 2, off + m, D, B,
                          self.pool_prefix.data_ptr() + base * D * 4, None,
                          self._tmp_planes.data_ptr() if full else None, 1, _stream())
                if full:
                    self.planes[:, L // B].copy_(self._tmp_planes[:, 0])
            self.length += m
            pos += m
