"""Key-axis sharded indexer across the GPUs of one node.

The scoring contraction — the cost of every method — is split along the key
axis: key blocks of ``block`` tokens are assigned block-cyclically (block b ->
rank b mod G), which keeps pooled blocks whole and balances causal prefill
(a contiguous split would give rank 0 ~G times rank G-1's work).  Per layer:

  1. routing (MISA): rank r routes the row slice [r*T/G, (r+1)*T/G) and an
     all-gather assembles every row's heads (T x h int32);
  2. every rank scores all T rows against its own keys (row t sees the local
     keys whose global index is < n_t) and keeps a local top-k *with scores*;
  3. local key indices are mapped to global ones (the map is monotone, so the
     per-rank lists stay ascending);
  4. an all-to-all by row slice hands rank r the G local lists of its rows;
  5. the merge kernel selects the global top-k of each row with the same
     (score desc, index asc) rule — top-k over a union equals top-k over the
     per-part top-k's.

Rows come out row-sliced (rank r owns rows [r*T/G, (r+1)*T/G)); ``gather=True``
all-gathers them.  Decode (a few rows against long prefixes, ``decode``) routes every
row locally (tiny), scores the shard with the key-split decode path, and one
all-gather of the (T x k) local lists lets every rank merge every row.  The key cache is replicated here so that routing and the
partial-block pooling need no extra exchange; only the scoring work is sharded.
MISA-dagger: the coarse top-k' is sharded and merged like the top-k; each rank then
re-ranks its own rows' merged candidates against the (replicated) key set.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .engine import IndexerEngine, PreparedInputs, prepare_inputs


@dataclass(frozen=True)
class KeyShardLayout:
    """Block-cyclic assignment of key blocks to ``n_shards`` ranks."""

    n_shards: int
    shard: int
    block: int

    def local_count(self, n) -> np.ndarray:
        """Number of global keys < n owned by this shard (vectorised over n)."""
        n = np.asarray(n, dtype=np.int64)
        G, r, B = self.n_shards, self.shard, self.block
        fb, rem = n // B, n % B
        owned_full = np.where(fb > r, (fb - r - 1) // G + 1, 0)
        partial = np.where(fb % G == r, rem, 0)
        return owned_full * B + partial

    def local_keys(self, L: int) -> np.ndarray:
        """Global indices of this shard's keys, in local order."""
        G, r, B = self.n_shards, self.shard, self.block
        blocks = np.arange(r, -(-L // B), G, dtype=np.int64)
        idx = (blocks[:, None] * B + np.arange(B, dtype=np.int64)[None, :]).reshape(-1)
        return idx[idx < L]

    def to_global(self, i) -> np.ndarray:
        i = np.asarray(i, dtype=np.int64)
        G, r, B = self.n_shards, self.shard, self.block
        return np.where(i >= 0, ((i // B) * G + r) * B + i % B, -1)


def row_slices(T: int, G: int) -> tuple[int, int]:
    """Rows per rank after padding T up to a multiple of G."""
    per = -(-T // G)
    return per, per * G


def exchange_by_rows(idx: torch.Tensor, scores: torch.Tensor, world: int, group=None):
    """(T_pad, k) local lists on every rank -> (world, T_pad/world, k) lists of this rank's rows.

    NCCL uses one all-to-all; other backends (gloo in the CPU tests) all-gather and slice.
    """
    T_pad, k = idx.shape
    per = T_pad // world
    if world == 1:
        return idx.view(1, per, k), scores.view(1, per, k)
    backend = dist.get_backend(group)
    if backend == "nccl":
        out_i = torch.empty_like(idx)
        out_s = torch.empty_like(scores)
        dist.all_to_all_single(out_i, idx.contiguous(), group=group)
        dist.all_to_all_single(out_s, scores.contiguous(), group=group)
        return out_i.view(world, per, k), out_s.view(world, per, k)
    rank = dist.get_rank(group)
    gi = [torch.empty_like(idx) for _ in range(world)]
    gs = [torch.empty_like(scores) for _ in range(world)]
    dist.all_gather(gi, idx.contiguous(), group=group)
    dist.all_gather(gs, scores.contiguous(), group=group)
    sl = slice(rank * per, (rank + 1) * per)
    return torch.stack([g[sl] for g in gi]), torch.stack([g[sl] for g in gs])


def gather_lists(idx: torch.Tensor, scores: torch.Tensor, world: int, group=None):
    """(T, k) local lists on every rank -> (world, T, k) lists of every rank (decode exchange)."""
    if world == 1:
        return idx[None], scores[None]
    gi = torch.empty((world,) + tuple(idx.shape), dtype=idx.dtype, device=idx.device)
    gs = torch.empty((world,) + tuple(scores.shape), dtype=scores.dtype, device=scores.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(gi, idx.contiguous(), group=group)
        dist.all_gather_into_tensor(gs, scores.contiguous(), group=group)
    else:
        dist.all_gather(list(gi.unbind(0)), idx.contiguous(), group=group)
        dist.all_gather(list(gs.unbind(0)), scores.contiguous(), group=group)
    return gi, gs


class ShardedIndexer:
    """Key-sharded DSA / MISA indexer for one rank of a ``torch.distributed`` group."""

    def __init__(self, method: str = "misa", *, world: int, rank: int, group=None, shard_block: int | None = None,
                 **engine_kwargs):
        if method not in ("dsa", "misa", "misa_hier"):
            raise ValueError(f"sharded execution supports 'dsa', 'misa' and 'misa_hier', got {method!r}")
        self.method = method
        self.world, self.rank, self.group = world, rank, group
        self.engine = IndexerEngine(method, **engine_kwargs)
        self.layout = KeyShardLayout(world, rank, shard_block or self.engine.B)
        self.k = self.engine.k
        kc = self.k if method != "misa_hier" else max(self.engine.kprime, self.k)
        if world * kc > 16384:  # misa_merge_topk holds the union of the per-rank lists in registers
            raise ValueError(f"world_size * candidate budget = {world * kc} exceeds the merge capacity (16384)")
        self._cache: dict = {}
        self.last_fallback_rows = 0

    def _local_keys(self, x: PreparedInputs) -> torch.Tensor:
        """This shard's keys, gathered on every call: a key buffer may be rewritten in place
        between layers (or be a temporary the allocator hands back at the same address), so
        nothing keyed on its address may be cached.  Only the index list is cached (it
        depends on L alone); the gather is one pass over L*D*2 bytes."""
        idx = self._cache.get(("idx", x.L, x.keys.device))
        if idx is None:
            idx = torch.from_numpy(self.layout.local_keys(x.L)).to(x.keys.device)
            self._cache = {("idx", x.L, x.keys.device): idx}
        return x.keys.index_select(0, idx)

    def run(self, keys, queries, weights, prefix_len=None, *, gather: bool = False):
        x = prepare_inputs(keys, queries, weights, prefix_len)
        G, r, k = self.world, self.rank, self.k
        dev = x.keys.device
        per, T_pad = row_slices(x.T, G)
        stream = torch.cuda.current_stream().cuda_stream

        heads, hq = None, x.Hp
        r0, r1 = min(x.T, r * per), min(x.T, (r + 1) * per)
        if self.method != "dsa":
            xs = PreparedInputs(x.keys, x.queries[r0:r1], x.weights[r0:r1], x.prefix[r0:r1], x.prefix_host[r0:r1],
                                x.L, r1 - r0, x.H, x.Hp, x.d, x.D, None)
            h_loc, hq, _ = self.engine.route(xs) if r1 > r0 else (None, 8, None)
            buf = torch.full((per, hq), -1, dtype=torch.int32, device=dev)
            if r1 > r0:
                buf[: r1 - r0] = h_loc
            allh = torch.empty((G * per, hq), dtype=torch.int32, device=dev)
            if G > 1:
                dist.all_gather_into_tensor(allh, buf, group=self.group)
            else:
                allh.copy_(buf)
            heads = allh[: x.T].contiguous()

        # local scoring against this shard's keys
        n_loc = self.layout.local_count(x.prefix_host)
        K_loc = self._local_keys(x)
        xl = PreparedInputs(K_loc, x.queries, x.weights, torch.from_numpy(n_loc.astype(np.int32)).to(dev), n_loc,
                            K_loc.shape[0], x.T, x.H, x.Hp, x.d, x.D, None)
        kc = k if self.method != "misa_hier" else max(self.engine.kprime, k)  # coarse budget
        loc_i = torch.full((T_pad, kc), -1, dtype=torch.int32, device=dev)
        loc_s = torch.full((T_pad, kc), float("-inf"), dtype=torch.float32, device=dev)
        self.last_fallback_rows = self.engine.select(xl, heads, hq, kc, loc_i[: x.T], tag="shard",
                                                     scores=loc_s[: x.T])
        _lib.call("misa_shard_map_indices", loc_i.data_ptr(), loc_i.numel(), self.layout.block, G, r, stream)

        parts_i, parts_s = exchange_by_rows(loc_i, loc_s, G, self.group)
        merged = torch.empty((per, kc), dtype=torch.int32, device=dev)
        _lib.call("misa_merge_topk", parts_s.data_ptr(), parts_i.data_ptr(), G, per * kc, per, kc, kc,
                  merged.data_ptr(), kc, stream)
        if self.method != "misa_hier":
            out = merged
        else:  # MISA-dagger fine stage on this rank's rows (dsa.py:95-115 on the merged candidates)
            out = torch.full((per, k), -1, dtype=torch.int32, device=dev)
            if r1 > r0:
                xs = PreparedInputs(x.keys, x.queries[r0:r1], x.weights[r0:r1], x.prefix[r0:r1],
                                    x.prefix_host[r0:r1], x.L, r1 - r0, x.H, x.Hp, x.d, x.D, None)
                self.engine.refine(xs, merged[: r1 - r0], k, out[: r1 - r0])
        if gather:
            full = torch.empty((G * per, k), dtype=torch.int32, device=dev)
            if G > 1:
                dist.all_gather_into_tensor(full, out, group=self.group)
            else:
                full.copy_(out)
            return full[: x.T]
        return out

    def decode(self, keys, queries, weights, prefix_len=None, *, cache=None):
        """Decode step, key-sharded: every rank returns the global top-k of every row.

        ``keys`` / ``cache`` hold the replicated key set (the router needs every pooled
        block); each rank scores only its block-cyclic shard."""
        if cache is not None:
            keys = cache.keys[:cache.length, :cache.d]
        G, r, k = self.world, self.rank, self.k
        Tq, L = int(queries.shape[0]), int(keys.shape[0])
        if prefix_len is None:
            prefix_len = np.full(Tq, L, dtype=np.int64)
        x = prepare_inputs(keys, queries, weights, prefix_len)
        dev = x.keys.device
        stream = torch.cuda.current_stream().cuda_stream
        eng = self.engine
        heads, hq = None, x.Hp
        if self.method != "dsa":
            heads, hq, _ = eng.route(x, cache=cache)
        kc = k if self.method != "misa_hier" else max(eng.kprime, k)
        n_loc = self.layout.local_count(x.prefix_host)
        K_loc = self._local_keys(x)
        xl = PreparedInputs(K_loc, x.queries, x.weights, torch.from_numpy(n_loc.astype(np.int32)).to(dev), n_loc,
                            K_loc.shape[0], x.T, x.H, x.Hp, x.d, x.D, None)
        loc_i = torch.full((x.T, kc), -1, dtype=torch.int32, device=dev)
        loc_s = torch.full((x.T, kc), float("-inf"), dtype=torch.float32, device=dev)
        if K_loc.shape[0] > 0:
            eng.dense_select(xl, heads, hq, kc, loc_i, scores=loc_s)
        _lib.call("misa_shard_map_indices", loc_i.data_ptr(), loc_i.numel(), self.layout.block, G, r, stream)
        parts_i, parts_s = gather_lists(loc_i, loc_s, G, self.group)
        merged = torch.empty((x.T, kc), dtype=torch.int32, device=dev)
        _lib.call("misa_merge_topk", parts_s.data_ptr(), parts_i.data_ptr(), G, x.T * kc, x.T, kc, kc,
                  merged.data_ptr(), kc, stream)
        if self.method != "misa_hier":
            return merged
        out = torch.empty((x.T, k), dtype=torch.int32, device=dev)
        eng.refine(x, merged, k, out)
        return out
