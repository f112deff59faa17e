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
  4. pruning: tau_t = min over ranks of each rank's (k/G)-th local score
     (one all-reduce(MIN) of T floats).  The G ranks hold at least G*(k/G) = k
     entries >= tau_t, so the global k-th score is >= tau_t and no entry below
     it can be selected; each rank keeps only its entries >= tau_t (about k/G)
     in lists of ``prune_cap`` slots — the exchange ships ~G x less than the
     unpruned T*k*8 bytes per rank;
  5. an all-to-all by row slice hands rank r the G pruned lists of its rows;
     rows whose kept count exceeded the cap on any rank (the all-reduce(MAX) of
     the counts says which, identically on every rank) are exchanged again
     unpruned, and only for those rows;
  6. the merge kernel selects the global top-k of each row with the same
     (score desc, index asc) rule — top-k over a union equals top-k over the
     per-part top-k's; more than 16384 candidates per row (e.g. MISA-dagger's
     k' = 8192 on 4-8 GPUs) are merged in rounds of groups of lists.

Rows come out row-sliced (rank r owns rows [r*T/G, (r+1)*T/G)); ``gather=True``
all-gathers them.  Decode (a few rows against long prefixes, ``decode``) routes every
row locally (tiny), scores the shard with the key-split decode path, prunes the same
way, and one all-gather of the pruned lists lets every rank merge every row.  The key
cache is replicated here so that routing and the partial-block pooling need no extra
exchange; only the scoring work is sharded.  MISA-dagger: the coarse top-k' is sharded,
pruned and merged like the top-k; each rank then re-ranks its own rows' merged
candidates against the (replicated) key set.

Collectives: one code path for every backend — ``all_to_all_single`` and
``all_gather_into_tensor`` on whole row blocks.  NCCL moves device tensors directly;
gloo (the CPU tests, and the 1-GPU dev check of the N > 1 path) gets host copies of
the same tensors, so both transports run the same calls on the same layouts.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .engine import IndexerEngine, PreparedInputs, prepare_inputs

MERGE_CAPACITY = 16384  # elements one merge CTA holds in registers (select.cu dispatch_capacity)


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


def prune_params(k: int, world: int) -> tuple[int, int]:
    """(m, cap): tau is the min over ranks of the m-th local score, m = ceil(k/G), and a
    rank keeps at most cap of its entries >= tau.  About m + O(sqrt(m)) are expected (the
    min of G order statistics sits a few sqrt(m) ranks below m); cap = 1.5m + 8 leaves room
    for that spread (k = 2048 on 8 GPUs: 392 of 2048 slots).  Rows over the cap on any rank
    are exchanged unpruned."""
    m = -(-k // world)
    return m, min(k, m + m // 2 + 8)


# ----------------------------------------------------------------- transport
def _staged(t: torch.Tensor, group) -> bool:
    return t.is_cuda and dist.get_backend(group) != "nccl"


def all_to_all_rows(t: torch.Tensor, world: int, group=None, in_splits=None, out_rows=None) -> torch.Tensor:
    """Rows of ``t`` split into ``world`` consecutive blocks (equal, or ``in_splits`` rows),
    block r sent to rank r; returns the received blocks concatenated in rank order
    (``out_rows`` rows in total when the splits are uneven)."""
    if world == 1:
        return t
    src = t.cpu() if _staged(t, group) else t.contiguous()
    tail = tuple(src.shape[1:])
    if in_splits is None:
        out = torch.empty_like(src)
        dist.all_to_all_single(out, src, group=group)
    else:
        out = torch.empty((int(sum(out_rows)),) + tail, dtype=src.dtype, device=src.device)
        dist.all_to_all_single(out, src, output_split_sizes=[int(x) for x in out_rows],
                               input_split_sizes=[int(x) for x in in_splits], group=group)
    return out.to(t.device) if out.device != t.device else out


def all_gather_rows(t: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """(R, ...) on every rank -> (world, R, ...) in rank order."""
    if world == 1:
        return t[None]
    src = t.cpu() if _staged(t, group) else t.contiguous()
    out = torch.empty((world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    out = out.view((world,) + tuple(src.shape))
    return out.to(t.device) if out.device != t.device else out


def all_reduce_(t: torch.Tensor, op, group=None) -> torch.Tensor:
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def exchange_by_rows(idx: torch.Tensor, scores: torch.Tensor, world: int, group=None):
    """(T_pad, c) lists on every rank -> (world, T_pad/world, c) lists of this rank's rows."""
    T_pad, c = idx.shape
    per = T_pad // world
    return (all_to_all_rows(idx, world, group).view(world, per, c),
            all_to_all_rows(scores, world, group).view(world, per, c))


def gather_lists(idx: torch.Tensor, scores: torch.Tensor, world: int, group=None):
    """(T, c) local lists on every rank -> (world, T, c) lists of every rank (decode exchange)."""
    return all_gather_rows(idx, world, group), all_gather_rows(scores, world, group)


# ------------------------------------------------------------- device ops
class DeviceListOps:
    """The list kernels of the exchange (select.cu), behind a small interface so that the
    CPU tests can drive the same exchange code with host implementations."""

    @staticmethod
    def _stream():
        return torch.cuda.current_stream().cuda_stream

    def kth(self, s: torch.Tensor, m: int) -> torch.Tensor:
        tau = torch.empty(s.shape[0], dtype=torch.float32, device=s.device)
        _lib.call("misa_list_kth", s.data_ptr(), s.stride(0), s.shape[0], s.shape[1], m, tau.data_ptr(),
                  self._stream())
        return tau

    def prune(self, s, i, tau, cap):
        R = s.shape[0]
        os_ = torch.empty((R, cap), dtype=torch.float32, device=s.device)
        oi = torch.empty((R, cap), dtype=torch.int32, device=s.device)
        cnt = torch.empty(R, dtype=torch.int32, device=s.device)
        _lib.call("misa_list_prune", s.data_ptr(), i.data_ptr(), s.stride(0), R, s.shape[1], tau.data_ptr(), cap,
                  os_.data_ptr(), oi.data_ptr(), cnt.data_ptr(), self._stream())
        return os_, oi, cnt

    def merge(self, ps, pi, n_rows, k_out, want_scores=False):
        """(P, n_rows, c) part lists -> (n_rows, k_out) merged (+ scores)."""
        P, _, c = ps.shape
        out = torch.empty((n_rows, k_out), dtype=torch.int32, device=ps.device)
        outs = torch.empty((n_rows, k_out), dtype=torch.float32, device=ps.device) if want_scores else None
        if n_rows:
            _lib.call("misa_merge_topk", ps.data_ptr(), pi.data_ptr(), P, ps.stride(0), n_rows, c, k_out,
                      out.data_ptr(), k_out, None if outs is None else outs.data_ptr(), self._stream())
        return out, outs


def merge_lists(ops, ps: torch.Tensor, pi: torch.Tensor, k_out: int) -> torch.Tensor:
    """Global top-k of (P, R, c) per-part lists: one merge when P*c fits a merge CTA,
    else rounds that merge groups of lists (keeping scores) until one list is left."""
    P, R, c = ps.shape
    while P * c > MERGE_CAPACITY:
        g = max(2, MERGE_CAPACITY // c)
        if c > MERGE_CAPACITY // 2:
            raise ValueError(f"list length {c} cannot be merged pairwise within {MERGE_CAPACITY}")
        ng = -(-P // g)
        ks = min(k_out, g * c)
        ns = torch.empty((ng, R, ks), dtype=torch.float32, device=ps.device)
        ni = torch.empty((ng, R, ks), dtype=torch.int32, device=ps.device)
        for j in range(ng):
            a, b = j * g, min(P, (j + 1) * g)
            oi, os_ = ops.merge(ps[a:b], pi[a:b], R, ks, want_scores=True)
            ni[j], ns[j] = oi, os_
        ps, pi, P, c = ns, ni, ng, ks
    out, _ = ops.merge(ps.contiguous(), pi.contiguous(), R, k_out)
    return out


class PrunedExchange:
    """Steps 4-6 of the module docstring for one (T_pad, kc) set of local lists."""

    def __init__(self, world: int, rank: int, group=None, ops=None, prune: bool = True):
        self.world, self.rank, self.group = world, rank, group
        self.ops = ops or DeviceListOps()
        self.prune = prune and world > 1
        self.last = {}

    def _pruned(self, loc_s, loc_i, kc):
        m, cap = prune_params(kc, self.world)
        tau = all_reduce_(self.ops.kth(loc_s, m), dist.ReduceOp.MIN, self.group)
        ps, pi, cnt = self.ops.prune(loc_s, loc_i, tau, cap)
        over = all_reduce_(cnt.clone(), dist.ReduceOp.MAX, self.group) > cap  # same on every rank
        return ps, pi, cap, over

    def _plain_rows(self, loc_i, loc_s, kc):
        pi, ps = exchange_by_rows(loc_i, loc_s, self.world, self.group)
        self.last = {"payload_rows": loc_i.shape[0], "cols": kc, "overflow_rows": 0}
        return merge_lists(self.ops, ps, pi, kc)

    def rows(self, loc_i: torch.Tensor, loc_s: torch.Tensor, kc: int) -> torch.Tensor:
        """(T_pad, kc) local lists -> merged (T_pad/world, kc) top-kc of this rank's rows."""
        G, r = self.world, self.rank
        T_pad = loc_i.shape[0]
        per = T_pad // G
        if not self.prune or prune_params(kc, G)[1] >= kc:
            return self._plain_rows(loc_i, loc_s, kc)
        ps, pi, cap, over = self._pruned(loc_s, loc_i, kc)
        gi, gs = exchange_by_rows(pi, ps, G, self.group)
        merged = merge_lists(self.ops, gs, gi, kc)
        over_rows = torch.nonzero(over).flatten()
        n_over = int(over_rows.numel())
        self.last = {"payload_rows": T_pad, "cols": cap, "overflow_rows": n_over}
        if n_over:
            # rows whose pruned list was truncated on some rank: their full lists, sent to
            # each row's owner (the overflow set is identical on every rank)
            owner = torch.div(over_rows, per, rounding_mode="floor")
            splits = torch.bincount(owner, minlength=G).cpu().tolist()
            mine = over_rows[owner == r]
            fi = all_to_all_rows(loc_i.index_select(0, over_rows), G, self.group, splits, [len(mine)] * G)
            fs = all_to_all_rows(loc_s.index_select(0, over_rows), G, self.group, splits, [len(mine)] * G)
            if len(mine):
                fix = merge_lists(self.ops, fs.view(G, len(mine), kc), fi.view(G, len(mine), kc), kc)
                merged.index_copy_(0, mine - r * per, fix)
        return merged

    def all_rows(self, loc_i: torch.Tensor, loc_s: torch.Tensor, kc: int) -> torch.Tensor:
        """(T, kc) local lists -> merged (T, kc) on every rank (decode)."""
        G = self.world
        if not self.prune or prune_params(kc, G)[1] >= kc:
            gi, gs = gather_lists(loc_i, loc_s, G, self.group)
            return merge_lists(self.ops, gs, gi, kc)
        ps, pi, cap, over = self._pruned(loc_s, loc_i, kc)
        gi, gs = gather_lists(pi, ps, G, self.group)
        merged = merge_lists(self.ops, gs, gi, kc)
        over_rows = torch.nonzero(over).flatten()
        if over_rows.numel():
            fi, fs = gather_lists(loc_i.index_select(0, over_rows), loc_s.index_select(0, over_rows), G,
                                  self.group)
            merged.index_copy_(0, over_rows, merge_lists(self.ops, fs, fi, kc))
        return merged


class ShardedIndexer:
    """Key-sharded DSA / MISA / MISA-dagger indexer for one rank of a ``torch.distributed`` group."""

    def __init__(self, method: str = "misa", *, world: int, rank: int, group=None, shard_block: int | None = None,
                 prune: bool = True, **engine_kwargs):
        if method not in ("dsa", "misa", "misa_hier"):
            raise ValueError(f"sharded execution supports 'dsa', 'misa' and 'misa_hier', got {method!r}")
        self.method = method
        self.world, self.rank, self.group = world, rank, group
        self.engine = IndexerEngine(method, **engine_kwargs)
        self.layout = KeyShardLayout(world, rank, shard_block or self.engine.B)
        self.k = self.engine.k
        kc = self.k if method != "misa_hier" else max(self.engine.kprime, self.k)
        if world > 1 and kc > MERGE_CAPACITY // 2:  # two lists must fit one merge CTA
            raise ValueError(f"candidate budget {kc} exceeds the sharded merge limit {MERGE_CAPACITY // 2}")
        self.exchange = PrunedExchange(world, rank, group, prune=prune)
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

    def _local_inputs(self, x: PreparedInputs) -> PreparedInputs:
        n_loc = self.layout.local_count(x.prefix_host)
        K_loc = self._local_keys(x)
        return PreparedInputs(K_loc, x.queries, x.weights, torch.from_numpy(n_loc.astype(np.int32)).to(x.keys.device),
                              n_loc, K_loc.shape[0], x.T, x.H, x.Hp, x.d, x.D, None)

    def run(self, keys, queries, weights, prefix_len=None, *, gather: bool = False):
        x = prepare_inputs(keys, queries, weights, prefix_len)
        G, r, k = self.world, self.rank, self.k
        dev = x.keys.device
        per, T_pad = row_slices(x.T, G)
        stream = torch.cuda.current_stream().cuda_stream

        heads, hq = None, x.Hp
        r0, r1 = min(x.T, r * per), min(x.T, (r + 1) * per)
        if self.method != "dsa":
            h_loc, hq, _ = self.engine.route(x.rows(r0, r1)) if r1 > r0 else (None, 8, None)
            buf = torch.full((per, hq), -1, dtype=torch.int32, device=dev)
            if r1 > r0:
                buf[: r1 - r0] = h_loc
            heads = all_gather_rows(buf, G, self.group).view(G * per, hq)[: x.T].contiguous()

        # local scoring against this shard's keys: top-kc with scores for every row
        xl = self._local_inputs(x)
        kc = k if self.method != "misa_hier" else max(self.engine.kprime, k)  # coarse budget
        loc_i = torch.full((T_pad, kc), -1, dtype=torch.int32, device=dev)
        loc_s = torch.full((T_pad, kc), float("-inf"), dtype=torch.float32, device=dev)
        self.last_fallback_rows = self.engine.select(xl, heads, hq, kc, loc_i[: x.T], tag="shard",
                                                     scores=loc_s[: x.T])
        _lib.call("misa_shard_map_indices", loc_i.data_ptr(), loc_i.numel(), self.layout.block, G, r, stream)

        merged = self.exchange.rows(loc_i, loc_s, kc)
        if self.method != "misa_hier":
            out = merged
        else:  # MISA-dagger fine stage on this rank's rows (dsa.py:95-115 on the merged candidates)
            out = torch.full((per, k), -1, dtype=torch.int32, device=dev)
            if r1 > r0:
                self.engine.refine(x.rows(r0, r1), merged[: r1 - r0], k, out[: r1 - r0])
        if gather:
            return all_gather_rows(out, G, self.group).view(G * per, k)[: x.T]
        return out

    def decode(self, keys, queries, weights, prefix_len=None, *, cache=None):
        """Decode step, key-sharded: every rank returns the global top-k of every row.

        ``keys`` / ``cache`` hold the replicated key set (the router needs every pooled
        block); each rank scores only its block-cyclic shard."""
        if cache is not None:
            keys = cache.keys[:cache.length, :cache.d]
        k = self.k
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
        xl = self._local_inputs(x)
        loc_i = torch.full((x.T, kc), -1, dtype=torch.int32, device=dev)
        loc_s = torch.full((x.T, kc), float("-inf"), dtype=torch.float32, device=dev)
        if xl.L > 0:
            eng.dense_select(xl, heads, hq, kc, loc_i, scores=loc_s)
        _lib.call("misa_shard_map_indices", loc_i.data_ptr(), loc_i.numel(), self.layout.block, self.world,
                  self.rank, stream)
        merged = self.exchange.all_rows(loc_i, loc_s, kc)
        if self.method != "misa_hier":
            return merged
        out = torch.empty((x.T, k), dtype=torch.int32, device=dev)
        eng.refine(x, merged, k, out)
        return out
