"""Key-sharded (multi-GPU) host logic on CPU: shard layout math and the gloo world_size-2
exchange + merge pipeline, with the oracle standing in for the per-rank local top-k."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import misa_oracle as O
from paper_2605_07363_b200 import sharded as S
from paper_2605_07363_b200.sharded import KeyShardLayout, exchange_by_rows, row_slices


@pytest.mark.parametrize("G,B,L", [(2, 16, 100), (4, 8, 257), (8, 1024, 20000), (3, 5, 1)])
def test_layout_partitions_keys(G, B, L):
    owned = [KeyShardLayout(G, r, B).local_keys(L) for r in range(G)]
    allk = np.sort(np.concatenate(owned))
    assert allk.tolist() == list(range(L))  # disjoint cover
    for r in range(G):
        lay = KeyShardLayout(G, r, B)
        loc = owned[r]
        assert np.all(np.diff(loc) > 0)
        assert lay.to_global(np.arange(loc.shape[0])).tolist() == loc.tolist()  # monotone map
        ns = np.arange(0, L + 1)
        brute = np.searchsorted(loc, ns, side="left")  # local keys with global index < n
        assert lay.local_count(ns).tolist() == brute.tolist()
    # block-cyclic balance of causal work: per-rank sum of local prefix lengths
    work = [KeyShardLayout(G, r, B).local_count(np.arange(1, L + 1)).sum() for r in range(G)]
    if L >= 8 * G * B:
        assert max(work) / max(1, min(work)) < 1.3


def _merge_np(parts_i, parts_s, k):
    """Reference merge: union of the per-rank lists, (score desc, index asc), ascending output."""
    out = np.full((parts_i.shape[1], k), -1, np.int64)
    for t in range(parts_i.shape[1]):
        pairs = [(float(parts_s[p, t, j]), int(parts_i[p, t, j]))
                 for p in range(parts_i.shape[0]) for j in range(parts_i.shape[2]) if parts_i[p, t, j] >= 0]
        pairs.sort(key=lambda x: (-x[0], x[1]))
        sel = sorted(i for _, i in pairs[:k])
        out[t, : len(sel)] = sel
    return out


def _worker(rank, world, port, L, H, d, k, B, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, Q, W = O.synthetic_prefill(77, L, H, d)
        lay = KeyShardLayout(world, rank, B)
        loc = lay.local_keys(L)
        n_loc = lay.local_count(np.arange(1, L + 1))
        per, T_pad = row_slices(L, world)
        li = np.full((T_pad, k), -1, np.int64)
        ls = np.full((T_pad, k), -np.inf)
        for t in range(L):
            if n_loc[t] == 0:
                continue
            keys = K[loc[: n_loc[t]]]
            sc = O.gated_relu_scores(keys, Q[t], W[t], "fast32")
            sel = O.topk_tokens(sc, k)  # local indices, ascending
            li[t, : sel.shape[0]] = lay.to_global(sel)
            ls[t, : sel.shape[0]] = sc[sel]
        pi, ps = exchange_by_rows(torch.from_numpy(li), torch.from_numpy(ls), world)
        got = _merge_np(pi.numpy(), ps.numpy(), k)
        ok = True
        for j in range(per):
            t = rank * per + j
            if t >= L:
                continue
            ref = O.dsa_select(K[: t + 1], Q[t], W[t], k, "fast32")["selection"]
            row = got[j][got[j] >= 0]
            ok &= row.tolist() == ref.tolist()
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_exchange_and_merge_equal_dense(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    L, H, d, k, B = 300, 8, 16, 24, 16
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, H, d, k, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def _decode_worker(rank, world, port, L, H, d, k, B, q):
    """Decode exchange: every rank all-gathers the (T, k) local lists and merges every row."""
    from paper_2605_07363_b200.sharded import gather_lists
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, Q, W = O.synthetic_prefill(91, L, H, d)
        T = 5
        rows = np.arange(L - T, L)  # decode rows see (almost) the whole prefix
        lay = KeyShardLayout(world, rank, B)
        loc = lay.local_keys(L)
        li = np.full((T, k), -1, np.int64)
        ls = np.full((T, k), -np.inf)
        for j, t in enumerate(rows):
            n_loc = int(lay.local_count(t + 1))
            if n_loc == 0:
                continue
            sc = O.gated_relu_scores(K[loc[:n_loc]], Q[t], W[t], "fast32")
            sel = O.topk_tokens(sc, k)
            li[j, : sel.shape[0]] = lay.to_global(sel)
            ls[j, : sel.shape[0]] = sc[sel]
        gi, gs = gather_lists(torch.from_numpy(li), torch.from_numpy(ls), world)
        got = _merge_np(gi.numpy(), gs.numpy(), k)
        ok = True
        for j, t in enumerate(rows):
            ref = O.dsa_select(K[: t + 1], Q[t], W[t], k, "fast32")["selection"]
            row = got[j][got[j] >= 0]
            ok &= row.tolist() == ref.tolist()
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_sharded_decode_gather_and_merge_equal_dense():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, L, H, d, k, B = 2, 400, 8, 16, 24, 16
    port = _free_port()
    procs = [ctx.Process(target=_decode_worker, args=(r, world, port, L, H, d, k, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


class HostListOps:
    """Host stand-ins for the list kernels (misa_list_kth / misa_list_prune / misa_merge_topk),
    so the CPU test drives the product's PrunedExchange (collectives, pruning, overflow
    re-exchange, merge rounds) unchanged."""

    def kth(self, s, m):
        out = torch.full((s.shape[0],), float("-inf"))
        for r in range(s.shape[0]):
            v = s[r][s[r] > float("-inf")]
            if v.numel() >= m:
                out[r] = torch.sort(v, descending=True).values[m - 1]
        return out

    def prune(self, s, i, tau, cap):
        R = s.shape[0]
        os_ = torch.full((R, cap), float("-inf"))
        oi = torch.full((R, cap), -1, dtype=torch.int32)
        cnt = torch.zeros(R, dtype=torch.int32)
        for r in range(R):
            keep = torch.nonzero((i[r] >= 0) & (s[r] >= tau[r])).flatten()
            cnt[r] = keep.numel()
            keep = keep[:cap]
            os_[r, : keep.numel()] = s[r, keep]
            oi[r, : keep.numel()] = i[r, keep]
        return os_, oi, cnt

    def merge(self, ps, pi, n_rows, k_out, want_scores=False):
        out = torch.full((n_rows, k_out), -1, dtype=torch.int32)
        outs = torch.full((n_rows, k_out), float("-inf"))
        for t in range(n_rows):
            pairs = [(float(ps[p, t, j]), int(pi[p, t, j])) for p in range(ps.shape[0])
                     for j in range(ps.shape[2]) if pi[p, t, j] >= 0]
            pairs.sort(key=lambda x: (-x[0], x[1]))
            sel = sorted(pairs[:k_out], key=lambda x: x[1])
            out[t, : len(sel)] = torch.tensor([i for _, i in sel], dtype=torch.int32)
            outs[t, : len(sel)] = torch.tensor([v for v, _ in sel])
        return out, outs if want_scores else None


def _pruned_worker(rank, world, port, L, H, d, k, B, merge_cap, q):
    """Local top-k lists from the oracle -> the product's PrunedExchange over gloo (prefill
    row exchange and decode all-gather) == the dense selection, with pruning active,
    overflow rows re-exchanged and, with a small merge capacity, merge rounds."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S.MERGE_CAPACITY = merge_cap
        K, Q, W = O.synthetic_prefill(78, L, H, d)
        lay = KeyShardLayout(world, rank, B)
        loc = lay.local_keys(L)
        n_loc = lay.local_count(np.arange(1, L + 1))
        per, T_pad = row_slices(L, world)
        li = torch.full((T_pad, k), -1, dtype=torch.int32)
        ls = torch.full((T_pad, k), float("-inf"))
        for t in range(L):
            if n_loc[t] == 0:
                continue
            sc = O.gated_relu_scores(K[loc[: n_loc[t]]], Q[t], W[t], "fast32")
            sel = O.topk_tokens(sc, k)
            li[t, : sel.shape[0]] = torch.from_numpy(lay.to_global(sel).astype(np.int32))
            ls[t, : sel.shape[0]] = torch.from_numpy(sc[sel].astype(np.float32))
        ex = S.PrunedExchange(world, rank, ops=HostListOps())
        merged = ex.rows(li, ls, k)
        stats = dict(ex.last)
        ok = True
        for j in range(per):
            t = rank * per + j
            if t >= L:
                continue
            ref = O.topk_tokens(O.gated_relu_scores(K[: t + 1], Q[t], W[t], "fast32").astype(np.float32), k)
            row = merged[j][merged[j] >= 0].numpy()
            ok &= row.tolist() == ref.tolist()
        dec_rows = np.arange(L - 6, L)
        md = ex.all_rows(li[dec_rows], ls[dec_rows], k)
        for j, t in enumerate(dec_rows):
            ref = O.topk_tokens(O.gated_relu_scores(K[: t + 1], Q[t], W[t], "fast32").astype(np.float32), k)
            ok &= md[j][md[j] >= 0].numpy().tolist() == ref.tolist()
        q.put((rank, (bool(ok), stats)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,merge_cap", [(2, 16384), (3, 192)])
def test_gloo_pruned_exchange_equals_dense(world, merge_cap):
    """The pruned key-shard exchange (tau = min over ranks of the (k/G)-th local score,
    prune, all-to-all, overflow rows unpruned, merge rounds when G*cap > capacity) selects
    exactly the dense top-k (scores rounded to f32 on both sides, as the kernels emit)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    L, H, d, k, B = 300, 8, 16, 96, 64
    port = _free_port()
    procs = [ctx.Process(target=_pruned_worker, args=(r, world, port, L, H, d, k, B, merge_cap, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=150) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v[0] for v in res.values()), res
    st = res[0][1]
    assert st["cols"] < k  # pruned lists are shorter than the local top-k
    if world == 3:  # early rows (< m keys on some rank: no bound) overflow the cap on rank 0 -> unpruned
        assert 0 < st["overflow_rows"] < L


def test_prune_bound_is_sound():
    """min over shards of the ceil(k/G)-th local score never exceeds the global k-th score."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        G = int(rng.integers(2, 9))
        k = int(rng.integers(1, 64))
        parts = [np.round(rng.standard_normal(int(rng.integers(0, 80))), 1) for _ in range(G)]
        allv = np.concatenate(parts)
        if allv.size < k:
            continue
        m, cap = S.prune_params(k, G)
        taus = [np.sort(p)[::-1][m - 1] if p.size >= m else -np.inf for p in parts]
        assert min(taus) <= np.sort(allv)[::-1][k - 1]
        assert m <= cap <= k
