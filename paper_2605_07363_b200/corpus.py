"""Archived workload corpora (MISAWKLD v1, ``workload.py:202-254``) -> one batched device call.

The reference archives corpora as one MISAWKLD file per single-query workload
(``cli.py:305-316`` ``_save_corpus``: ``workload_L{L}_d{di}_r{rep}_s{seed}.bin``) and replays a
file through ``load_workload`` + ``indexer.select`` (``cli.py:319-330``), one query at a time on
the CPU.  Here a whole corpus becomes one varlen batch: every workload is a sequence of L_s keys
with one query row at prefix L_s, packed at block-aligned offsets
(``engine.prepare_varlen`` layout).  The f64 payloads are uploaded as stored (pinned staging)
and rounded to bf16 on the device straight into that layout (``misa_pack_rows_f64``), which
also reports whether any value was not bf16-representable.

``select_corpus(indexer, corpus)`` returns, per workload, the ``SelectionResult`` that
``indexer.select(load_workload(path))`` returns (selection, heads, candidates, ledger), from a
single engine call for the whole corpus.
"""

from __future__ import annotations

import math
import os
import re
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .config import BLOCK_ATTENTION
from .engine import IndexerOutput, PreparedInputs, SeqLayout, head_dim_pad, heads_pad
from .routing import _ledger
from .types import CostEntry, CostLedger, HeadSet, SelectionResult, TokenSelection
from .workload import _HEADER, FORMAT_VERSION, MAGIC, IndexerWorkload, load_workload, save_workload

_NAME = re.compile(r"workload_L(\d+)_d(\d+)_r(\d+)_s(\d+)\.bin$")


@dataclass(frozen=True)
class CorpusEntry:
    path: str
    prefix_len: int
    head_dim: int
    n_heads: int
    seed: int | None  # parsed from the reference's file name, when it follows it


def read_header(path) -> tuple[int, int, int]:
    """(prefix_len, head_dim, n_heads) of a MISAWKLD file, validated exactly as
    ``load_workload`` validates it (same errors), without reading the payload."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        raw = f.read(_HEADER.size)
    if len(raw) < _HEADER.size:
        raise ValueError("workload file too short for header")
    magic, version, L, d, H = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise ValueError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != FORMAT_VERSION:
        raise ValueError(f"unsupported workload format version {version}")
    expected = _HEADER.size + 8 * (L * d + H * d + H)
    if size != expected:
        raise ValueError(f"workload file has {size} bytes, expected {expected}")
    if L < 1:
        raise ValueError("prefix must contain at least one key")
    return int(L), int(d), int(H)


class Corpus:
    """An ordered set of MISAWKLD files of one (n_heads, head_dim) shape."""

    def __init__(self, paths):
        paths = [str(p) for p in paths]
        if not paths:
            raise ValueError("empty corpus")
        entries = []
        for p in paths:
            L, d, H = read_header(p)
            m = _NAME.search(os.path.basename(p))
            entries.append(CorpusEntry(p, L, d, H, int(m.group(4)) if m else None))
        shapes = {(e.n_heads, e.head_dim) for e in entries}
        if len(shapes) != 1:
            raise ValueError(f"corpus mixes (n_heads, head_dim) shapes {sorted(shapes)}")
        self.entries = entries
        self.n_heads, self.head_dim = shapes.pop()

    @classmethod
    def open(cls, source) -> "Corpus":
        """A directory (every ``*.bin``, sorted by name) or an explicit list of files."""
        if isinstance(source, (str, Path)) and Path(source).is_dir():
            return cls(sorted(str(p) for p in Path(source).glob("*.bin")))
        if isinstance(source, (str, Path)):
            return cls([source])
        return cls(list(source))

    def __len__(self) -> int:
        return len(self.entries)

    def workload(self, i: int) -> IndexerWorkload:
        """The reference's view of file i (``load_workload``: seed 0, no label)."""
        return load_workload(self.entries[i].path)

    # ------------------------------------------------------------ device batch
    def to_device(self, block_size: int, device="cuda") -> "CorpusBatch":
        """Pack every workload for one varlen engine call (see module docstring)."""
        dev = torch.device(device)
        S, H, d = len(self.entries), self.n_heads, self.head_dim
        D, Hp = head_dim_pad(d), heads_pad(H)
        lens = np.array([e.prefix_len for e in self.entries], np.int64)
        align = math.lcm(int(block_size), 128)
        padded = -(-lens // align) * align
        key0 = np.concatenate([[0], np.cumsum(padded)[:-1]]).astype(np.int64)
        keys = torch.zeros(int(padded.sum()), D, dtype=torch.bfloat16, device=dev)
        queries = torch.zeros(S, Hp, D, dtype=torch.bfloat16, device=dev)
        weights = torch.zeros(S, Hp, dtype=torch.float32, device=dev)
        inexact = torch.zeros(1, dtype=torch.int64, device=dev)   # keys / queries not bf16-exact
        bad = torch.zeros((), dtype=torch.int64, device=dev)      # non-finite values
        gates_inexact = torch.zeros((), dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream()
        # double-buffered pinned staging of the f64 payloads; the device rounds them into place
        cap = int(max(lens.max() * d + H * d + H, 1))
        stage = [torch.empty(cap, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        dstage = [torch.empty(cap, dtype=torch.float64, device=dev) for _ in range(2)]
        done = [None, None]
        for s, e in enumerate(self.entries):
            b = s % 2
            if done[b] is not None:
                done[b].synchronize()  # the copy out of staging buffer b has been consumed
            n = e.prefix_len * d + H * d + H
            with open(e.path, "rb") as f:
                f.seek(_HEADER.size)
                f.readinto(memoryview(stage[b].numpy()[:n]).cast("B"))
            src = dstage[b]
            src[:n].copy_(stage[b][:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            done[b] = ev
            _lib.call("misa_pack_rows_f64", src.data_ptr(), e.prefix_len, d, e.prefix_len, e.prefix_len,
                      keys.data_ptr(), D, int(key0[s]), inexact.data_ptr(), stream.cuda_stream)
            _lib.call("misa_pack_rows_f64", src.data_ptr() + 8 * e.prefix_len * d, H, d, H, Hp,
                      queries.data_ptr(), D, s * Hp, inexact.data_ptr(), stream.cuda_stream)
            g = src[e.prefix_len * d + H * d: n]
            weights[s, :H].copy_(g)
            gates_inexact += (g.float().double() != g).sum()
            bad += (~torch.isfinite(src[:n])).sum()
        if int(bad.item()):  # IndexerWorkload's check (workload.py:71-73)
            raise ValueError("corpus workloads must contain only finite values")
        prefix = torch.from_numpy(lens.astype(np.int32)).to(dev)
        seq = SeqLayout(torch.from_numpy(key0.astype(np.int32)).to(dev), key0, align, int(block_size))
        x = PreparedInputs(keys, queries, weights, prefix, lens, int(lens.max()), S, H, Hp, d, D, None, None, seq)
        n_inexact = int(inexact.item())
        return CorpusBatch(self, x, n_inexact == 0 and int(gates_inexact.item()) == 0, n_inexact)


@dataclass
class CorpusBatch:
    corpus: Corpus
    inputs: PreparedInputs
    bf16_exact: bool
    n_inexact: int  # key / query elements that bf16 does not represent


def save_corpus(workloads, directory, names=None) -> list[str]:
    """Write workloads as MISAWKLD files (``save_workload``); default names follow the
    reference's ``workload_L{L}_d0_r{i}_s{seed}.bin``."""
    target = Path(directory)
    target.mkdir(parents=True, exist_ok=True)
    out = []
    for i, w in enumerate(workloads):
        name = names[i] if names is not None else f"workload_L{w.prefix_len}_d0_r{i}_s{w.seed}.bin"
        save_workload(w, target / name)
        out.append(str(target / name))
    return out


def _results(indexer, batch: CorpusBatch, res: IndexerOutput) -> list[SelectionResult]:
    x = batch.inputs
    k = indexer.budget_k
    topk = res.topk.cpu().numpy()
    heads = None if res.heads is None else res.heads.cpu().numpy()
    cand = None if res.candidates is None else res.candidates.cpu().numpy()
    out = []
    for s, e in enumerate(batch.corpus.entries):
        L = e.prefix_len
        o = topk[s]
        sel = TokenSelection(o[o >= 0].astype(np.int64), k, L)
        if indexer.method == "dsa":
            ledger = CostLedger((CostEntry("token_scan", "token", e.n_heads * L),))
            out.append(SelectionResult(selection=sel, ledger=ledger))
            continue
        hh = heads[s]
        hs = HeadSet(hh[hh >= 0].astype(np.int64), e.n_heads)
        w = _Shape(L, e.n_heads)
        m_blocks = -(-L // indexer.block_size)
        if indexer.method == "misa":
            out.append(SelectionResult(selection=sel, ledger=_ledger(w, m_blocks, len(hs), indexer.router_score),
                                       heads=hs))
            continue
        c = cand[s]
        cs = TokenSelection(np.sort(c[c >= 0]).astype(np.int64), indexer.candidate_kprime, L)
        ledger = _ledger(w, m_blocks, len(hs), indexer.router_score, refine=e.n_heads * len(cs))
        out.append(SelectionResult(selection=sel, ledger=ledger, heads=hs, candidates=cs))
    return out


@dataclass(frozen=True)
class _Shape:  # what routing._ledger reads from a workload
    prefix_len: int
    n_heads: int


def select_corpus(indexer, corpus, *, batch: CorpusBatch | None = None) -> list[SelectionResult]:
    """Per-workload ``indexer.select(workload)`` results for a whole corpus, one device call."""
    if not isinstance(corpus, Corpus):
        corpus = Corpus.open(corpus)
    indexer.fit()
    block = getattr(indexer, "block_size", 1024)
    if batch is None:
        batch = corpus.to_device(block)
    eng = indexer.engine()
    res = eng.run_prepared(batch.inputs)
    return _results(indexer, batch, res)


__all__ = ["Corpus", "CorpusBatch", "CorpusEntry", "read_header", "save_corpus", "select_corpus"]
