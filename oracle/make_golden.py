"""Generate golden vectors by running the REFERENCE package itself — TEST INFRASTRUCTURE.

Run in the build container (where ``/root/reference`` exists):

    python oracle/make_golden.py

It imports ``misa`` from ``/root/reference/pkg/src`` (read-only; never copied),
runs the reference estimators / pure functions on seeded, bf16-rounded batched
causal inputs, and writes ``tests/golden/*.npz``.  The committed fixtures pin
both the numpy oracle (``oracle/misa_oracle.py``) and the CUDA path; the GPU
box never reads ``/root/reference``.

Row t of every batched case is the reference run on
``IndexerWorkload(keys=K[:n_t], queries=Q[t], gate_weights=W[t])`` with
``n_t = t + 1`` (causal prefill), the ``truncated()`` semantics of
``workload.py:91-110``.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import misa  # noqa: E402  (the reference package)
from misa_oracle import synthetic_prefill  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")

# name: (seed, L, H, d, h, B, k, kprime, raw_gates, rows or None=all)
CASES = {
    "tiny_softmax": (1, 96, 8, 16, 3, 8, 12, 24, False, None),
    "tiny_signed": (2, 64, 6, 20, 2, 5, 7, 15, True, None),
    "small_h64": (3, 300, 64, 32, 8, 32, 40, 96, False, None),
    "glm_h32": (4, 512, 32, 64, 8, 64, 64, 160, False, None),
    # C1: the BASELINE.json configs[0] shape, sampled rows (inputs regenerated from seed).
    "c1_sampled": (0, 4096, 64, 128, 8, 64, 2048, 8192, False,
                   [0, 1, 62, 63, 64, 65, 511, 1000, 2046, 2047, 2048, 2049, 3000, 4095]),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_case(name, seed, L, H, d, h, B, k, kprime, raw, rows):
    K, Q, W = synthetic_prefill(seed, L, H, d, raw_gates=raw)
    rows = list(range(L)) if rows is None else rows
    R = len(rows)
    out = {
        "meta": np.array([seed, L, H, d, h, B, k, kprime, int(raw)], np.int64),
        "rows": np.array(rows, np.int64),
        "sha_K": np.array(sha(K)), "sha_Q": np.array(sha(Q)), "sha_W": np.array(sha(W)),
    }
    store_inputs = L * d <= 64 * 1024
    if store_inputs:
        out.update(K=K, Q=Q, W=W)
    for prec in ("fast32", "reference64"):
        dsa_sel = np.full((R, k), -1, np.int64)
        misa_sel = np.full((R, k), -1, np.int64)
        hier_sel = np.full((R, k), -1, np.int64)
        hier_cand = np.full((R, kprime), -1, np.int64)
        heads = np.full((R, h), -1, np.int64)
        imp = np.zeros((R, H))
        ledgers = np.zeros((R, 3, 3), np.int64)  # method x (token, block, refine)
        for i, t in enumerate(rows):
            n = t + 1
            w = misa.IndexerWorkload(keys=K[:n], queries=Q[t], gate_weights=W[t], seed=seed)
            r_d = misa.DSAIndexer(budget_k=k, precision_mode=prec).select(w)
            r_m = misa.MISAIndexer(budget_k=k, active_heads_h=h, block_size=B, precision_mode=prec).select(w)
            r_h = misa.HierarchicalMISAIndexer(budget_k=k, active_heads_h=h, block_size=B,
                                              candidate_kprime=kprime, precision_mode=prec).select(w)
            for arr, res in ((dsa_sel, r_d), (misa_sel, r_m), (hier_sel, r_h)):
                idx = res.selection.indices
                arr[i, : idx.shape[0]] = idx
            c = r_h.candidates.indices
            hier_cand[i, : c.shape[0]] = c
            heads[i, : len(r_m.heads)] = r_m.heads.head_indices
            summary = misa.build_block_summary(w.keys, B)
            imp[i] = misa.route_head_importance(w, summary, precision=prec).values
            for j, res in enumerate((r_d, r_m, r_h)):
                lg = res.ledger
                ledgers[i, j] = (lg.token_dot_products, lg.block_dot_products, lg.refine_dot_products)
        out[f"{prec}_dsa"] = dsa_sel
        out[f"{prec}_misa"] = misa_sel
        out[f"{prec}_hier"] = hier_sel
        out[f"{prec}_hier_cand"] = hier_cand
        out[f"{prec}_heads"] = heads
        out[f"{prec}_importance"] = imp
        out[f"{prec}_ledger"] = ledgers
        if prec == "fast32" and L <= 600:
            # dense per-row scores of the last row (all heads, routed heads) for score tolerance tests
            t = rows[-1]
            w = misa.IndexerWorkload(keys=K[: t + 1], queries=Q[t], gate_weights=W[t], seed=seed)
            out["fast32_last_dsa_scores"] = misa.dsa_score(w, precision=prec).values
            hs = misa.HeadSet(head_indices=heads[-1][heads[-1] >= 0], n_heads=H)
            out["fast32_last_misa_scores"] = misa.misa_score(w, hs, precision=prec).values
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"[golden] {name}: L={L} H={H} d={d} rows={R} inputs_stored={store_inputs}")


def pooling_and_needles():
    """Pooling / incremental-append goldens and reference needle workloads."""
    rng = np.random.default_rng(11)
    keys = rng.standard_normal((37, 5))
    out = {"keys": keys}
    for B in (1, 4, 8, 64):
        s = misa.build_block_summary(keys, B)
        out[f"bounds_{B}"] = s.boundaries
        out[f"pooled_{B}"] = s.pooled_keys
    # incremental from empty, B=4
    s = misa.build_block_summary(np.empty((0, 5)), 4)
    for row in keys:
        s = misa.incremental_append(s, row)
    out["incr_bounds_4"] = s.boundaries
    out["incr_pooled_4"] = s.pooled_keys
    np.savez_compressed(os.path.join(OUT, "pooling.npz"), **out)

    cfg = misa.IndexerConfig()  # H=64, d=64, k=2048, B=1024, h=8
    nd = {}
    specs = [(7, 2048, 0.5, None), (8, 4096, 0.1, 5), (9, 4096, 0.9, None)]
    for i, (seed, L, depth, align) in enumerate(specs):
        w = misa.gen_needle_workload(seed, L, depth, 32, 10.0, cfg, noise_scale=0.01, align_head=align)
        k = min(cfg.budget_k, L // 4)
        nd[f"spec{i}"] = np.array([seed, L, depth, -1 if align is None else align], np.float64)
        nd[f"sha{i}"] = np.array(sha(w.keys) + sha(w.queries) + sha(w.gate_weights))
        nd[f"label{i}"] = np.array([w.label.start, w.label.length, w.label.aligned_head])
        nd[f"k{i}"] = np.array(k)
        for prec in ("reference64", "fast32"):
            nd[f"{prec}_dsa{i}"] = misa.DSAIndexer(budget_k=k, precision_mode=prec).select(w).selection.indices
            r = misa.MISAIndexer(budget_k=k, precision_mode=prec).select(w)
            nd[f"{prec}_misa{i}"] = r.selection.indices
            nd[f"{prec}_heads{i}"] = r.heads.head_indices
    np.savez_compressed(os.path.join(OUT, "needles.npz"), **nd)
    print("[golden] pooling + needles")


def archived_corpus():
    """A small MISAWKLD corpus written by the REFERENCE's own save_workload (tests/golden/corpus/),
    with the reference estimators' selections on it (fast32 and reference64).  Values are
    bf16-rounded before saving (the device contract is exact on them); the needle workload
    keeps the reference generator's layout."""
    cdir = os.path.join(OUT, "corpus")
    os.makedirs(cdir, exist_ok=True)
    for f in os.listdir(cdir):
        os.remove(os.path.join(cdir, f))
    cfg = misa.IndexerConfig(n_heads=16, head_dim=32, budget_k=128, block_size=128, active_heads_h=4,
                             candidate_kprime=512)
    bf = lambda a: np.asarray(torch.from_numpy(np.asarray(a)).to(torch.bfloat16).double())  # noqa: E731
    specs = [("random", 21, 300), ("random", 22, 900), ("needle", 23, 1800), ("random", 24, 2100)]
    names, out = [], {}
    for i, (kind, seed, L) in enumerate(specs):
        if kind == "random":
            w = misa.gen_random_workload(seed, L, cfg)
        else:
            w = misa.gen_needle_workload(seed, L, 0.4, 32, 10.0, cfg, noise_scale=0.01)
        w = misa.IndexerWorkload(keys=bf(w.keys), queries=bf(w.queries),
                                 gate_weights=np.asarray(w.gate_weights, np.float32).astype(np.float64), seed=seed)
        name = f"workload_L{L}_d0_r{i}_s{seed}.bin"
        misa.save_workload(w, os.path.join(cdir, name))
        names.append(name)
        for prec in ("fast32", "reference64"):
            kw = dict(budget_k=cfg.budget_k, precision_mode=prec)
            rk = dict(kw, active_heads_h=cfg.active_heads_h, block_size=cfg.block_size)
            r_d = misa.DSAIndexer(**kw).select(w)
            r_m = misa.MISAIndexer(**rk).select(w)
            r_h = misa.HierarchicalMISAIndexer(**rk, candidate_kprime=cfg.candidate_kprime).select(w)
            out[f"{prec}_dsa{i}"] = r_d.selection.indices
            out[f"{prec}_misa{i}"] = r_m.selection.indices
            out[f"{prec}_heads{i}"] = r_m.heads.head_indices
            out[f"{prec}_hier{i}"] = r_h.selection.indices
            out[f"{prec}_hier_cand{i}"] = r_h.candidates.indices
            for tag, r in (("dsa", r_d), ("misa", r_m), ("hier", r_h)):
                lg = r.ledger
                out[f"{prec}_ledger_{tag}{i}"] = np.array(
                    [lg.token_dot_products, lg.block_dot_products, lg.refine_dot_products], np.int64)
    out["names"] = np.array(names)
    out["cfg"] = np.array([cfg.n_heads, cfg.head_dim, cfg.budget_k, cfg.block_size, cfg.active_heads_h,
                           cfg.candidate_kprime], np.int64)
    np.savez_compressed(os.path.join(cdir, "reference_selections.npz"), **out)
    print(f"[golden] corpus: {len(names)} MISAWKLD files")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    only = sys.argv[1:]
    for name, args in CASES.items():
        if not only or name in only:
            run_case(name, *args)
    if not only or "pooling" in only:
        pooling_and_needles()
    if not only or "corpus" in only:
        archived_corpus()
