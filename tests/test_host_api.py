"""CPU-only tests: the C-ABI library surface, host-side logic and the reference-mirroring API."""

import io
import os
import re

import numpy as np
import pytest
from sklearn.base import clone

from oracle import misa_oracle as O

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(REPO, "include", "misa_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(misa_\w+)\(", src, re.M)))


def test_abi_library_exports_every_header_symbol():
    from paper_2605_07363_b200 import _build, _lib
    if not os.path.exists(_build.LIB):
        _build.build()
    lib = _lib.load()
    names = _header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES or n in _lib.EXTRA, f"{n} not typed in _lib"
    assert lib.misa_abi_version() == 2
    # argument validation happens before any device work: a bad shape is EINVAL -> ValueError
    with pytest.raises(ValueError):
        _lib.call("misa_pool_keys", None, 10, 128, 4, None, None, None, 0, None)
    with pytest.raises(ValueError):
        _lib.call("misa_select_topk", None, None, 4, None, 1, 8, 0, None, 8, None, None, None)


def test_sass_contains_tcgen05_and_tma():
    """The shipped library carries tcgen05 MMAs, TMEM loads, TMA and cp.async gathers in SASS."""
    import shutil
    import subprocess
    from paper_2605_07363_b200 import _build
    if not os.path.exists(_build.LIB):
        _build.build()
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _build.LIB], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG", "LDGSTS"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2605_07363_b200 import DSAIndexer, IndexerWorkload
    K, Q, W = O.synthetic_prefill(0, 64, 8, 16, T=1)
    with pytest.raises((RuntimeError, AssertionError)):
        DSAIndexer(budget_k=8).select(IndexerWorkload(K, Q[0], W[0]))


def test_config_and_types_mirror_reference():
    from paper_2605_07363_b200 import (IndexerConfig, TokenSelection, HeadSet, ScoreVector, CostEntry, CostLedger,
                                       REFERENCE64, FAST32, dtype_for)
    cfg = IndexerConfig()
    assert (cfg.n_heads, cfg.active_heads_h, cfg.budget_k, cfg.candidate_kprime, cfg.block_size, cfg.head_dim) == \
        (64, 8, 2048, 8192, 1024, 64)
    for bad in (dict(active_heads_h=65), dict(candidate_kprime=100), dict(block_size=0),
                dict(precision_mode="float16"), dict(hisa_block_m=0)):
        with pytest.raises(ValueError):
            IndexerConfig(**bad)
    assert IndexerConfig().resolved_hisa_m(128) == 32
    assert dtype_for(REFERENCE64) == np.float64 and dtype_for(FAST32) == np.float32
    with pytest.raises(ValueError):
        TokenSelection(np.array([3, 1]), 4, 10)
    with pytest.raises(ValueError):
        TokenSelection(np.array([0, 1, 2]), 2, 10)
    sel = TokenSelection(np.array([1, 5]), 2, 10)
    assert 5 in sel and 4 not in sel
    with pytest.raises(ValueError):
        sel.indices[0] = 9
    with pytest.raises(ValueError):
        HeadSet(np.array([0, 4]), 4)
    with pytest.raises(ValueError):
        ScoreVector(np.array([1.0, np.nan]), "token")
    with pytest.raises(ValueError):
        CostEntry("x", "flops", 1)
    led = CostLedger((CostEntry("router", "block", 3), CostEntry("token_scan", "token", 5)))
    assert led.total() == 8 and led.stage_labels == ("router", "token_scan")


def test_estimator_surface():
    from paper_2605_07363_b200 import (METHODS, make_indexer, MISAIndexer, HierarchicalMISAIndexer, DSAIndexer)
    assert METHODS == ("dsa", "misa", "misa_hier")
    for m in METHODS:
        est = make_indexer(m)
        params = est.get_params()
        assert type(est)(**params).get_params() == params
        assert clone(est).get_params() == params
    assert (MISAIndexer().budget_k, MISAIndexer().active_heads_h, MISAIndexer().block_size) == (2048, 8, 1024)
    assert HierarchicalMISAIndexer().candidate_kprime == 8192
    swept = [clone(MISAIndexer(budget_k=8)).set_params(active_heads_h=h) for h in (1, 2, 4)]
    assert [e.active_heads_h for e in swept] == [1, 2, 4]
    assert DSAIndexer(budget_k=8).fit() is not None
    with pytest.raises(ValueError):
        DSAIndexer(budget_k=0).fit()
    with pytest.raises(ValueError):
        make_indexer("block_sparse")


def test_workload_generators_match_reference_generators():
    from paper_2605_07363_b200 import IndexerConfig, gen_needle_workload, gen_random_workload, save_workload, \
        load_workload
    cfg = IndexerConfig(n_heads=16, head_dim=32)
    w = gen_needle_workload(3, 256, 0.5, 8, 10.0, cfg, align_head=5)
    K, Q, W, label = O.needle_workload(3, 256, 0.5, 8, 10.0, 16, 32, align_head=5)
    assert np.array_equal(w.keys, K) and np.array_equal(w.queries, Q) and np.array_equal(w.gate_weights, W)
    assert (w.label.start, w.label.length, w.label.aligned_head) == label
    r = gen_random_workload(7, 16, IndexerConfig(n_heads=4, head_dim=4, active_heads_h=2))
    assert abs(r.gate_weights.sum() - 1) < 1e-12
    buf = io.BytesIO()
    save_workload(r, buf)
    back = load_workload(io.BytesIO(buf.getvalue()))
    assert np.array_equal(back.keys, r.keys) and np.array_equal(back.gate_weights, r.gate_weights)
    with pytest.raises(ValueError):
        load_workload(io.BytesIO(b"NOTMAGIC" + buf.getvalue()[8:]))
    t = w.truncated(100)
    assert t.prefix_len == 100 and t.label is None


def test_work_lists():
    from paper_2605_07363_b200.engine import IndexerEngine, heads_pad, heads_per_query, head_dim_pad
    assert (heads_pad(6), heads_pad(64), heads_pad(33)) == (8, 64, 64)
    assert (heads_per_query(3), heads_per_query(8), heads_per_query(9)) == (8, 8, 16)
    assert (head_dim_pad(20), head_dim_pad(128)) == (64, 128)
    with pytest.raises(ValueError):
        head_dim_pad(129)
    lens = np.arange(1, 1001)
    items, tiles = IndexerEngine.group_items(lens, 32, 1, 100)
    # groups whose longest row exceeds 100, longest first, tiles = ceil(max/128)
    assert tiles.tolist() == sorted(tiles.tolist(), reverse=True)
    for g, nt in zip(items.tolist(), tiles.tolist()):
        assert nt == -(-int(lens[g * 32: g * 32 + 32].max()) // 128)
    assert 0 not in items.tolist() and 3 in items.tolist()
    eng = IndexerEngine.__new__(IndexerEngine)
    eng.B = 64
    tl, ch, cols = IndexerEngine._route_items(eng, np.arange(1, 20001), 64, 3)
    assert set(ch.tolist()) == {0, 1, 2}
    assert np.all(cols % 16 == 0) and np.all(cols <= 128)
    assert (ch == 0).sum() == (20000 * 64 + 127) // 128
