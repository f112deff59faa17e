"""CPU tests of the MISAWKLD corpus layer (workload.py:202-254, cli.py:305-330): headers,
naming, validation — everything before the device batch."""

import os

import numpy as np
import pytest

from paper_2605_07363_b200 import IndexerConfig, gen_needle_workload, gen_random_workload, load_workload, save_workload
from paper_2605_07363_b200.corpus import Corpus, read_header, save_corpus


def _cfg():
    return IndexerConfig(n_heads=8, head_dim=16, budget_k=8, block_size=16, active_heads_h=2, candidate_kprime=32)


def test_save_and_open_roundtrip(tmp_path):
    cfg = _cfg()
    ws = [gen_random_workload(3, 40, cfg), gen_needle_workload(4, 70, 0.5, 8, 10.0, cfg)]
    paths = save_corpus(ws, tmp_path)
    assert [os.path.basename(p) for p in paths] == ["workload_L40_d0_r0_s3.bin", "workload_L70_d0_r1_s4.bin"]
    c = Corpus.open(tmp_path)
    assert len(c) == 2 and (c.n_heads, c.head_dim) == (8, 16)
    assert [e.seed for e in c.entries] == [3, 4]
    assert [e.prefix_len for e in c.entries] == [40, 70]
    for i, w in enumerate(ws):
        got = c.workload(i)
        assert np.array_equal(got.keys, w.keys) and np.array_equal(got.queries, w.queries)
        assert np.array_equal(got.gate_weights, w.gate_weights) and got.seed == 0  # format drops the seed
    assert read_header(paths[1]) == (70, 16, 8)


def test_header_validation_matches_load_workload(tmp_path):
    w = gen_random_workload(1, 10, _cfg())
    p = tmp_path / "w.bin"
    save_workload(w, p)
    raw = p.read_bytes()
    cases = {
        "short.bin": raw[:10],
        "magic.bin": b"XISAWKLD" + raw[8:],
        "version.bin": raw[:8] + (2).to_bytes(4, "little") + raw[12:],
        "size.bin": raw + b"\0" * 8,
    }
    for name, blob in cases.items():
        q = tmp_path / name
        q.write_bytes(blob)
        with pytest.raises(ValueError) as e1:
            read_header(q)
        with pytest.raises(ValueError) as e2:
            load_workload(q)
        assert str(e1.value) == str(e2.value), name


def test_corpus_rejects_mixed_shapes_and_empty(tmp_path):
    save_workload(gen_random_workload(1, 10, _cfg()), tmp_path / "a.bin")
    save_workload(gen_random_workload(1, 10, IndexerConfig(n_heads=4, head_dim=16, active_heads_h=2)), tmp_path / "b.bin")
    with pytest.raises(ValueError, match="mixes"):
        Corpus.open(tmp_path)
    with pytest.raises(ValueError, match="empty"):
        Corpus([])


def test_archived_corpus_is_readable(golden_dir):
    """The committed parity corpus (written by the reference's own save_workload)."""
    c = Corpus.open(os.path.join(golden_dir, "corpus"))
    g = np.load(os.path.join(golden_dir, "corpus", "reference_selections.npz"))
    assert [os.path.basename(e.path) for e in c.entries] == sorted(g["names"].tolist())
    H, d = int(g["cfg"][0]), int(g["cfg"][1])
    assert (c.n_heads, c.head_dim) == (H, d)
    for i in range(len(c)):
        assert c.workload(i).bf16_exact
