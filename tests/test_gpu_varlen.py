"""Several independent key sequences in one device call (C3 "batched queries"; the
reference evaluates independent workloads / prefixes one at a time, workload.py:91-110,
harness.py:368-394).  Every row of a packed call must equal the same row run on its own
sequence alone (same kernels: bit-identical), and sampled rows must match the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import misa_oracle as O  # noqa: E402
from test_gpu_parity import Census, _mag, check_heads, check_topk  # noqa: E402

pytestmark = pytest.mark.gpu


def _seqs(lens_k, lens_q, H, d, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    K = torch.randn(int(sum(lens_k)), d, device="cuda", generator=g).bfloat16()
    Q = torch.randn(int(sum(lens_q)), H, d, device="cuda", generator=g).bfloat16()
    W = torch.softmax(torch.randn(int(sum(lens_q)), H, device="cuda", generator=g), -1).float()
    ck = np.concatenate([[0], np.cumsum(lens_k)])
    cq = np.concatenate([[0], np.cumsum(lens_q)])
    return K, Q, W, ck, cq


@pytest.mark.parametrize("method,H,d,B,k", [
    ("misa", 64, 128, 1024, 512),
    ("dsa", 32, 128, 1024, 512),
    ("misa_hier", 16, 64, 256, 256),
    ("misa", 8, 64, 64, 64),          # 16 rows per router tile: tiles span several sequences
])
def test_varlen_rows_equal_per_sequence_runs(method, H, d, B, k):
    from paper_2605_07363_b200 import IndexerEngine
    lens_k = [3000, 9000, 700, 1, 4100, 20000]
    lens_q = [3000, 333, 1, 1, 57, 2048]  # causal prefill tails of each sequence
    K, Q, W, ck, cq = _seqs(lens_k, lens_q, H, d, seed=61)
    kw = dict(budget_k=k, active_heads_h=8, block_size=B, candidate_kprime=4 * k)
    eng = IndexerEngine(method, **kw)
    res = eng.run_varlen(K, ck, Q, W, cq, need_importance=method != "dsa")
    torch.cuda.synchronize()
    for s in range(len(lens_k)):
        a, b = int(cq[s]), int(cq[s + 1])
        if a == b:
            continue
        ref = IndexerEngine(method, **kw).run(K[ck[s]:ck[s + 1]], Q[a:b], W[a:b], need_importance=method != "dsa")
        torch.cuda.synchronize()
        assert torch.equal(res.topk[a:b], ref.topk), (method, s)
        if method != "dsa":
            assert torch.equal(res.heads[a:b], ref.heads), (method, s)
            assert torch.equal(res.importance[a:b], ref.importance), (method, s)
        if method == "misa_hier":
            assert torch.equal(res.candidates[a:b], ref.candidates), (method, s)


def test_varlen_explicit_prefixes_match_oracle():
    """Two sequences of different lengths with explicit per-row prefixes, against the oracle
    (the reference's selection of each row on its own IndexerWorkload)."""
    from paper_2605_07363_b200 import IndexerEngine
    H, d, B, k, h = 64, 128, 1024, 1024, 8
    lens_k, lens_q = [50000, 23000], [6, 5]
    K, Q, W, ck, cq = _seqs(lens_k, lens_q, H, d, seed=62)
    pl = np.array([1, 1500, 20000, 37777, 49999, 50000, 900, 4096, 12000, 22999, 23000])
    out = {m: IndexerEngine(m, budget_k=k, active_heads_h=h, block_size=B, candidate_kprime=4096).run_varlen(
        K, ck, Q, W, cq, prefix_len=pl) for m in ("dsa", "misa", "misa_hier")}
    torch.cuda.synchronize()
    Kn = K.double().cpu().numpy()
    Qn, Wn = Q.double().cpu().numpy(), W.double().cpu().numpy()
    cd, cm, ch = Census(), Census(), Census()
    seq_of = np.repeat(np.arange(2), lens_q)
    for t in range(len(pl)):
        s = seq_of[t]
        keys = Kn[ck[s]: ck[s] + pl[t]]
        qs, ws = Qn[t], Wn[t]
        check_topk(out["dsa"].topk[t].cpu().numpy(), O.gated_relu_scores(keys, qs, ws, "fast32"),
                   _mag(keys, qs, ws), k, cd, f"dsa t={t}")
        _, pooled = O.block_pool(keys, B)
        E = O.route_head_importance(qs, ws, pooled, precision="fast32")
        gh = out["misa"].heads[t].cpu().numpy()
        check_heads(gh, E, h, f"heads t={t}")
        gh = gh[gh >= 0]
        ms = O.misa_score(keys, qs, ws, gh, "fast32")
        hm = np.abs(ws[gh]) @ np.abs(qs[gh] @ keys.T)
        check_topk(out["misa"].topk[t].cpu().numpy(), ms, hm, k, cm, f"misa t={t}")
        check_topk(out["misa_hier"].sorted_candidates()[t].cpu().numpy(), ms, hm, 4096, ch, f"hier coarse t={t}")
    for c in (cd, cm, ch):
        assert c.recall() >= 0.999, c.recall()
