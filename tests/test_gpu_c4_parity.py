"""Headline-shape parity (C4: causal prefill L = T = 131072, H = 64, h = 8, d = 128,
B = 1024, k = 2048, k' = 8192) of all three methods against the CPU oracle, plus a
direct check of the k' = 8192 coarse selector shape (topk5<512,32>, cap 4096).

Same protocol as test_gpu_parity.py: bf16 inputs shared by both
sides, oracle at fast32; heads bit-exact except documented ties (TAU_E); top-k exact
except elements within TAU_S of the k-th score; recall >= 99.9 % per method.  The
MISA-dagger check covers both stages at the shape the bench runs: the coarse top-k'
(routed scores, thresholded k' = 8192 path) against the oracle's top-k' with the GPU's
heads, then the all-head re-rank inside the GPU's candidates.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import misa_oracle as O  # noqa: E402
from test_gpu_parity import TAU_S, Census, _mag, check_heads, check_topk  # noqa: E402

pytestmark = pytest.mark.gpu

L = T = 131072
H, h, D, B, K_BUDGET, KP = 64, 8, 128, 1024, 2048, 8192


@pytest.fixture(scope="module")
def c4():
    from paper_2605_07363_b200 import IndexerEngine, prepare_inputs
    gen = torch.Generator(device="cuda").manual_seed(0)
    K = torch.randn(L, D, device="cuda", generator=gen).bfloat16()
    Q = torch.randn(T, H, D, device="cuda", generator=gen).bfloat16()
    W = torch.softmax(torch.randn(T, H, device="cuda", generator=gen), -1).float()
    x = prepare_inputs(K, Q, W)
    out = {}
    fallback = {}
    for method in ("dsa", "misa", "misa_hier"):
        eng = IndexerEngine(method, budget_k=K_BUDGET, active_heads_h=h, block_size=B, candidate_kprime=KP)
        r = eng.run_prepared(x, need_importance=method == "misa")
        torch.cuda.synchronize()
        keep = {"topk": r.topk.clone()}
        if r.heads is not None:
            keep["heads"] = r.heads.clone()
        if r.importance is not None:
            keep["importance"] = r.importance.clone()
        if r.candidates is not None:
            keep["candidates"] = r.sorted_candidates().clone()
        out[method] = keep
        fallback[method] = eng.last_fallback_rows
        del eng
        torch.cuda.empty_cache()
    rng = np.random.default_rng(1)
    rows = sorted(set([0, 1, 1023, 1024, 2047, 2048, 2049, 4095, 8191, 8192, 8193, 16383, 32768, 65535, 65536,
                       98304, T - 2, T - 1] + rng.integers(0, T, 6).tolist()))
    Kn = K.double().cpu().numpy()
    sel = torch.tensor(rows, device="cuda")
    Qn = Q[sel].double().cpu().numpy()
    Wn = W[sel].double().cpu().numpy()
    return dict(Kn=Kn, Qn=Qn, Wn=Wn, rows=rows, out={m: {k: v[sel].cpu().numpy() for k, v in d.items()}
                                                    for m, d in out.items()}, fallback=fallback)


def test_c4_dsa_rows_match_oracle(c4):
    cd = Census()
    for i, t in enumerate(c4["rows"]):
        n = t + 1
        keys, qs, ws = c4["Kn"][:n], c4["Qn"][i], c4["Wn"][i]
        scores = O.gated_relu_scores(keys, qs, ws, "fast32")
        check_topk(c4["out"]["dsa"]["topk"][i], scores, _mag(keys, qs, ws), K_BUDGET, cd, f"C4 dsa t={t}")
    assert cd.recall() >= 0.999, (cd.recall(), cd.ties)
    assert c4["fallback"]["dsa"] <= 1 + T // 10000
    print(f"[c4] dsa rows {cd.rows} recall {cd.recall():.6f} ties {cd.ties}")


def test_c4_misa_rows_match_oracle(c4):
    cm = Census()
    flips = 0
    for i, t in enumerate(c4["rows"]):
        n = t + 1
        keys, qs, ws = c4["Kn"][:n], c4["Qn"][i], c4["Wn"][i]
        _, pooled = O.block_pool(keys, B)
        E = O.route_head_importance(qs, ws, pooled, precision="fast32")
        np.testing.assert_allclose(c4["out"]["misa"]["importance"][i][:H], E, rtol=2e-5, atol=1e-9)
        gh = c4["out"]["misa"]["heads"][i]
        flips += check_heads(gh, E, h, f"C4 heads t={t}")
        gh = gh[gh >= 0]
        ms = O.misa_score(keys, qs, ws, gh, "fast32")
        hm = np.abs(ws[gh]) @ np.abs(qs[gh] @ keys.T)
        check_topk(c4["out"]["misa"]["topk"][i], ms, hm, K_BUDGET, cm, f"C4 misa t={t}")
    assert cm.recall() >= 0.999, (cm.recall(), cm.ties)
    assert flips <= 1
    assert c4["fallback"]["misa"] <= 1 + T // 10000
    print(f"[c4] misa rows {cm.rows} recall {cm.recall():.6f} ties {cm.ties} head flips {flips}")


def test_c4_misa_hier_rows_match_oracle(c4):
    """Both MISA-dagger stages at k' = 8192: the coarse cut (thresholded, cap-4096 selector)
    and the all-head re-rank inside the candidates (routing.py:144-174, dsa.py:95-115)."""
    cc, cf = Census(), Census()
    for i, t in enumerate(c4["rows"]):
        n = t + 1
        keys, qs, ws = c4["Kn"][:n], c4["Qn"][i], c4["Wn"][i]
        gh = c4["out"]["misa_hier"]["heads"][i]
        assert gh.tolist() == c4["out"]["misa"]["heads"][i].tolist()  # same router
        gh = gh[gh >= 0]
        ms = O.misa_score(keys, qs, ws, gh, "fast32")
        hm = np.abs(ws[gh]) @ np.abs(qs[gh] @ keys.T)
        cand = c4["out"]["misa_hier"]["candidates"][i]
        check_topk(cand, ms, hm, KP, cc, f"C4 hier-coarse t={t}")
        cand = cand[cand >= 0]
        assert cand.shape[0] == min(KP, n)
        fine = O.gated_relu_scores(keys[cand], qs, ws, "fast32")
        exp = O.topk_within(fine, cand, K_BUDGET)
        got = c4["out"]["misa_hier"]["topk"][i]
        got = got[got >= 0]
        assert got.shape[0] == min(K_BUDGET, n)
        cf.total += exp.shape[0]
        cf.rows += 1
        cf.hit += len(set(got.tolist()) & set(exp.tolist()))
        if got.tolist() != exp.tolist():
            kth = np.sort(fine)[::-1][min(K_BUDGET, cand.shape[0]) - 1]
            fm = _mag(keys[cand], qs, ws)
            pos = {c: j for j, c in enumerate(cand.tolist())}
            for c in set(got.tolist()) ^ set(exp.tolist()):
                cf.ties += 1
                assert abs(fine[pos[c]] - kth) <= TAU_S * (fm[pos[c]] + abs(kth)), (t, c)
    assert cc.recall() >= 0.999 and cf.recall() >= 0.999, (cc.recall(), cf.recall())
    assert c4["fallback"]["misa_hier"] <= 1 + T // 10000
    print(f"[c4] misa_hier rows {cc.rows} coarse recall {cc.recall():.6f} (ties {cc.ties}) "
          f"fine recall {cf.recall():.6f} (ties {cf.ties})")


def _pack(scores_row: np.ndarray, keys: np.ndarray, cap: int):
    """Per-quadrant candidate lists as the fused filter writes them: quadrant q holds the
    32-key chunks c with c % 4 == q, ascending by key; element = key << 32 | f32 bits."""
    lists = np.zeros((4, cap), dtype=np.uint64)
    cnt = np.zeros(4, dtype=np.int32)
    quad = (keys // 32) % 4
    bits = scores_row.astype(np.float32).view(np.uint32).astype(np.uint64)
    for q in range(4):
        sel = np.nonzero(quad == q)[0]
        cnt[q] = sel.shape[0]
        m = min(cap, sel.shape[0])
        lists[q, :m] = (keys[sel[:m]].astype(np.uint64) << np.uint64(32)) | bits[sel[:m]]
    return lists, cnt


@pytest.mark.parametrize("cap,mode", [(4096, "ordered"), (4096, "scores"), (3072, "ordered"), (3072, "runs")])
def test_coarse_selector_kprime_8192(cap, mode):
    """misa_select_topk at the MISA-dagger C4 coarse shape (k = 8192; cap 3072 per quadrant is
    the engine's choice at beta = 1.2, topk5<512,24>; 4096 is topk5<512,32>), rows of up to
    131072 keys with forced ties and -0/+0, against a (score desc, index asc) sort;
    under/overflowing rows are flagged.  mode "runs": the unordered variant
    (misa_select_topk_runs) must give the same set as 4 ascending runs, and the re-rank
    selector over those runs (misa_select_dense_runs) the same top-k as over the sorted set."""
    from paper_2605_07363_b200 import _lib
    from paper_2605_07363_b200.engine import IndexerEngine
    k = 8192
    _, _, eng_cap = IndexerEngine("misa", budget_k=2048).selector_params(k, L)
    assert eng_cap == 3072
    rng = np.random.default_rng(7)
    R = 320  # > 2 rows per SM: the persistent kernel's prefetch ring wraps
    n_rows = rng.integers(20000, L + 1, R)
    n_rows[:3] = [L, 12000, 9000]
    cand = np.zeros((R, 4, cap), dtype=np.uint64)
    cnt = np.zeros((R, 4), dtype=np.int32)
    expect = []
    for r in range(R):
        n = int(n_rows[r])
        s = rng.standard_normal(n).astype(np.float32)
        if r % 3 == 0:
            s = np.round(s * 8) / 8  # heavy ties: the index tie-break decides
        s[rng.integers(0, n, 50)] = -0.0
        s[rng.integers(0, n, 50)] = 0.0
        target = int(2.9 * cap) if r != 1 else 6000  # row 1 underflows (< k candidates of n >= k keys)
        if r == 2:
            target = n  # row 2: every one of its 9000 keys is a candidate
        tau = np.sort(s)[::-1][min(target, n) - 1]
        keys = np.nonzero(s >= tau)[0]
        lists, c = _pack(s[keys], keys, cap)
        cand[r], cnt[r] = lists, c
        order = sorted(keys.tolist(), key=lambda i: (-float(s[i]), i))[:k]  # -0.0 == +0.0 ties
        expect.append((sorted(order), s))
    # row 3: one quadrant over capacity -> overflow flag
    cnt[3, 1] = cap + 1
    prefix = torch.from_numpy(n_rows.astype(np.int32)).cuda()
    cd = torch.from_numpy(cand.view(np.int64).reshape(-1)).cuda()
    cc = torch.from_numpy(cnt.reshape(-1)).cuda()
    out = torch.empty(R, k, dtype=torch.int32, device="cuda")
    sc = torch.empty(R, k, device="cuda") if mode == "scores" else None
    flags = torch.zeros(R, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    runs = torch.empty(R, 4, dtype=torch.int32, device="cuda")
    if mode == "runs":
        _lib.call("misa_select_topk_runs", cd.data_ptr(), cc.data_ptr(), cap, prefix.data_ptr(), R, k, L,
                  out.data_ptr(), k, runs.data_ptr(), flags.data_ptr(), stream)
    else:
        _lib.call("misa_select_topk", cd.data_ptr(), cc.data_ptr(), cap, prefix.data_ptr(), R, k, L, out.data_ptr(),
                  k, None if sc is None else sc.data_ptr(), flags.data_ptr(), stream)
    torch.cuda.synchronize()
    fl = flags.cpu().numpy()
    got = out.cpu().numpy()
    rn = runs.cpu().numpy()
    assert fl[1] != 0 and fl[3] != 0
    for r in range(R):
        if r in (1, 3):
            continue
        assert fl[r] == 0, r
        exp, s = expect[r]
        row = got[r, : len(exp)]
        if mode == "runs":
            assert rn[r].sum() == len(exp), r
            o = np.concatenate([[0], np.cumsum(rn[r])])
            for q in range(4):
                assert np.all(np.diff(row[o[q]:o[q + 1]]) > 0), (r, q)
            assert sorted(row.tolist()) == exp, r
        else:
            assert row.tolist() == exp, r
        assert (got[r, len(exp):] == -1).all()
        if sc is not None:
            np.testing.assert_array_equal(sc[r, : len(exp)].cpu().numpy(), s[exp])
    if mode != "runs":
        return
    # re-rank selection over the runs == over the ascending set (fine scores: fresh, tied)
    ok = np.array([r not in (1, 3) for r in range(R)])
    rows = torch.from_numpy(np.nonzero(ok)[0]).cuda()
    ci = out[rows].contiguous()
    nc = (ci >= 0).sum(1).to(torch.int32)
    fine = torch.round(torch.randn(ci.shape, device="cuda") * 4) / 4
    fine[ci < 0] = 0
    kf = 2048
    o1 = torch.empty(rows.numel(), kf, dtype=torch.int32, device="cuda")
    _lib.call("misa_select_dense_runs", fine.data_ptr(), k, ci.data_ptr(), k, nc.data_ptr(),
              runs[rows].contiguous().data_ptr(), rows.numel(), kf, o1.data_ptr(), kf, stream)
    torch.cuda.synchronize()
    f = fine.cpu().numpy()
    c = ci.cpu().numpy()
    for i in range(rows.numel()):
        m = c[i] >= 0
        order = sorted(range(int(m.sum())), key=lambda j: (-float(f[i, j]), int(c[i, j])))[:kf]
        assert o1[i].cpu().numpy()[: len(order)].tolist() == sorted(c[i, order].tolist()), i
