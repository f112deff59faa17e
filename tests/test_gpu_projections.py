"""FP8 upstream indexer projections (outside the reference):
the row-wise e4m3 quantization kernel against a torch restatement, the projections against
fp32 GEMMs of the same (dequantized) operands, and the projected q / k / w through the indexer."""
import math

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def test_quantize_rows_fp8_matches_torch():
    from paper_2605_07363_b200 import quantize_rows_fp8
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(300, 1040, device="cuda", generator=g).bfloat16() * 3
    x[7] = 0  # a zero row: scale 1, zeros
    x[9, 5] = 1e4  # one large element sets the row's scale
    q, s = quantize_rows_fp8(x)
    amax = x.float().abs().amax(1)
    exp_s = torch.where(amax > 0, amax / 448, torch.ones_like(amax))
    assert torch.allclose(s, exp_s, rtol=2e-7, atol=0)
    # the kernel multiplies by the IEEE f32 quotient 448 / amax (torch's scalar / tensor takes a
    # reciprocal, which differs in the last bit and flips e4m3 ties)
    inv = torch.where(amax > 0, (448.0 / amax.double()).float(), torch.ones_like(amax))
    ref = (x.float() * inv[:, None]).clamp(-448, 448).to(torch.float8_e4m3fn)  # RNE, saturating
    assert torch.equal(q.view(torch.uint8), ref.view(torch.uint8))
    assert float(q[9, 5].float()) == 448.0 and torch.count_nonzero(q[7].float()) == 0


def test_projections_match_fp32_gemm_of_the_fp8_operands():
    from paper_2605_07363_b200 import IndexerProjections, quantize_rows_fp8
    g = torch.Generator(device="cuda").manual_seed(1)
    T, dm, dq, H, d = 512, 1024, 768, 32, 128
    proj = IndexerProjections(dm, H, d, d_q=dq, seed=3)
    h = torch.randn(T, dm, device="cuda", generator=g).bfloat16()
    c = torch.randn(T, dq, device="cuda", generator=g).bfloat16()
    q, k, w = proj(h, c)
    assert q.shape == (T, H, d) and k.shape == (T, d) and w.shape == (T, H)
    assert q.dtype == torch.bfloat16 and k.dtype == torch.bfloat16 and w.dtype == torch.float32
    Wq, Wk, Ww = proj.dequantized_weights()
    h8, sh = quantize_rows_fp8(h)
    c8, sc = quantize_rows_fp8(c)
    hd, cd = h8.float() * sh[:, None], c8.float() * sc[:, None]
    for got, exp in ((q.float().view(T, -1), cd @ Wq.T), (k.float(), hd @ Wk.T),
                     (w, (hd @ Ww.T).bfloat16().float() / math.sqrt(H))):
        err = (got - exp).abs().max().item()
        assert err <= 1e-2 * exp.abs().max().item() + 1e-3, err  # bf16 output rounding
    # and close to the projection of the unquantized activations (e4m3: 3 mantissa bits)
    ref = h.float() @ Wk.T
    rel = ((k.float() - ref).norm() / ref.norm()).item()
    assert rel < 0.08, rel


def test_projected_inputs_feed_the_indexer():
    """The projections' outputs are the engine's input layouts: a causal MISA layer runs on
    them and equals the same layer on the bf16 copies the oracle would see."""
    from paper_2605_07363_b200 import IndexerEngine, IndexerProjections
    g = torch.Generator(device="cuda").manual_seed(2)
    T, dm, H, d = 2048, 512, 64, 128
    proj = IndexerProjections(dm, H, d, seed=5)
    h = torch.randn(T, dm, device="cuda", generator=g).bfloat16()
    q, k, w = proj(h)
    eng = IndexerEngine("misa", budget_k=256, active_heads_h=8, block_size=128)
    a = eng.run(k, q, w).topk.clone()
    b = eng.run(k.clone(), q.clone(), w.clone()).topk
    assert torch.equal(a, b)
    assert int((a[-1] >= 0).sum()) == 256 and bool((w < 0).any())  # signed gates reach the indexer
