"""Upstream indexer projections in FP8 ("upstream indexer projections
(FP8, signed weights)").  Outside the reference package — SPEC.md:8 and :187 leave FP8 out
of its scope, and SPEC.md:89 notes that the paper does not say how the gates w^I are made;
PAPER.md:98 describes DeepSeek-V3.2's indexer as FP8.  Here so that the indexer's inputs can be
produced on the device from hidden states, the way a model layer would:

    q^I_t = (c_t W_q^T) reshaped (H, d)      bf16   (c_t: the query-side input, e.g. the query latent)
    k^I_s =  h_s W_k^T                       bf16   (one key row per token, shared by the heads)
    w^I_t = (h_t W_w^T) / sqrt(H)            f32    (signed gates: no softmax, both signs allowed)

Weights are held in FP8 e4m3 with one scale per output channel, activations are quantized per
token on the fly (``misa_quant_rows_fp8``, csrc/quant.cu), and each projection is one cuBLASLt
row-wise-scaled FP8 GEMM (``torch._scaled_mm``: a plain library GEMM, bf16 out).  The outputs
feed ``IndexerEngine.run`` unchanged; the indexer itself stays on its bf16 parity path.
"""

from __future__ import annotations

import math

import torch

from . import _lib


def quantize_rows_fp8(x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """x (R, C) -> (e4m3 (R, C), f32 scales (R,)) with x ~= q.float() * scale[:, None]."""
    if x.ndim != 2 or not x.is_cuda:
        raise ValueError("x must be a 2-D CUDA tensor")
    xb = x.to(torch.bfloat16).contiguous()
    R, C = xb.shape
    if C % 16:
        raise ValueError(f"the reduced dimension must be a multiple of 16 (cuBLASLt FP8), got {C}")
    q = torch.empty(R, C, dtype=torch.float8_e4m3fn, device=x.device)
    s = torch.empty(R, dtype=torch.float32, device=x.device)
    _lib.call("misa_quant_rows_fp8", xb.data_ptr(), R, C, q.data_ptr(), s.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    return q, s


class IndexerProjections:
    """FP8 projections hidden states -> (q^I, k^I, w^I) for the indexer.

    ``weights`` = (W_q (H*d, d_q), W_k (d, d_model), W_w (H, d_model)) in any float dtype, or
    None for a seeded random initialisation (N(0, 1/fan_in)); they are quantized once."""

    def __init__(self, d_model: int, n_heads: int = 64, head_dim: int = 128, d_q: int | None = None, *,
                 weights=None, seed: int = 0, device="cuda"):
        self.d_model, self.H, self.d = int(d_model), int(n_heads), int(head_dim)
        self.d_q = int(d_q or d_model)
        for name, v in (("d_model", self.d_model), ("d_q", self.d_q)):
            if v % 16:
                raise ValueError(f"{name} must be a multiple of 16, got {v}")
        if (self.H * self.d) % 16 or self.d % 16 or self.H % 16:
            raise ValueError("n_heads, head_dim and n_heads*head_dim must be multiples of 16")
        dev = torch.device(device)
        if weights is None:
            g = torch.Generator(device="cpu").manual_seed(seed)
            weights = (torch.randn(self.H * self.d, self.d_q, generator=g) / math.sqrt(self.d_q),
                       torch.randn(self.d, self.d_model, generator=g) / math.sqrt(self.d_model),
                       torch.randn(self.H, self.d_model, generator=g) / math.sqrt(self.d_model))
        wq, wk, ww = (torch.as_tensor(w).to(dev) for w in weights)
        shapes = ((self.H * self.d, self.d_q), (self.d, self.d_model), (self.H, self.d_model))
        for w, shp, nm in zip((wq, wk, ww), shapes, ("W_q", "W_k", "W_w")):
            if tuple(w.shape) != shp:
                raise ValueError(f"{nm} must be {shp}, got {tuple(w.shape)}")
        # per-output-channel e4m3 weights: rows of W are output channels
        self.wq, self.sq = quantize_rows_fp8(wq)
        self.wk, self.sk = quantize_rows_fp8(wk)
        self.ww, self.sw = quantize_rows_fp8(ww)

    @staticmethod
    def _gemm(a8, sa, w8, sw) -> torch.Tensor:
        # (M, K) row-major x (K, N) column-major (= W8^T), row-wise scales on both sides
        return torch._scaled_mm(a8, w8.t(), scale_a=sa[:, None], scale_b=sw[None, :], out_dtype=torch.bfloat16)

    def __call__(self, hidden: torch.Tensor, query_input: torch.Tensor | None = None):
        """hidden (T, d_model) -> q (T, H, d) bf16, k (T, d) bf16, w (T, H) f32.  ``query_input``
        (T, d_q) feeds W_q when given (DeepSeek-V3.2 projects queries from the query latent)."""
        if hidden.ndim != 2 or hidden.shape[1] != self.d_model:
            raise ValueError(f"hidden must be (T, {self.d_model})")
        cq = hidden if query_input is None else query_input
        if cq.ndim != 2 or cq.shape[1] != self.d_q or cq.shape[0] != hidden.shape[0]:
            raise ValueError(f"query_input must be (T, {self.d_q})")
        h8, sh = quantize_rows_fp8(hidden)
        c8, sc = (h8, sh) if query_input is None else quantize_rows_fp8(cq)
        q = self._gemm(c8, sc, self.wq, self.sq).view(-1, self.H, self.d)
        k = self._gemm(h8, sh, self.wk, self.sk)
        w = self._gemm(h8, sh, self.ww, self.sw).float() * (1.0 / math.sqrt(self.H))
        return q, k, w

    def dequantized_weights(self):
        """(W_q, W_k, W_w) as the f32 values the FP8 GEMMs actually multiply by."""
        return tuple(w8.float() * s[:, None] for w8, s in ((self.wq, self.sq), (self.wk, self.sk),
                                                           (self.ww, self.sw)))


__all__ = ["IndexerProjections", "quantize_rows_fp8"]
