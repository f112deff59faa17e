"""Sparse attention over the indexer's selection — the downstream consumer of the top-k
(Eq. 3, Sparse MLA in its MQA mode).  Outside the reference
package (SPEC.md:8 lists it as out of its scope); here so that an indexer layer can be timed
together with the attention it feeds.

    u[t, h] = sum_{s in T_t} softmax_s(scale * q[t, h] . c[s]) * c[s, :d_v]

with one latent row c[s] per token shared by all heads (MQA), T_t = the indexer's top-k of
row t (ascending, -1 padded).  ``misa_sparse_attention`` (csrc/sattn.cu): tcgen05, the
selected rows gathered 128 at a time, online softmax with a lazily raised max, P in bf16.
"""

from __future__ import annotations

import math

import torch

from . import _lib


def sparse_attention(queries: torch.Tensor, kv: torch.Tensor, topk: torch.Tensor, head_dim_v: int,
                     scale: float | None = None) -> torch.Tensor:
    """queries (T, H, d_qk), kv (L, d_qk), topk (T, k) int32 (each row's tokens first, -1
    after) -> (T, H, d_v) f32.  d_qk in {128, 256}; d_v <= d_qk (64/128/256); H <= 128."""
    if queries.ndim != 3 or kv.ndim != 2 or topk.ndim != 2:
        raise ValueError("queries (T, H, d), kv (L, d), topk (T, k)")
    T, H, d = queries.shape
    if kv.shape[1] != d or topk.shape[0] != T:
        raise ValueError("queries / kv / topk shapes disagree")
    if H > 128:
        raise ValueError("at most 128 query heads per row")
    dev = queries.device
    if H == 128 and queries.dtype == torch.bfloat16 and queries.is_contiguous():
        q = queries  # already the kernel's layout: no padded copy
    else:
        q = torch.zeros(T, 128, d, dtype=torch.bfloat16, device=dev)
        q[:, :H] = queries.to(torch.bfloat16)
    c = kv.to(torch.bfloat16).contiguous()
    tk = topk.to(torch.int32)
    if tk.stride(1) != 1:
        tk = tk.contiguous()
    out = torch.empty(T, H, head_dim_v, dtype=torch.float32, device=dev)
    s = 1.0 / math.sqrt(d) if scale is None else float(scale)
    _lib.call("misa_sparse_attention", q.data_ptr(), T, H, d, c.data_ptr(), c.shape[0], tk.data_ptr(), tk.stride(0),
              tk.shape[1], head_dim_v, s, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return out


__all__ = ["sparse_attention"]
