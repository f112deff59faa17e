"""Host-side argument validation of the indexer's neighbours (FP8 projections, sparse
attention): errors are raised before any device work, so these run without a GPU."""
import pytest

torch = pytest.importorskip("torch")


def test_projection_dims_validated():
    from paper_2605_07363_b200 import IndexerProjections
    with pytest.raises(ValueError):
        IndexerProjections(100)  # d_model not a multiple of 16
    with pytest.raises(ValueError):
        IndexerProjections(1024, n_heads=8, head_dim=120)
    with pytest.raises(ValueError):
        IndexerProjections(1024, d_q=1000)


def test_quantize_rows_needs_a_cuda_matrix():
    from paper_2605_07363_b200 import quantize_rows_fp8
    with pytest.raises(ValueError):
        quantize_rows_fp8(torch.zeros(4, 32))  # host tensor
    with pytest.raises(ValueError):
        quantize_rows_fp8(torch.zeros(32))


def test_sparse_attention_shapes_validated():
    from paper_2605_07363_b200 import sparse_attention
    q, kv, tk = torch.zeros(2, 8, 128), torch.zeros(10, 128), torch.zeros(2, 4, dtype=torch.int32)
    with pytest.raises(ValueError):
        sparse_attention(q[0], kv, tk, 128)  # queries must be (T, H, d)
    with pytest.raises(ValueError):
        sparse_attention(q, torch.zeros(10, 64), tk, 128)  # head dims disagree
    with pytest.raises(ValueError):
        sparse_attention(torch.zeros(2, 200, 128), kv, tk, 128)  # > 128 heads
