"""Real ShardedIndexer (prefill and decode) with two ranks over gloo sharing the one GPU of
the test box: every rank's result equals the single-GPU engine (NCCL only changes the
transport of the same all-gather / all-to-all)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_prefill_and_decode_equal_single_gpu(world):
    """world = 4 adds MISA-dagger at k' = 8192 with merge rounds (4 x 8192 > 16384)."""
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(repo, "tools", "sharded_smoke.py"), str(world)],
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0 and "sharded smoke ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_bench_two_rank_path_runs():
    """bench.py's N>1 path end to end (torchrun, 2 ranks sharing the box's one GPU over gloo
    via MISA_BENCH_SHARED_GPU): one JSON line from rank 0 with exact recall."""
    import json
    import socket
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, MISA_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(repo, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--L", "8192"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=repo)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["topk_recall_vs_cpu_reference"] == 1.0 and d["e2e"]["value"] > 0
