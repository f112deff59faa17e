"""Real ShardedIndexer (prefill and decode) with two ranks over gloo sharing the one GPU of
the test box: every rank's result equals the single-GPU engine (NCCL only changes the
transport of the same all-gather / all-to-all)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_two_rank_sharded_prefill_and_decode_equal_single_gpu():
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(repo, "tools", "sharded_smoke.py")], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "sharded smoke ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
