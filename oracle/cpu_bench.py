"""CPU baseline timing of the reference algorithm (oracle port) — TEST/BENCH INFRASTRUCTURE.

Used only by ``bench.py`` (cpu_baseline leg and ``--impl reference``).  Times the
reference's per-query path (``estimators.py:185-188`` -> ``routing.py:123-141``:
pool the prefix, route, score the routed heads, top-k; precision fast32, as
BASELINE.md §3 prescribes) on a stratified sample of causal rows, one process
per host core with single-threaded BLAS, and extrapolates to one layer as
sum_t t_hat(n_t) / cores with t_hat linear in the prefix length n.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import tempfile
import time

import numpy as np

_K = None


def _init(path):
    global _K
    _K = np.load(path, mmap_mode="r")


def _row(args):
    method, n, q, w, k, h, B, kp = args
    from oracle import misa_oracle as O
    keys = np.asarray(_K[:n])
    t0 = time.perf_counter()
    if method == "dsa":
        O.dsa_select(keys, q, w, k, "fast32")
    elif method == "misa":
        O.misa_select(keys, q, w, k, h, B, precision="fast32")
    else:
        O.misa_hier_select(keys, q, w, k, h, B, kp, precision="fast32")
    return n, time.perf_counter() - t0


def sample_rows(L: int, T: int, count: int) -> np.ndarray:
    """Stratified rows over the causal range: first, last, block-boundary-ish and evenly spaced."""
    first = L - T
    return np.unique(np.linspace(0, T - 1, count).round().astype(np.int64))


def cpu_model() -> str:
    """The host CPU's model name (state the core count and the CPU model)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def time_layer(method: str, K: np.ndarray, Q_rows: np.ndarray, W_rows: np.ndarray, rows: np.ndarray, L: int,
               T: int, *, k: int, h: int, B: int, kp: int, cores: int | None = None) -> dict:
    """K: (L, d) float64 (bf16-exact); Q_rows/W_rows: the sampled rows' queries/gates."""
    cores = cores or os.cpu_count() or 1
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "K.npy")
        np.save(path, np.ascontiguousarray(K, dtype=np.float64))
        ns = (L - T) + rows + 1
        jobs = [(method, int(n), Q_rows[i], W_rows[i], k, h, B, kp) for i, n in enumerate(ns)]
        ctx = mp.get_context("spawn")
        t0 = time.perf_counter()
        with ctx.Pool(cores, initializer=_init, initargs=(path,)) as pool:
            res = pool.map(_row, jobs, chunksize=1)
        wall = time.perf_counter() - t0
    n = np.array([r[0] for r in res], dtype=np.float64)
    s = np.array([r[1] for r in res], dtype=np.float64)
    A = np.stack([np.ones_like(n), n], 1)
    coef, *_ = np.linalg.lstsq(A, s, rcond=None)
    a, b = float(coef[0]), float(coef[1])
    all_n = np.arange(L - T + 1, L + 1, dtype=np.float64)
    layer_s = float(np.sum(np.maximum(a + b * all_n, 0.0))) / cores
    return {"ms_per_layer": layer_s * 1e3, "cores": cores, "rows": int(len(jobs)), "cpu_s": float(s.sum()),
            "wall_s": wall, "fit_a_s": a, "fit_b_s_per_key": b}
