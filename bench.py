#!/usr/bin/env python
"""Benchmark: MISA indexer ms/layer at 128K causal prefill (H=64, h=8) vs the dense DSA kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--L 131072]

One step = one indexer layer: all T = L query rows of a causal prefill scored
against the L-key cache, top-k = 2048 per row (BASELINE.json configs[3] shape,
the C4 workload of SURVEY.md §8).  Inputs are synthetic (torch randn keys and
queries, softmax gates, seed 0) and device-resident for ``value``; ``e2e``
repeats the step through the public estimator API on pinned host K/Q/W: every
step copies the inputs host->device and the top-k device->host, in row chunks
whose copies overlap the scoring of the neighbouring chunks.  The
queries (2 GiB) exceed the 126 MB L2, so no explicit L2 flush is used.

Under torchrun (N > 1) the key axis is sharded block-cyclically across ranks,
each rank emits a local top-k with scores and an NCCL all-gather + merge kernel
produces the global top-k (strong scaling: the layer is fixed); timing is the
max over ranks.

``--impl reference`` times the reference algorithm on the host CPU (the oracle
port in ``oracle/``; the reference is Python and cannot be compiled) on the same
config and metric: a bounded stratified sample of rows per step, extrapolated
to one layer.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "indexer ms/layer at 128K (H^I=64,h=8) + speedup vs dense DSA; top-k recall"


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--L", type=int, default=131072)
    p.add_argument("--H", type=int, default=64)
    p.add_argument("--h", type=int, default=8)
    p.add_argument("--d", type=int, default=128)
    p.add_argument("--B", type=int, default=1024)
    p.add_argument("--k", type=int, default=2048)
    p.add_argument("--kprime", type=int, default=8192)
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-hier", action="store_true", help="skip timing MISA-dagger (k'=--kprime)")
    p.add_argument("--hier", action="store_true", help=argparse.SUPPRESS)  # the default now
    p.add_argument("--no-needle", action="store_true", help="skip the needle-retrieval recall leg")
    p.add_argument("--no-sattn", action="store_true", help="skip the sparse-attention consumer leg")
    p.add_argument("--no-decode", action="store_true", help="skip the C5 decode-step leg")
    p.add_argument("--no-sweep", action="store_true", help="skip the C2 / C3 prefill configs")
    p.add_argument("--no-c5", action="store_true", help="skip the C5 1M-key causal prefill leg")
    return p.parse_args()


def _workload_name(a):
    return f"C4 causal prefill L=T={a.L} H={a.H} h={a.h} d={a.d} B={a.B} k={a.k}"


def _config(a, world):
    """The workload config, identical in both arms (ours / --impl reference)."""
    return {"workload": _workload_name(a), "L": a.L, "T": a.L, "H": a.H, "h": a.h, "d": a.d, "B": a.B, "k": a.k,
            "parallelism": f"key-sharded x{world}" if world > 1 else "single device",
            "l2": _l2_note(a)}


def _l2_note(a):
    qb = a.L * a.H * a.d * 2
    if qb > 126 * 2**20:
        return f"inputs larger than L2 (queries {qb / 2**30:.2f} GiB read once per step); no explicit flush"
    return f"queries {qb / 2**20:.0f} MiB fit the 126 MB L2: steps after the first may hit L2"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["hbm_gbs"], pk["bf16_tflops"], pk["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def run_reference(a):
    """--impl reference: the reference algorithm (oracle port) on host cores, same metric/config."""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_bench
    from oracle import misa_oracle as O
    gen = torch.Generator().manual_seed(0)
    K = torch.randn(a.L, a.d, generator=gen).bfloat16().double().numpy()
    cores = os.cpu_count() or 1
    rows = cpu_bench.sample_rows(a.L, a.L, max(64, 8 * cores))
    rng = np.random.default_rng(0)
    Qr = O.bf16_round(rng.standard_normal((len(rows), a.H, a.d)))
    Wr = O.softmax_rows(rng.standard_normal((len(rows), a.H)))
    vals = []
    info = None
    for i in range(a.warmup + a.steps):
        info = cpu_bench.time_layer("misa", K, Qr, Wr, rows, a.L, a.L, k=a.k, h=a.h, B=a.B, kp=a.kprime,
                                    cores=cores)
        if i >= a.warmup:
            vals.append(info["ms_per_layer"])
    v = statistics.median(vals)
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "ms/layer", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64/f32 (fast32)", "data": "synthetic",
            "config": _config(a, int(os.environ.get("WORLD_SIZE", "1"))),
            "value_is_extrapolated": True,
            "cpu_baseline": {"value": v, "unit": "ms/layer", "cores": cores, "cpu_model": cpu_bench.cpu_model(),
                             "kind": "port",
                             "sample": f"{info['rows']} stratified causal rows per step, per-row reference "
                                       f"misa select (pool+route+score+top-k, fast32), extrapolated "
                                       f"linearly in prefix length over all {a.L} rows / {cores} cores: a full "
                                       f"layer on the CPU would not fit the driver's run, so each step is a "
                                       f"bounded sample and the value is an extrapolation"},
            "e2e": {"value": v, "unit": "ms/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _time_steps(fn, steps, warmup, barrier):
    import torch
    for _ in range(warmup):
        fn()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    barrier()
    return e0.elapsed_time(e1) / steps


def c5_prefill_leg(a, tc_burst, barrier):
    """C5 on one GPU: causal prefill at L = T = 2^20 (row passes bounded by the workspace),
    MISA and the dense DSA kernel, plus sampled-row recall against the CPU oracle."""
    import torch
    from paper_2605_07363_b200 import IndexerEngine, prepare_inputs
    from oracle import misa_oracle as O
    L5 = T5 = 1 << 20
    g5 = torch.Generator(device="cuda").manual_seed(5)
    K5 = torch.randn(L5, a.d, device="cuda", generator=g5).bfloat16()
    Q5 = torch.randn(T5, a.H, a.d, device="cuda", generator=g5).bfloat16()
    W5 = torch.softmax(torch.randn(T5, a.H, device="cuda", generator=g5), -1).float()
    x5 = prepare_inputs(K5, Q5, W5)
    em = IndexerEngine("misa", budget_k=a.k, active_heads_h=a.h, block_size=a.B)
    out = torch.empty(T5, a.k, dtype=torch.int32, device="cuda")
    ms_m = _time_steps(lambda: em.run_prepared(x5, out=out), 2, 1, barrier)
    passes = -(-T5 // em.row_chunk(x5))
    rows = [2048, 262144, 786432, T5 - 1]
    sel = torch.tensor(rows, device="cuda")
    got = out[sel].cpu().numpy()
    del em
    torch.cuda.empty_cache()
    ed = IndexerEngine("dsa", budget_k=a.k)
    ms_d = _time_steps(lambda: ed.run_prepared(x5, out=out), 1, 1, barrier)
    del ed
    Kn = K5.double().cpu().numpy()
    Qn, Wn = Q5[sel].double().cpu().numpy(), W5[sel].double().cpu().numpy()
    del x5, K5, Q5, W5, out
    torch.cuda.empty_cache()
    hit = tot = 0
    for i, t in enumerate(rows):
        ref = O.misa_select(Kn[: t + 1], Qn[i], Wn[i], a.k, a.h, a.B, precision="fast32")["selection"]
        g = got[i][got[i] >= 0]
        hit += len(set(g.tolist()) & set(ref.tolist()))
        tot += len(ref)
    P5 = L5 * (L5 + 1) // 2
    return {"workload": f"C5 causal prefill L=T={L5} H={a.H} h={a.h} d={a.d} B={a.B} k={a.k}, 1 GPU",
            "misa_ms": round(ms_m, 2), "dsa_ms": round(ms_d, 2), "speedup_vs_dsa": round(ms_d / ms_m, 3),
            "row_passes": passes, "misa_scores_per_s": P5 / (ms_m * 1e-3),
            "misa_tensor_frac_burst": round(2.0 * a.h * a.d * P5 / (ms_m * 1e-3) / 1e12 / tc_burst, 4),
            "topk_recall_vs_cpu_reference": round(hit / tot, 6), "recall_rows": rows}


def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2605_07363_b200 import _lib, MISAIndexer, DSAIndexer, IndexerEngine, prepare_inputs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # dev check of the N>1 path on a 1-GPU box: every rank on cuda:0, gloo transport
    shared = os.environ.get("MISA_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    L, T = a.L, a.L
    gen = torch.Generator(device="cuda").manual_seed(0)
    K = torch.randn(L, a.d, device="cuda", generator=gen).bfloat16()
    Q = torch.randn(T, a.H, a.d, device="cuda", generator=gen).bfloat16()
    W = torch.softmax(torch.randn(T, a.H, device="cuda", generator=gen), -1).float()
    hbm, tc_burst, tc_sust, peak_src = _peaks()

    if world > 1:
        from paper_2605_07363_b200.sharded import ShardedIndexer
        eng_m = ShardedIndexer("misa", world=world, rank=rank, budget_k=a.k, active_heads_h=a.h, block_size=a.B)
        eng_d = ShardedIndexer("dsa", world=world, rank=rank, budget_k=a.k, block_size=a.B)
    else:
        eng_m = IndexerEngine("misa", budget_k=a.k, active_heads_h=a.h, block_size=a.B)
        eng_d = IndexerEngine("dsa", budget_k=a.k)

    class _Out:
        def __init__(self, topk):
            self.topk = topk
    x = prepare_inputs(K, Q, W) if world == 1 else None

    def step_m():
        return eng_m.run_prepared(x) if world == 1 else eng_m.run(K, Q, W)

    def step_d():
        return eng_d.run_prepared(x) if world == 1 else eng_d.run(K, Q, W)

    # --- MISA (the headline value), with clocks sampled during the timed region
    launches0 = _lib.launch_count
    with Clocks(local) as clk:
        misa_ms = _time_steps(step_m, a.steps, a.warmup, barrier)
    launches = (_lib.launch_count - launches0) // (a.steps + a.warmup) * a.steps
    misa_ms = max_over_ranks(misa_ms)
    clocks = clk.summary()
    fallback = eng_m.last_fallback_rows if hasattr(eng_m, "last_fallback_rows") else 0

    # --- per-stage device times of one MISA step (events on the launching stream)
    stages = {}
    if world == 1:
        eng_m.stage_events = []
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record()
        res_m = step_m()
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record()
        torch.cuda.synchronize()
        ev = eng_m.stage_events + [("end", t1)]
        for (n0, e0), (_, e1) in zip(ev, ev[1:]):
            stages[n0] = stages.get(n0, 0.0) + e0.elapsed_time(e1)
        eng_m.stage_events = None
    else:
        res_m = _Out(eng_m.run(K, Q, W, gather=True))

    # --- dense DSA on the same inputs (the comparison kernel)
    dsa_ms = max_over_ranks(_time_steps(step_d, a.steps, a.warmup, barrier))
    dstages = {}
    if world == 1:
        eng_d.stage_events = []
        res_d = step_d()
        torch.cuda.synchronize()
        ev = eng_d.stage_events
        for (n0, e0), (_, e1) in zip(ev, ev[1:]):
            dstages[n0] = dstages.get(n0, 0.0) + e0.elapsed_time(e1)
        eng_d.stage_events = None
    else:
        res_d = _Out(eng_d.run(K, Q, W, gather=True))

    # --- the other BASELINE.json prefill configs (C2 DSv3.2 32K, C3 GLM-5 H=32 64K), 1 GPU
    sweep = None
    if world == 1 and not a.no_sweep:
        sweep = []
        for name, Ls, Hs in (("C2 DeepSeek-V3.2 shape, causal prefill L=T=32768, H=64, h=8", 32768, 64),
                             ("C3 GLM-5 shape, causal prefill L=T=65536, H=32, h=8", 65536, 32)):
            g3 = torch.Generator(device="cuda").manual_seed(2)
            Ks = torch.randn(Ls, a.d, device="cuda", generator=g3).bfloat16()
            Qs = torch.randn(Ls, Hs, a.d, device="cuda", generator=g3).bfloat16()
            Ws = torch.softmax(torch.randn(Ls, Hs, device="cuda", generator=g3), -1).float()
            xs = prepare_inputs(Ks, Qs, Ws)
            em = IndexerEngine("misa", budget_k=a.k, active_heads_h=a.h, block_size=a.B)
            ed = IndexerEngine("dsa", budget_k=a.k)
            ms_m = _time_steps(lambda: em.run_prepared(xs), 10, 3, barrier)
            ms_d = _time_steps(lambda: ed.run_prepared(xs), 5, 2, barrier)
            Ps = Ls * (Ls + 1) // 2
            sweep.append({"workload": name, "misa_ms": round(ms_m, 3), "dsa_ms": round(ms_d, 3),
                          "speedup_vs_dsa": round(ms_d / ms_m, 3), "misa_scores_per_s": Ps / (ms_m * 1e-3),
                          "misa_tensor_frac_burst": round(2.0 * a.h * a.d * Ps / (ms_m * 1e-3) / 1e12 / tc_burst, 4)})
            del Ks, Qs, Ws, xs, em, ed

    hier_ms = None
    res_h = None
    hstages = {}
    if not a.no_hier and world == 1:
        eng_h = IndexerEngine("misa_hier", budget_k=a.k, active_heads_h=a.h, block_size=a.B,
                              candidate_kprime=a.kprime)
        hier_ms = _time_steps(lambda: eng_h.run_prepared(x), a.steps, a.warmup, barrier)
        eng_h.stage_events = []
        res_h = eng_h.run_prepared(x)
        torch.cuda.synchronize()
        ev = eng_h.stage_events
        hstages = {}
        for (n0, e0), (_, e1) in zip(ev, ev[1:]):
            hstages[n0] = hstages.get(n0, 0.0) + e0.elapsed_time(e1)
        eng_h.stage_events = None
        res_h = type("R", (), {"topk": res_h.topk})()  # drop the views into the engine's workspace
        del eng_h

    # --- e2e through the public API: pinned host buffers, H2D each step, D2H of the top-k
    e2e = None
    if not a.no_e2e:
        Kh, Qh, Wh = K.cpu().pin_memory(), Q.cpu().pin_memory(), W.cpu().pin_memory()
        Kd, Qd, Wd = torch.empty_like(K), torch.empty_like(Q), torch.empty_like(W)
        out_h = torch.empty(T, a.k, dtype=torch.int32).pin_memory()
        est = MISAIndexer(budget_k=a.k, active_heads_h=a.h, block_size=a.B)
        if world > 1:
            est_engine = eng_m

        def step_e2e():
            if world == 1:  # public API on pinned host tensors: copy-overlapped row-chunk pipeline
                est.select_batch(Kh, Qh, Wh, out=out_h)  # the caller's pinned result buffer
                return
            Kd.copy_(Kh, non_blocking=True)
            Qd.copy_(Qh, non_blocking=True)
            Wd.copy_(Wh, non_blocking=True)
            r = est_engine.run(Kd, Qd, Wd)  # this rank's row slice of the global top-k
            out_h[: r.shape[0]].copy_(r, non_blocking=True)

        e2e_ms = max_over_ranks(_time_steps(step_e2e, a.steps, max(1, a.warmup), barrier))
        h2d = K.numel() * 2 + Q.numel() * 2 + W.numel() * 4
        e2e = {"value": e2e_ms, "unit": "ms/layer", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(T * a.k * 4)}

    # --- C5: key-sharded decode step at 1M keys (all ranks; max over ranks)
    sdec = None
    if world > 1 and not a.no_decode:
        from paper_2605_07363_b200.sharded import ShardedIndexer
        Ld, Td = 1 << 20, 64
        g2 = torch.Generator(device="cuda").manual_seed(1)
        Kd = torch.randn(Ld, a.d, device="cuda", generator=g2).bfloat16()
        Qd = torch.randn(Td, a.H, a.d, device="cuda", generator=g2).bfloat16()
        Wd = torch.softmax(torch.randn(Td, a.H, device="cuda", generator=g2), -1).float()
        sd = ShardedIndexer("misa", world=world, rank=rank, budget_k=a.k, active_heads_h=a.h, block_size=a.B)
        dms = max_over_ranks(_time_steps(lambda: sd.decode(Kd, Qd, Wd), 10, 3, barrier))
        sdec = {"method": "misa", "L": Ld, "T": Td, "ms_per_step": round(dms, 4),
                "what": "key-sharded decode step: local key-split scoring + long-row top-k with scores, "
                        "NCCL all-gather of the row lists, merge on every rank"}
        del Kd, Qd, Wd

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # --- recall vs the CPU reference algorithm on sampled rows (oracle, fast32, same bf16 inputs),
    # for every method timed here: the reference's selection of row t on IndexerWorkload(K[:t+1], Q[t], W[t])
    from oracle import misa_oracle as O
    rows = sorted(set(r for r in [2048, 8191, 8192, 8193, T // 4, T // 2, 3 * T // 4, T - 1] if r < T))
    Kn = K.double().cpu().numpy()
    hits = {m: [0, 0] for m in ("dsa", "misa", "misa_hier") if m != "misa_hier" or res_h is not None}
    iou = []
    for t in rows:
        n = t + 1
        qs, ws = Q[t].double().cpu().numpy(), W[t].double().cpu().numpy()
        got = {"dsa": res_d.topk[t], "misa": res_m.topk[t]}
        if res_h is not None:
            got["misa_hier"] = res_h.topk[t]
        got = {m: set(v[v >= 0].tolist()) for m, v in ((m, g.cpu().numpy()) for m, g in got.items())}
        for m in hits:
            if m == "dsa":
                ref = O.dsa_select(Kn[:n], qs, ws, a.k, "fast32")["selection"]
            elif m == "misa":
                ref = O.misa_select(Kn[:n], qs, ws, a.k, a.h, a.B, precision="fast32")["selection"]
            else:
                ref = O.misa_hier_select(Kn[:n], qs, ws, a.k, a.h, a.B, a.kprime, precision="fast32")["selection"]
            hits[m][0] += len(got[m] & set(ref.tolist()))
            hits[m][1] += len(ref)
        iou.append(len(got["misa"] & got["dsa"]) / len(got["misa"] | got["dsa"]))
    recall_by = {m: round(hv[0] / hv[1], 6) for m, hv in hits.items()}
    recall = recall_by["misa"]

    # --- roofline of the dominant kernel (MISA token scoring, tcgen05)
    P = L * (L + 1) // 2                       # causal scored pairs per layer
    flops_misa = 2.0 * a.h * a.d * P           # 2*h*d per score
    filt_ms = stages.get("sel:filter")
    traffic = None
    prof = os.path.join(REPO, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("score_filter_misa", {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roof = None
    if filt_ms:
        ach = flops_misa / (filt_ms * 1e-3) / 1e12
        roof = {"kernel": "score_kernel<128,8,FILTER> (MISA routed-head scoring + fused top-k filter)",
                "bound": "tensor", "achieved": round(ach, 1), "peak": tc_burst, "unit": "TFLOP/s",
                "frac": round(ach / tc_burst, 4), "frac_vs_sustained_peak": round(ach / tc_sust, 4),
                "traffic": traffic,
                "peak_source": f"{peak_src} bf16_tflops (burst; the sustained figure was measured at a lower "
                               f"clock than this run's, so it is reported beside it, not as the bound)",
                "flops_per_launch": flops_misa, "launch_ms": round(filt_ms, 3)}
    layer_frac = flops_misa / (misa_ms * 1e-3) / 1e12 / tc_burst
    # per-kernel roofline fractions of the MISA layer (SURVEY.md §8(d) algorithmic work)
    kernel_fracs = {}
    if stages:
        D, Hp = (64 if a.d <= 64 else 128), max(8, 1 << (a.H - 1).bit_length())
        hq = max(8, 1 << (a.h - 1).bit_length())
        stride = 32
        def hb(name, nbytes):
            ms = stages.get(name)
            if ms:
                kernel_fracs[name] = {"bound": "hbm", "bytes": int(nbytes), "GB_s": round(nbytes / ms / 1e6, 1),
                                      "frac": round(nbytes / ms / 1e6 / hbm, 4)}
        hb("route_scores", T * Hp * D * 2 + T * Hp * 4)
        hb("route_select", T * Hp * 4 * 2 + T * hq * 4)
        hb("sel:threshold", T * ((L + stride - 1) // stride) * 4 // 2)
        hb("sel:sample", T * hq * D * 2 + L * D * 2)
        hb("sel:select", T * a.k * 4)
        if filt_ms:
            kernel_fracs["sel:filter"] = {"bound": "tensor", "TFLOP_s": round(ach, 1), "frac": round(ach / tc_burst, 4)}

    cpu = None
    if not a.no_cpu and world == 1:
        from oracle import cpu_bench
        cores = os.cpu_count() or 1
        srows = cpu_bench.sample_rows(L, T, max(64, 8 * cores))
        Qs = Q[torch.as_tensor(srows)].double().cpu().numpy()
        Ws = W[torch.as_tensor(srows)].double().cpu().numpy()
        info = cpu_bench.time_layer("misa", Kn, Qs, Ws, srows, L, T, k=a.k, h=a.h, B=a.B, kp=a.kprime, cores=cores)
        cpu = {"value": round(info["ms_per_layer"], 1), "unit": "ms/layer", "cores": cores,
               "cpu_model": cpu_bench.cpu_model(), "kind": "port",
               "sample": f"{info['rows']} stratified causal rows of this workload, per-row reference misa select "
                         f"(pool+route+score+top-k, fast32) in {cores} single-BLAS-thread processes "
                         f"({info['cpu_s']:.1f} s CPU), extrapolated linearly in prefix length to all {T} rows"}

    decode = None
    if world == 1 and not a.no_decode:
        sys.path.insert(0, os.path.join(REPO, "tools"))
        from decode_bench import decode_numbers
        decode = {"what": "per-token decode step (C5 shapes): T query rows vs a PooledKeyCache of L keys, "
                          "eager engine.decode and CUDA-graph DecodeGraph replay, ms per step",
                  "rows": decode_numbers()}

    # --- the selection's consumer: sparse attention over this layer's MISA top-k
    sattn = None
    if world == 1 and not a.no_sattn:
        from paper_2605_07363_b200.sparse_attention import sparse_attention
        gq = torch.Generator(device="cuda").manual_seed(1)
        qa = torch.randn(T, 128, 128, device="cuda", generator=gq).bfloat16()
        tk = res_m.topk
        ms_sa = _time_steps(lambda: sparse_attention(qa, K, tk, 128), 3, 1, barrier)
        n_sel = int((tk >= 0).sum().item())
        fl = 2.0 * 2 * 128 * 128 * n_sel  # QK + PV over every selected token of every row
        sattn = {"workload": f"MQA sparse attention over the MISA top-{a.k}: T={T} rows, 128 heads, "
                             f"d_qk=d_v=128, latent rows = the layer's keys, bf16 in / f32 out",
                 "ms": round(ms_sa, 3), "TFLOP_s": round(fl / ms_sa / 1e9, 1),
                 "frac_tensor_burst": round(fl / ms_sa / 1e9 / tc_burst, 4)}
        del qa
        torch.cuda.empty_cache()

    # --- the indexer's producer: FP8 upstream projections of this layer's rows
    proj = None
    if world == 1 and not a.no_sattn:
        from paper_2605_07363_b200 import IndexerProjections
        dm, dqc = 7168, 1536  # DeepSeek-V3.2: hidden size, query latent
        pj = IndexerProjections(dm, a.H, a.d, d_q=dqc, seed=2)
        gh = torch.Generator(device="cuda").manual_seed(3)
        hid = torch.randn(T, dm, device="cuda", generator=gh).bfloat16()
        cql = torch.randn(T, dqc, device="cuda", generator=gh).bfloat16()
        ms_pj = _time_steps(lambda: pj(hid, cql), 3, 1, barrier)
        fl = 2.0 * T * (dqc * a.H * a.d + dm * (a.d + a.H))
        proj = {"workload": f"FP8 e4m3 projections of T={T} rows: q from a {dqc}-wide query latent "
                            f"({a.H}x{a.d}), k and signed w from {dm}-wide hidden states; per-token "
                            f"activation quantization included",
                "ms": round(ms_pj, 3), "TFLOP_s": round(fl / ms_pj / 1e9, 1),
                "note": "cuBLASLt row-wise-scaled FP8 GEMMs (library) + misa_quant_rows_fp8"}
        del hid, cql, pj
        torch.cuda.empty_cache()

    c5 = None
    if world == 1 and not a.no_c5:
        del eng_m, eng_d, x
        torch.cuda.empty_cache()
        c5 = c5_prefill_leg(a, tc_burst, barrier)

    needle = None
    if world == 1 and not a.no_needle:
        sys.path.insert(0, os.path.join(REPO, "tools"))
        from needle_bench import needle_numbers
        needle = needle_numbers(L=L, k=a.k, h=a.h, B=a.B, kprime=a.kprime)

    line = {
        "metric": METRIC, "value": round(misa_ms, 3), "unit": "ms/layer", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(misa_ms, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (torch randn keys/queries, softmax gates, seed 0)",
        "config": _config(a, world),
        "dsa_ms_per_layer": round(dsa_ms, 3), "speedup_vs_dsa": round(dsa_ms / misa_ms, 3),
        "topk_recall_vs_cpu_reference": round(recall, 6), "topk_recall_by_method": recall_by, "recall_rows": rows,
        "misa_iou_vs_dsa_random_data": round(float(np.mean(iou)), 4),
        "scores_per_s": P / (misa_ms * 1e-3), "layer_tensor_frac": round(layer_frac, 4),
        "layer_tensor_frac_note": "MISA FLOPs / layer time / burst bf16 peak",
        "kernel_fracs": kernel_fracs,
        "misa_stages_ms": {k: round(v, 4) for k, v in stages.items()},
        "dsa_stages_ms": {k: round(v, 4) for k, v in dstages.items()},
        "fallback_rows": fallback,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": int(launches),
        "decode": decode, "sharded_decode": sdec, "configs": sweep, "c5_prefill": c5, "needle": needle,
        "sparse_attention": sattn, "fp8_projections": proj,
    }
    if hier_ms is not None:
        line["misa_hier_ms_per_layer"] = round(hier_ms, 3)
        line["misa_hier_speedup_vs_dsa"] = round(dsa_ms / hier_ms, 3)
        line["misa_hier_stages_ms"] = {k: round(v, 4) for k, v in hstages.items()}
        rms = hstages.get("refine")
        if rms:
            n_ref = float(np.minimum(np.arange(1, T + 1, dtype=np.float64), a.kprime).sum())
            fl = 2.0 * a.H * a.d * n_ref
            gb = n_ref * (64 if a.d <= 64 else 128) * 2
            line["misa_hier_refine_roofline"] = {
                "kernel": "refine_kernel (all-head re-score of the gathered k' candidates)",
                "TFLOP_s": round(fl / rms / 1e9, 1), "frac_tensor_burst": round(fl / rms / 1e9 / tc_burst, 4),
                "gather_TB_s": round(gb / rms / 1e9, 2),
                "gather_note": "candidate key rows gathered from the L2-resident key set; tools/ubench_gather.cu "
                               "measured 15.7 TB/s for the same cp.async gather with nothing else running"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = _args()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
