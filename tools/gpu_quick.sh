#!/bin/bash
# Quick GPU iteration: GPU tests + bench (no CPU leg / e2e / decode / sweeps / C5) -> gpurun_out/
mkdir -p gpurun_out
python -m paper_2605_07363_b200._build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-e2e --no-decode --no-sweep --no-needle --no-c5 --steps 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/pytest_gpu.log
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
except Exception as e:
    print("bench failed", e); raise SystemExit
keys = ["value", "dsa_ms_per_layer", "speedup_vs_dsa", "topk_recall_vs_cpu_reference", "topk_recall_by_method", "layer_tensor_frac", "fallback_rows", "misa_hier_ms_per_layer"]
print({k: d.get(k) for k in keys})
print("misa", d.get("misa_stages_ms")); print("dsa", d.get("dsa_stages_ms")); print("hier", d.get("misa_hier_stages_ms"))
print("roof", d.get("roofline")); print("clocks", d.get("clocks"))
PY
