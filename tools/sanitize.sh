#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the small-shape GPU
# paths: smoke() (pool, route, sampled scoring, tau, filter, topk5, refine, dense + long-row
# selection, decode) and the kernel / decode / varlen unit tests.
# Usage: bash tools/sanitize.sh TAG   -> gpurun_out/TAG_sanitize_<tool>.log
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
TESTS="tests/test_gpu_kernels.py tests/test_gpu_varlen.py tests/test_gpu_decode.py tests/test_gpu_boundary.py tests/test_gpu_invariants.py tests/test_gpu_sparse_attention.py tests/test_gpu_projections.py"
SEL="not c4 and not c5 and not 1048576"
for tool in memcheck racecheck synccheck initcheck; do
  log=gpurun_out/${TAG}_sanitize_${tool}.log
  echo "== $tool smoke" > $log
  timeout 900 $CS --tool $tool --print-limit 20 --target-processes all \
    python -c "import __graft_entry__ as g; g.smoke()" >> $log 2>&1
  echo "rc=$?" >> $log
  echo "== $tool tests" >> $log
  timeout 1500 $CS --tool $tool --print-limit 20 --target-processes all \
    python -m pytest $TESTS -x -q -m gpu -p no:cacheprovider -k "$SEL" >> $log 2>&1
  echo "rc=$?" >> $log
done
grep -H -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" gpurun_out/${TAG}_sanitize_*.log
