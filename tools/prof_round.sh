#!/bin/bash
# Round-end evidence: default bench line, ncu launch list of a short bench, full ncu
# captures of the named kernels (one launch each).  Usage: bash tools/prof_round.sh TAG [kernel-regex ...]
set -u
TAG=$1; shift
mkdir -p gpurun_out
python -m paper_2605_07363_b200._build > /dev/null
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e \
  --no-decode --no-sweep --no-needle > /dev/null 2>&1
# each argument: a kernel-name regex over demangled names (e.g. 'score_kernel<\(int\)128, \(int\)8, \(bool\)1>'
# for the MISA filter scorer, 'refine_kernel' with METHOD=misa_hier); the first matching launch is captured
i=0
for k in "$@"; do
  i=$((i + 1))
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -c 1 \
    -o gpurun_out/${TAG}_k$i python tools/prof_run.py --method ${METHOD:-misa} > /dev/null 2>&1
done
ls gpurun_out | grep $TAG
