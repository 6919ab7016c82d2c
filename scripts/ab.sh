#!/bin/bash
# Same-session A/B timing of several builds: ab.sh DIR1 DIR2 ...
# Each DIR is a full copy of the repo (e.g. ab/A, ab/B — git-ignored) with its
# own in-tree libcudapre.so; each variant runs its own bench.py AB_REPS times,
# interleaved.  AB_ARGS: extra bench.py arguments (e.g. "--config C4").
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; : > gpurun_out/ab.txt
for rep in $(seq 1 ${AB_REPS:-3}); do
  for d in "$@"; do
    line=$(timeout 300 python "$d/bench.py" --no-e2e --no-cpu-baseline ${AB_ARGS} 2>/dev/null | grep '^{')
    echo "$d ${AB_ARGS} $(echo "$line" | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']['per_kernel_ms']; print(d['value'], r)")" >> gpurun_out/ab.txt
  done
done
