#!/bin/bash
# A/B timing of env variants in one box session: ab.sh "ENV=1" "ENV=2" ...
# (perf experiments; each variant runs the bench 3x, interleaved; AB_ARGS
# are extra bench.py arguments, e.g. "--config C4")
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; : > gpurun_out/ab.txt
for rep in $(seq 1 ${AB_REPS:-3}); do
  for v in "$@"; do
    line=$(env $v timeout 300 python bench.py --no-e2e --no-cpu-baseline ${AB_ARGS} 2>/dev/null | grep '^{')
    echo "$v ${AB_ARGS} $(echo "$line" | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']['per_kernel_ms']; print(d['value'], r.get('k2_filter'), r.get('k1_extremes(+seed)'), d.get('k2_lookback_spins_per_step'))")" >> gpurun_out/ab.txt
  done
done
