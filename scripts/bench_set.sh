#!/bin/bash
# Quick bench sweep (under gpurun): one summary line per argument set.
# usage: bench_set.sh "--config C4" "--config C5" ...
cd "${GRAFT_REPO_ROOT:-.}"
for a in "$@"; do
  echo "== $a"
  python bench.py $a --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d['roofline']
print(d['value'], d['ms_per_step'], r['per_kernel_ms'], 'frac', r['frac'], 'host', d['host_step2']['value'])"
done
