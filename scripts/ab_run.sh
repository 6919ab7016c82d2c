#!/bin/bash
# Same-session A/B of repo copies under ab/ (git-ignored): AB_DIRS="ab/X ab/Y" AB_CFGS="C4 C5" AB_REPS=2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; : > gpurun_out/ab.txt
for d in ${AB_DIRS}; do (cd $d && python -c "import paper_1405_3454_b200.build as b; b.build()") > /dev/null 2>&1; done
for rep in $(seq 1 ${AB_REPS:-2}); do for cfg in ${AB_CFGS}; do for d in ${AB_DIRS}; do
  line=$(cd $d && timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
  echo "$d $cfg $(echo "$line" | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['roofline']['per_kernel_ms'])")" >> gpurun_out/ab.txt
done; done; done
