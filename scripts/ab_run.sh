cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; : > gpurun_out/ab.txt
for d in ab/A ab/D; do (cd $d && python -c "import paper_1405_3454_b200.build as b; b.build()") > /dev/null 2>&1; done
for rep in 1 2; do for cfg in C4 C5; do for d in ab/A ab/D; do
  line=$(cd $d && timeout 300 python bench.py --config $cfg --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
  echo "$d $cfg $(echo "$line" | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['roofline']['per_kernel_ms'])")" >> gpurun_out/ab.txt
done; done; done
