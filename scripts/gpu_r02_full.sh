#!/bin/bash
# Round-2 measurement session (under gpurun): tests, every config's bench line,
# launch lists and ncu captures.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; : > gpurun_out/status.txt
run() { local name=$1 t=$2; shift 2; local t0=$(date +%s); timeout "$t" "$@" > "gpurun_out/$name.log" 2>&1; echo "$name=$? $(( $(date +%s) - t0 ))s" >> gpurun_out/status.txt; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
python -c "import paper_1405_3454_b200.build as b, synth.cuda as s, oracle as o; b.build(); s.build(); o.build()" > gpurun_out/build.log 2>&1
[ -z "$NO_TESTS" ] && run pytest_gpu 2400 python -m pytest tests -m gpu -x -q
run smoke 300 python __graft_entry__.py smoke
run bench_C5 900 python bench.py
for c in C1 C2a C2b C3 C4 C4e0; do run bench_$c 900 python bench.py --config $c; done
run bench_T4 900 python bench.py --config T4
run bench_C5_ref 900 python bench.py --impl reference --steps 3 --warmup 1
if [ -z "$NO_NCU" ]; then
  for c in C5 C4 C3 C2a; do
    CMD="python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
    run ncu_launches_$c 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv $CMD
    run ncu_full_$c 1200 ncu --set full --clock-control none --import-source on -k "regex:k1_extremes|k2_filter" -s 6 -c 2 -o gpurun_out/prof_$c $CMD
  done
  CMD="python bench.py --config T4 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline"
  run ncu_launches_T4 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_T4.csv $CMD
  run ncu_full_T4 1200 ncu --set full --clock-control none --import-source on -k "regex:k1_extremes3|k2_filter3" -s 4 -c 2 -o gpurun_out/prof_T4 $CMD
fi
