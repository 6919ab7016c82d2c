#!/bin/bash
# Round-2 GPU session (run under gpurun from the repo root).  STEPS selects
# what runs (space-separated): smoke pytest bench_c5 bench_cfgs ncu_c5 ...
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; : > gpurun_out/status.txt
run() { local name=$1 t=$2; shift 2; local t0=$(date +%s); timeout "$t" "$@" > "gpurun_out/$name.log" 2>&1; echo "$name=$? $(( $(date +%s) - t0 ))s" >> gpurun_out/status.txt; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt
python -c "import paper_1405_3454_b200.build as b, synth.cuda as s, oracle as o; b.build(); s.build(); o.build()" > gpurun_out/build.log 2>&1
for s in ${STEPS:-smoke pytest bench_c5}; do
  case $s in
    smoke) run smoke 300 python __graft_entry__.py smoke ;;
    pytest) run pytest_gpu 1800 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} ;;
    pytest_not_slow) run pytest_gpu 1800 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-not c5}" ;;
    bench_c5) run bench_c5 600 python bench.py ;;
    bench_c5_quick) run bench_c5 600 python bench.py --no-e2e --no-cpu-baseline ;;
    bench_cfgs) for c in C2a C2b C3 C4 C4e0; do run bench_$c 600 python bench.py --config $c --no-cpu-baseline; done ;;
    ncu_c5)
      CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
      run ncu_launches 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $CMD
      run ncu_full 1200 ncu --set full --clock-control none --import-source on -k "regex:${NCU_REGEX:-k1_extremes|k2_filter}" -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-3} -o gpurun_out/prof_c5 $CMD ;;
    custom) run custom ${CUSTOM_T:-600} bash -c "$CUSTOM" ;;
  esac
done
