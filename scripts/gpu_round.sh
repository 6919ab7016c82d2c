#!/bin/bash
# GPU validation + measurement round (run under gpurun from the repo root).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/status.txt
run() { local name=$1 t=$2; shift 2; timeout "$t" "$@" > "gpurun_out/$name.log" 2>&1; echo "$name=$?" >> gpurun_out/status.txt; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
run smoke 300 python __graft_entry__.py smoke
run pytest_gpu 1800 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"}
run bench_c2b 300 python bench.py --config C2b --steps 50 --warmup 5 --no-cpu-baseline
run bench_c5 600 python bench.py
if [ -z "$NO_NCU" ]; then
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
run plain 300 $CMD && run ncu_launches 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD
run ncu_full 1200 ncu --set full --clock-control none --import-source on -k "regex:${NCU_REGEX:-k1_extremes|k2_filter}" -s ${NCU_SKIP:-4} -c ${NCU_COUNT:-2} -o gpurun_out/prof_c5 $CMD
fi
