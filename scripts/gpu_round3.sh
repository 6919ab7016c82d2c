#!/bin/bash
# 3D extension validation + measurement round (run under gpurun from the repo root).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/status3.txt
run() { local name=$1 t=$2; shift 2; timeout "$t" "$@" > "gpurun_out/$name.log" 2>&1; echo "$name=$?" >> gpurun_out/status3.txt; }
run pytest_gpu3 900 python -m pytest tests/test_gpu3.py -x -q
run bench_t4 600 python bench.py --config T4
run bench_t3 600 python bench.py --config T3 --no-cpu-baseline
run bench_t5 600 python bench.py --config T5 --no-cpu-baseline
run bench_t4_ref 600 python bench.py --config T4 --impl reference --steps 3 --warmup 1
if [ -z "$NO_NCU" ]; then
CMD="python bench.py --config T4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
run plain3 300 $CMD && run ncu3_launches 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv $CMD
run ncu3_full 1200 ncu --set full --clock-control none --import-source on -k "regex:k1_extremes3|k2_filter3" -s 2 -c 2 -o gpurun_out/prof3_t4 $CMD
fi
