cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; : > gpurun_out/status.txt
run() { local name=$1 t=$2; shift 2; local t0=$(date +%s); timeout "$t" "$@" > "gpurun_out/$name.log" 2>&1; echo "$name=$? $(( $(date +%s) - t0 ))s" >> gpurun_out/status.txt; }
python -c "import paper_1405_3454_b200.build as b, synth.cuda as s, oracle as o; b.build(); s.build(); o.build()" > gpurun_out/build.log 2>&1
run pytest_gpu 2400 python -m pytest tests -m gpu -x -q
run smoke 300 python __graft_entry__.py smoke
run bench_T4 900 python bench.py --config T4
run bench_T3 900 python bench.py --config T3 --no-cpu-baseline
run bench_T5 900 python bench.py --config T5 --no-cpu-baseline
run bench_C5 900 python bench.py
CMD="python bench.py --config T4 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline"
run ncu_launches_T4 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_T4.csv $CMD
run ncu_full_T4 1200 ncu --set full --clock-control none --import-source on -k "regex:k1_extremes3|k2_filter3" -s 4 -c 2 -o gpurun_out/prof_T4 $CMD
