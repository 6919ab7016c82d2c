cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; lscpu > gpurun_out/lscpu.txt; free -g >> gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c5" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 300 python bench.py --config C2b --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2b.log 2>&1; echo b2=$? >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench_c5.log 2>&1; echo b5=$? >> gpurun_out/status.txt
