# session 2: post-refactor GPU tests + bench + iteration sweeps
mkdir -p gpurun_out/s2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/s2/pytest_gpu.log
timeout 600 python bench.py --steps 4 --warmup 3 > gpurun_out/s2/bench.json 2> gpurun_out/s2/bench.err
timeout 900 python tools/guard_sweep.py --workload C4 --kidx 4 20 36 --pairs 6,0 6,-1 4,-1 3,-1 2,-1 8,2 > gpurun_out/s2/guard.json 2> gpurun_out/s2/guard.err
