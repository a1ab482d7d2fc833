mkdir -p gpurun_out/s10
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s10/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/s10/pytest_gpu.log
timeout 900 python bench.py --steps 4 --warmup 3 > gpurun_out/s10/bench.json 2> gpurun_out/s10/bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s10/smoke.log 2>&1; echo "rc $?" >> gpurun_out/s10/smoke.log
