mkdir -p gpurun_out/s23
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s23/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/s23/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s23/smoke.log 2>&1; echo "rc $?" >> gpurun_out/s23/smoke.log
timeout 900 python bench.py --steps 4 --warmup 3 > gpurun_out/s23/bench.json 2> gpurun_out/s23/bench.err
timeout 900 python bench.py --workload C2 --steps 24 --warmup 12 --kbatch 12 --streams 1 --no-alt --no-cpu-baseline --e2e-steps 12 > gpurun_out/s23/bench_c2.json 2> gpurun_out/s23/bench_c2.err
