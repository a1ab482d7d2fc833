mkdir -p gpurun_out/s32
for i in 1 2; do echo "default $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s32/apply.txt; done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s32/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/s32/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s32/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s32/bench.json 2> gpurun_out/s32/bench.err
timeout 900 python bench.py --workload C2 --steps 24 --warmup 12 --kbatch 12 --streams 1 --no-alt --no-cpu-baseline --e2e-steps 12 > gpurun_out/s32/bench_c2.json 2> gpurun_out/s32/bench_c2.err
timeout 900 python bench.py --workload C3 --steps 12 --warmup 4 --kbatch 4 --streams 2 --no-alt --no-cpu-baseline --e2e-steps 4 > gpurun_out/s32/bench_c3.json 2> gpurun_out/s32/bench_c3.err
timeout 1500 python bench.py --workload C5 --steps 2 --warmup 3 --streams 1 --no-alt --no-cpu-baseline --e2e-steps 1 > gpurun_out/s32/bench_c5.json 2> gpurun_out/s32/bench_c5.err
