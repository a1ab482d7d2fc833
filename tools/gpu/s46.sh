mkdir -p gpurun_out/s46
for i in 1 2; do echo "final $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s46/apply.txt; done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s46/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/s46/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s46/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s46/bench.json 2> gpurun_out/s46/bench.err
timeout 1500 python bench.py --workload C5 --steps 2 --warmup 3 --streams 1 --no-alt --no-cpu-baseline --e2e-steps 1 > gpurun_out/s46/bench_c5.json 2> gpurun_out/s46/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/s46/launches_bench.csv python bench.py --steps 1 --warmup 3 --streams 1 --e2e-steps 0 --no-cpu-baseline --no-alt > gpurun_out/s46/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_tmap|gram_kernel|xex_kernel|fft_pass_kernel|rr_kernel" -s 12 -c 11 -o gpurun_out/s46/lobpcg python tools/prof_lobpcg.py --maxit 12 > gpurun_out/s46/ncu_full.log 2>&1
