mkdir -p gpurun_out/s19
timeout 900 python bench.py --workload C2 --steps 24 --warmup 12 --kbatch 12 --streams 1 --no-alt --no-cpu-baseline --e2e-steps 12 > gpurun_out/s19/bench_c2.json 2> gpurun_out/s19/bench_c2.err
timeout 900 python bench.py --workload C3 --steps 12 --warmup 4 --kbatch 4 --streams 2 --no-alt --no-cpu-baseline --e2e-steps 4 > gpurun_out/s19/bench_c3.json 2> gpurun_out/s19/bench_c3.err
timeout 1500 python bench.py --workload C5 --steps 2 --warmup 1 --streams 1 --no-alt --no-cpu-baseline --e2e-steps 1 > gpurun_out/s19/bench_c5.json 2> gpurun_out/s19/bench_c5.err
