# round-2 profile session: bench line, launch list, ncu --set full of the top kernels
mkdir -p gpurun_out/s14
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s14/smi.txt
timeout 900 python bench.py --steps 4 --warmup 3 > gpurun_out/s14/bench.json 2> gpurun_out/s14/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/s14/launches.csv python bench.py --steps 1 --warmup 3 --streams 1 --e2e-steps 0 --no-cpu-baseline --no-alt > gpurun_out/s14/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_tmap_kernel|gram_kernel|xex_kernel|fft_pass_kernel" -s 40 -c 8 -o gpurun_out/s14/lobpcg python tools/prof_lobpcg.py --maxit 4 > gpurun_out/s14/ncu_full.log 2>&1
