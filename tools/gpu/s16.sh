mkdir -p gpurun_out/s16
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_tmap|gram_kernel|xex_kernel|fft_pass_kernel" -s 12 -c 10 -o gpurun_out/s16/lobpcg python tools/prof_lobpcg.py --maxit 12 > gpurun_out/s16/ncu_full.log 2>&1
timeout 600 python tools/kbatch_time.py C2 24 > gpurun_out/s16/kbatch_c2.txt 2>&1
timeout 900 python tools/kbatch_time.py C3 12 > gpurun_out/s16/kbatch_c3.txt 2>&1
