mkdir -p gpurun_out/s36
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rr_kernel" -s 10 -c 2 -o gpurun_out/s36/rr python tools/prof_lobpcg.py --maxit 14 > gpurun_out/s36/ncu.log 2>&1
