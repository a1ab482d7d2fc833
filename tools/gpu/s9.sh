mkdir -p gpurun_out/s9
timeout 300 python tools/c1_stall.py 1e-12 1e-10 1e-9 1e-8 1e-7 1e-6 > gpurun_out/s9/c1_drop.txt 2>&1
timeout 600 python tools/ab_option.py --key drop_tol --values 1e-12 1e-8 1e-6 --nk 3 > gpurun_out/s9/ab_drop.txt 2>&1
