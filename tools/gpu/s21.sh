mkdir -p gpurun_out/s21
timeout 900 python tools/ab_option.py --key sticky_lock --values 0 1 --nk 3 > gpurun_out/s21/ab_sticky.txt 2>&1
timeout 900 python tools/ab_option.py --key start_noise --values 0.001 0.01 0.0001 --nk 3 > gpurun_out/s21/ab_noise.txt 2>&1
timeout 900 python tools/ab_option.py --key gram_refresh --values 16 0 --nk 3 > gpurun_out/s21/ab_refresh.txt 2>&1
timeout 900 python tools/ab_option.py --key p_restart --values 1 0 --nk 3 > gpurun_out/s21/ab_prestart.txt 2>&1
