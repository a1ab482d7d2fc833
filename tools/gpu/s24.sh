mkdir -p gpurun_out/s24
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "jacobi" > gpurun_out/s24/eig.log 2>&1; echo "rc $?" >> gpurun_out/s24/eig.log
timeout 1200 python -m pytest tests/test_gpu_bands.py -x -q > gpurun_out/s24/bands.log 2>&1; echo "rc $?" >> gpurun_out/s24/bands.log
timeout 600 python tools/ab_option.py --key rr_method --values 0 1 --nk 3 > gpurun_out/s24/ab_rr.txt 2>&1
timeout 600 python tools/kbatch_time.py C2 24 > gpurun_out/s24/kbatch_c2.txt 2>&1
