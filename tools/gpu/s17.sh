mkdir -p gpurun_out/s17
timeout 900 python -m pytest tests/test_gpu_bands.py tests/test_gpu_parity.py -x -q -k "kbatch or apply_fourier or multi_k or full_size_n128 or precond" > gpurun_out/s17/tests.log 2>&1; echo "rc $?" >> gpurun_out/s17/tests.log
timeout 600 python tools/kbatch_time.py C2 24 > gpurun_out/s17/kbatch_c2.txt 2>&1
timeout 900 python tools/kbatch_time.py C3 12 > gpurun_out/s17/kbatch_c3.txt 2>&1
timeout 120 python tools/apply_time.py C4 15 eps=sdd > gpurun_out/s17/apply_sdd.txt 2>&1
timeout 120 python tools/apply_time.py C4 15 eps=sdd fuse_xex=0 >> gpurun_out/s17/apply_sdd.txt 2>&1
