mkdir -p gpurun_out/s15
timeout 900 python -m pytest tests/test_gpu_bands.py -x -q -k "kbatch or c1_vacuum or dense_oracle" > gpurun_out/s15/tests.log 2>&1; echo "rc $?" >> gpurun_out/s15/tests.log
timeout 600 python tools/kbatch_time.py C2 16 > gpurun_out/s15/kbatch_c2.txt 2>&1
timeout 600 python tools/kbatch_time.py C3 8 > gpurun_out/s15/kbatch_c3.txt 2>&1
