mkdir -p gpurun_out/s27
bash tools/build_variants.sh "nocols:-DPC_XEX_COLS=0" > gpurun_out/s27/build.log 2>&1
for i in 1 2; do
echo "cols $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s27/apply.txt
echo "nocols $(PCBAND_LIB=$PWD/var/nocols/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s27/apply.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s27/parity.log 2>&1; echo "rc $?" >> gpurun_out/s27/parity.log
