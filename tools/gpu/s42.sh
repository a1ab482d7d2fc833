mkdir -p gpurun_out/s42
bash tools/build_variants.sh "notwrec:-DPC_FFT_TWREC=0" > gpurun_out/s42/build.log 2>&1
for i in 1 2; do
echo "twrec $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s42/apply.txt
echo "notwrec $(PCBAND_LIB=$PWD/var/notwrec/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s42/apply.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s42/parity.log 2>&1; echo "rc $?" >> gpurun_out/s42/parity.log
