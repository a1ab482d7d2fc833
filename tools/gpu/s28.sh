mkdir -p gpurun_out/s28
bash tools/build_variants.sh "nohalo2:-DPC_XEX_HALO2=0" > gpurun_out/s28/build.log 2>&1
for i in 1 2; do
echo "halo2 $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s28/apply.txt
echo "nohalo2 $(PCBAND_LIB=$PWD/var/nohalo2/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s28/apply.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s28/parity.log 2>&1; echo "rc $?" >> gpurun_out/s28/parity.log
