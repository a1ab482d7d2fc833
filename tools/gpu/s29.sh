mkdir -p gpurun_out/s29
bash tools/build_variants.sh "notwrec:-DPC_XEX_TWREC=0" > gpurun_out/s29/build.log 2>&1
for i in 1 2; do
echo "twrec $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s29/apply.txt
echo "notwrec $(PCBAND_LIB=$PWD/var/notwrec/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s29/apply.txt
done
echo "twrec plane2 $(timeout 120 python tools/apply_time.py C4 15 plane_fuse=1 2>&1 | tail -1)" >> gpurun_out/s29/apply.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s29/parity.log 2>&1; echo "rc $?" >> gpurun_out/s29/parity.log
