mkdir -p gpurun_out/s26
bash tools/build_variants.sh "nofuse:-DPC_XEX_FUSE=0" > gpurun_out/s26/build.log 2>&1
for i in 1 2; do
echo "fused $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s26/apply.txt
echo "nofuse $(PCBAND_LIB=$PWD/var/nofuse/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s26/apply.txt
done
echo "fused sdd $(timeout 120 python tools/apply_time.py C4 15 eps=sdd 2>&1 | tail -1)" >> gpurun_out/s26/apply.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s26/parity.log 2>&1; echo "rc $?" >> gpurun_out/s26/parity.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/s26/bench.json 2> gpurun_out/s26/bench.err
