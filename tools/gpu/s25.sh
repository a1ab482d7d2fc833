mkdir -p gpurun_out/s25
bash tools/build_variants.sh "split2:-DPC_XEX_SPLIT=1" "split3:-DPC_XEX_SPLIT=1 -DPC_XEX_MINB=3" "split4:-DPC_XEX_SPLIT=1 -DPC_XEX_MINB=3 -DPC_XEX_TP=4 -DPC_XEX_NT=128" > gpurun_out/s25/build.log 2>&1
grep -h "xex_kernel" -A0 gpurun_out/s25/build.log | head -3
for v in split2 split3 split4; do
  echo "$v $(PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s25/apply.txt
  PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "apply_fourier or full_size_n128 or fused_xex" > gpurun_out/s25/parity_$v.log 2>&1; echo "rc $?" >> gpurun_out/s25/parity_$v.log
done
echo "default $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s25/apply.txt
for v in split2 split3; do cuobjdump -res-usage var/$v/libpcband.so 2>/dev/null | grep -A1 "xex_kernelILi128ELi1" | tail -1 >> gpurun_out/s25/regs.txt; done
