mkdir -p gpurun_out/s48
bash tools/build_variants.sh "zt4:-DPC_ZTP=4" "zt16:-DPC_ZTP=16" > gpurun_out/s48/build.log 2>&1
for i in 1 2; do
echo "default $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s48/apply.txt
for v in zt4 zt16; do
  echo "$v $(PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s48/apply.txt
done; done
