mkdir -p gpurun_out/s47
bash tools/build_variants.sh "t2n64m8:-DPC_XEX_TP=2 -DPC_XEX_NT=64 -DPC_XEX_MINB=8" "t4n128m5:-DPC_XEX_TP=4 -DPC_XEX_NT=128 -DPC_XEX_MINB=5" "t4n64m8:-DPC_XEX_TP=4 -DPC_XEX_NT=64 -DPC_XEX_MINB=8" > gpurun_out/s47/build.log 2>&1
for i in 1 2; do
echo "default $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s47/apply.txt
for v in t2n64m8 t4n128m5 t4n64m8; do
  echo "$v $(PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s47/apply.txt
done; done
