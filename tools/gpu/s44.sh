mkdir -p gpurun_out/s44
bash tools/build_variants.sh "t4n128:-DPC_XEX_TP=4 -DPC_XEX_NT=128 -DPC_XEX_MINB=4" "t8n128:-DPC_XEX_NT=128 -DPC_XEX_MINB=4" "t16n512:-DPC_XEX_TP=16 -DPC_XEX_NT=512 -DPC_XEX_MINB=1" > gpurun_out/s44/build.log 2>&1
for i in 1 2; do
echo "default $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s44/apply.txt
for v in t4n128 t8n128 t16n512; do
  echo "$v $(PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s44/apply.txt
done; done
