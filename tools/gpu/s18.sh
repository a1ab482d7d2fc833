mkdir -p gpurun_out/s18
bash tools/build_variants.sh "tp4m1:-DPC_XEXG_MINB=1" "tp8m1:-DPC_XEXG_TP=8 -DPC_XEXG_MINB=1" "tp4z32:-DPC_XEXG_ZC=32" "tp2m2:-DPC_XEXG_TP=2" > gpurun_out/s18/build.log 2>&1
for v in tp4m1 tp8m1 tp4z32 tp2m2; do
  echo "$v $(PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 120 python tools/apply_time.py C4 15 eps=sdd 2>&1 | tail -1)" >> gpurun_out/s18/apply.txt
done
echo "default $(timeout 120 python tools/apply_time.py C4 15 eps=sdd 2>&1 | tail -1)" >> gpurun_out/s18/apply.txt
