mkdir -p gpurun_out/s40
bash tools/build_variants.sh "kc8st4:-DPC_GRAM40_KC=8 -DPC_GRAM40_ST=4" "kc8st6:-DPC_GRAM40_KC=8 -DPC_GRAM40_ST=6" "kc16st3:-DPC_GRAM40_KC=16 -DPC_GRAM40_ST=3" "kc32st2:-DPC_GRAM40_KC=32 -DPC_GRAM40_ST=2" "kc32st3:-DPC_GRAM40_KC=32 -DPC_GRAM40_ST=3" > gpurun_out/s40/build.log 2>&1
for i in 1 2; do
echo "default $(timeout 120 python tools/bench_block.py --which 1 2>&1 | tail -1)" >> gpurun_out/s40/gram.txt
for v in kc8st4 kc8st6 kc16st3 kc32st2 kc32st3; do
  echo "$v $(PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 120 python tools/bench_block.py --which 1 2>&1 | tail -1)" >> gpurun_out/s40/gram.txt
done; done
