mkdir -p gpurun_out/s45
bash tools/build_variants.sh "oldshape:-DPC_XEX_TP=8 -DPC_XEX_NT=256 -DPC_XEX_MINB=2" > gpurun_out/s45/build.log 2>&1
for i in 1 2; do echo "new $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s45/apply.txt; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s45/parity.log 2>&1; echo "rc $?" >> gpurun_out/s45/parity.log
for v in new old; do
  if [ $v = old ]; then L=$PWD/var/oldshape/libpcband.so; else L=$PWD/paper_2511_17107_b200/libpcband.so; fi
  PCBAND_LIB=$L timeout 900 python bench.py --workload C2 --steps 24 --warmup 12 --kbatch 12 --streams 1 --no-alt --no-cpu-baseline --e2e-steps 0 > gpurun_out/s45/bench_c2_$v.json 2> gpurun_out/s45/bench_c2_$v.err
  PCBAND_LIB=$L timeout 900 python bench.py --workload C3 --steps 12 --warmup 4 --kbatch 4 --streams 2 --no-alt --no-cpu-baseline --e2e-steps 0 > gpurun_out/s45/bench_c3_$v.json 2> gpurun_out/s45/bench_c3_$v.err
done
