mkdir -p gpurun_out/s39
bash tools/build_variants.sh "rrtime:-DPC_RR_TIMING" > gpurun_out/s39/build.log 2>&1
echo "C4 $(PCBAND_LIB=$PWD/var/rrtime/libpcband.so timeout 300 python tools/rr_phases.py C4 5 2>&1 | tail -1)" >> gpurun_out/s39/rr.txt
echo "C2 $(PCBAND_LIB=$PWD/var/rrtime/libpcband.so timeout 300 python tools/rr_phases.py C2 5 2>&1 | tail -1)" >> gpurun_out/s39/rr.txt
timeout 900 python bench.py --workload C2 --steps 24 --warmup 12 --kbatch 12 --streams 1 --no-alt --no-cpu-baseline --e2e-steps 12 > gpurun_out/s39/bench_c2.json 2> gpurun_out/s39/bench_c2.err
timeout 900 python bench.py --workload C3 --steps 12 --warmup 4 --kbatch 4 --streams 2 --no-alt --no-cpu-baseline --e2e-steps 4 > gpurun_out/s39/bench_c3.json 2> gpurun_out/s39/bench_c3.err
timeout 1500 python -m pytest tests/test_gpu_bands.py tests/test_gpu_parity.py -x -q > gpurun_out/s39/tests.log 2>&1; echo "rc $?" >> gpurun_out/s39/tests.log
timeout 900 python bench.py > gpurun_out/s39/bench.json 2> gpurun_out/s39/bench.err
