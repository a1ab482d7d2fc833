mkdir -p gpurun_out/s37
bash tools/build_variants.sh "rrtime:-DPC_RR_TIMING"  > gpurun_out/s37/build.log 2>&1
for v in rrtime; do
  echo "$v C4 $(PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 300 python tools/rr_phases.py C4 5 2>&1 | tail -1)" >> gpurun_out/s37/rr.txt
  echo "$v C2 $(PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 300 python tools/rr_phases.py C2 5 2>&1 | tail -1)" >> gpurun_out/s37/rr.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "jacobi" > gpurun_out/s37/eig.log 2>&1; echo "rc $?" >> gpurun_out/s37/eig.log
timeout 1500 python -m pytest tests/test_gpu_bands.py -x -q > gpurun_out/s37/bands.log 2>&1; echo "rc $?" >> gpurun_out/s37/bands.log
timeout 900 python tools/ab_option.py --workload C2 --key jacobi_tol --values 1e-16 --nk 6 > gpurun_out/s37/ab_c2.txt 2>&1
timeout 900 python tools/ab_option.py --workload C4 --key jacobi_tol --values 1e-16 --nk 2 > gpurun_out/s37/ab_c4.txt 2>&1
