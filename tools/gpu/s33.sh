mkdir -p gpurun_out/s33
bash tools/build_variants.sh "rrtime:-DPC_RR_TIMING" > gpurun_out/s33/build.log 2>&1
PCBAND_LIB=$PWD/var/rrtime/libpcband.so timeout 300 python tools/rr_phases.py C4 5 > gpurun_out/s33/rr_c4.json 2>&1
PCBAND_LIB=$PWD/var/rrtime/libpcband.so timeout 300 python tools/rr_phases.py C2 5 > gpurun_out/s33/rr_c2.json 2>&1
timeout 900 python tools/ab_option.py --workload C4 --key jacobi_tol --values 1e-16 1e-13 1e-11 --nk 2 > gpurun_out/s33/ab_jtol_c4.txt 2>&1
timeout 600 python tools/ab_option.py --workload C2 --key jacobi_tol --values 1e-16 1e-13 1e-11 --nk 6 > gpurun_out/s33/ab_jtol_c2.txt 2>&1
