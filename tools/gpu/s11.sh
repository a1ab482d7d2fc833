mkdir -p gpurun_out/s11
(OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 timeout 1500 python tests/diag/oracle_path_rate.py C2 --out gpurun_out/s11/oracle_path_c2.json > gpurun_out/s11/oracle_c2.log 2>&1; OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 timeout 1200 python tests/diag/oracle_path_rate.py C3 --k 5,8,24 --out gpurun_out/s11/oracle_path_c3.json > gpurun_out/s11/oracle_c3.log 2>&1) &
BG=$!
nproc > gpurun_out/s11/nproc.txt
timeout 300 python tools/verbose_c4.py 5 > gpurun_out/s11/verbose_c4.json 2>&1
for sh in "16 2 2" "16 2 0" "16 4 4" "16 6 6" "16 10 10"; do
  set -- $sh
  echo "b=$1 na=$2 np=$3 $(timeout 120 python tools/bench_block.py --n 128 --b $1 --na $2 --np $3 --which 1 --reps 10 2>&1 | tail -1)" >> gpurun_out/s11/gram_small.txt
done
timeout 120 python tools/apply_time.py C4 15 eps=sdd > gpurun_out/s11/apply_sdd.txt 2>&1
timeout 120 python tools/apply_time.py C4 15 >> gpurun_out/s11/apply_sdd.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s11/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/s11/pytest_gpu.log
wait $BG
