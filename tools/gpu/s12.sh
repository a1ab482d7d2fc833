mkdir -p gpurun_out/s12
for sh in "16 6 6" "16 5 5" "16 7 7" "16 3 3" "16 8 8"; do
  set -- $sh
  echo "b=$1 na=$2 np=$3 $(timeout 120 python tools/bench_block.py --n 128 --b $1 --na $2 --np $3 --which 1 --reps 10 2>&1 | tail -1)" >> gpurun_out/s12/gram_small.txt
done
timeout 300 python tools/multik_time.py C2 --nk 8 --cols 10 > gpurun_out/s12/multik.txt 2>&1
timeout 300 python tools/multik_time.py C3 --nk 4 --cols 10 >> gpurun_out/s12/multik.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s12/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/s12/pytest_gpu.log
timeout 600 python bench.py --steps 4 --warmup 3 > gpurun_out/s12/bench.json 2> gpurun_out/s12/bench.err
