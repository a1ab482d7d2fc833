mkdir -p gpurun_out/s4
for sh in "16 10 10" "16 10 0" "16 5 5" "16 16 16" "16 2 2" "26 20 20" "12 6 6"; do
  set -- $sh
  echo "b=$1 na=$2 np=$3 $(timeout 120 python tools/bench_block.py --n 128 --b $1 --na $2 --np $3 --which 1 5 --reps 10 2>&1 | tail -1)" >> gpurun_out/s4/gram.txt 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_bands.py -x -q > gpurun_out/s4/bands.log 2>&1; echo "rc $?" >> gpurun_out/s4/bands.log
timeout 600 python -m pytest tests/test_gpu_bench.py -x -q > gpurun_out/s4/bench_test.log 2>&1; echo "rc $?" >> gpurun_out/s4/bench_test.log
timeout 600 python tools/ab_option.py --key gram_herm --values 0 1 --nk 3 > gpurun_out/s4/ab_gh.txt 2>&1
