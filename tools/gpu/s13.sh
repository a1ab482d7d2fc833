mkdir -p gpurun_out/s13
for sh in "16 10 0" "16 10 10" "16 9 9" "16 8 8" "16 6 6" "16 5 5" "16 4 4" "16 3 3" "16 2 2" "16 1 1"; do
  set -- $sh
  for g in 0 1; do
    echo "b=$1 na=$2 np=$3 narrow=$g $(timeout 120 python tools/bench_block.py --n 128 --b $1 --na $2 --np $3 --which 1 --reps 10 --opt gram_narrow $g 2>&1 | tail -1)" >> gpurun_out/s13/gram.txt
  done
done
timeout 600 python tools/ab_option.py --key gram_narrow --values 0 1 --nk 3 > gpurun_out/s13/ab.txt 2>&1
