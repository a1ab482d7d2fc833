mkdir -p gpurun_out/s5
for sh in "16 10 10" "16 10 0" "16 5 5" "16 16 16" "16 2 2" "16 7 7"; do
  set -- $sh
  for m in 1 2 3; do
    echo "b=$1 na=$2 np=$3 mode=$m $(timeout 120 python tools/bench_block.py --n 128 --b $1 --na $2 --np $3 --which 1 5 --reps 10 --opt gram_herm_mode $m 2>&1 | tail -1)" >> gpurun_out/s5/gram.txt 2>&1
  done
done
