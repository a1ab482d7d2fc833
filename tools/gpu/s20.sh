mkdir -p gpurun_out/s20
for cfg in "--streams 2 --kbatch 1" "--streams 1 --kbatch 2" "--streams 2 --kbatch 2" "--streams 1 --kbatch 4"; do
  echo "$cfg $(timeout 900 python bench.py --steps 8 --warmup 4 --no-alt --no-cpu-baseline --e2e-steps 0 $cfg 2>/dev/null | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["value"], j["iters"])')" >> gpurun_out/s20/c4_modes.txt
done
