mkdir -p gpurun_out/s49
for s in 2 3 2 3; do
  echo "streams $s $(timeout 900 python bench.py --steps 6 --warmup 3 --streams $s --no-alt --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["clocks"]["sm_mhz"], d["iters"])')" >> gpurun_out/s49/streams.txt
done
