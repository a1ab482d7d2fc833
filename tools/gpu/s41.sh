mkdir -p gpurun_out/s41
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s41/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/s41/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s41/smoke.log 2>&1
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo --no-alt --no-cpu-baseline > gpurun_out/s41/bench_2rank_gloo.json 2> gpurun_out/s41/bench_2rank_gloo.err
