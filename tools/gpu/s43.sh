mkdir -p gpurun_out/s43
for i in 1 2; do echo "final $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s43/apply.txt; done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/s43/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/s43/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s43/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s43/bench.json 2> gpurun_out/s43/bench.err
