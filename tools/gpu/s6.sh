mkdir -p gpurun_out/s6
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "plane or full_size" > gpurun_out/s6/plane_tests.log 2>&1; echo "rc $?" >> gpurun_out/s6/plane_tests.log
for pf in 0 1 2; do
  echo "plane_fuse=$pf $(timeout 120 python tools/apply_time.py C4 15 plane_fuse=$pf 2>&1 | tail -1)" >> gpurun_out/s6/apply.txt
  echo "plane_fuse=$pf $(timeout 120 python tools/apply_time.py C4 10 plane_fuse=$pf 2>&1 | tail -1)" >> gpurun_out/s6/apply.txt
done
