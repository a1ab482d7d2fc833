set -x
mkdir -p gpurun_out/s1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/s1/pytest_gpu.log
SAN=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $SAN --tool memcheck --leak-check no python tools/sanitize_run.py --plane > gpurun_out/s1/memcheck.log 2>&1; echo "rc $?" >> gpurun_out/s1/memcheck.log
timeout 900 $SAN --tool racecheck --racecheck-report analysis python tools/sanitize_run.py --quick > gpurun_out/s1/racecheck.log 2>&1; echo "rc $?" >> gpurun_out/s1/racecheck.log
timeout 900 $SAN --tool synccheck python tools/sanitize_run.py --quick > gpurun_out/s1/synccheck.log 2>&1; echo "rc $?" >> gpurun_out/s1/synccheck.log
timeout 600 python tests/diag/iter_compare.py --n 32 --nk 4 --which gpu --variants default,wguard_all,fullgram,guard3 > gpurun_out/s1/iter32.json 2> gpurun_out/s1/iter32.err
timeout 600 python tests/diag/iter_compare.py --n 64 --nk 4 --which gpu --variants default,wguard_all > gpurun_out/s1/iter64.json 2> gpurun_out/s1/iter64.err
