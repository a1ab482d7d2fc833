mkdir -p gpurun_out/s31
bash tools/build_variants.sh "widespan:-DPC_ZSPAN_TIGHT=0" "bounds:-DPC_FFT_BOUNDS=1" > gpurun_out/s31/build.log 2>&1
python - > gpurun_out/s31/occ.txt 2>&1 <<'PY'
import ctypes, torch
torch.zeros(1, device="cuda")
print(torch.cuda.get_device_properties(0))
PY
for i in 1 2; do
echo "tight $(timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s31/apply.txt
echo "widespan $(PCBAND_LIB=$PWD/var/widespan/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s31/apply.txt
echo "bounds $(PCBAND_LIB=$PWD/var/bounds/libpcband.so timeout 120 python tools/apply_time.py C4 15 2>&1 | tail -1)" >> gpurun_out/s31/apply.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s31/parity.log 2>&1; echo "rc $?" >> gpurun_out/s31/parity.log
