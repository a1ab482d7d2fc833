# Parity + timing of variant builds (var/<name>/libpcband.so): dense-oracle band tests and the
# isolated update launch.  usage (GPU box): VARIANTS="a b" bash tools/vtest.sh
cd ${GRAFT_REPO_ROOT:-.}
for v in $VARIANTS; do
  echo "== $v"
  PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 300 python -m pytest tests/test_gpu_bands.py -x -q -k "dense_oracle or option_variants or iterative" 2>&1 | tail -2
  PCBAND_LIB=$PWD/var/$v/libpcband.so python tools/bench_block.py --which ${WHICH:-3} 2>&1 | tail -1
done
