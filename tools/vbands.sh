# Variant builds (var/<name>/libpcband.so): full band-solver GPU tests and C4 throughput (6 k-points).
# usage (GPU box): VARIANTS="a b" bash tools/vbands.sh
cd ${GRAFT_REPO_ROOT:-.}
for v in $VARIANTS; do
  echo "== $v"
  PCBAND_LIB=$PWD/var/$v/libpcband.so timeout 600 python -m pytest tests/test_gpu_bands.py -q 2>&1 | tail -3
  PCBAND_LIB=$PWD/var/$v/libpcband.so python tools/conc_sweep.py --nk 6 --fracs 1 --streams 2 2>&1 | tail -1
done
