# Gram block-shape variants (var/<name>/libpcband.so) x gram_ks, isolated launches at b=16, na=nP=10.
cd ${GRAFT_REPO_ROOT:-.}
for ks in 2 1; do
  echo "default ks$ks $(python tools/bench_block.py --which 1 --b 16 --opt gram_ks $ks)"
  for v in $VARIANTS; do echo "$v ks$ks $(PCBAND_LIB=$PWD/var/$v/libpcband.so python tools/bench_block.py --which 1 --b 16 --opt gram_ks $ks)"; done
done
