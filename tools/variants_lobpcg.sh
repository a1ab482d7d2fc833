# Tuning builds of libpcband (separate build dirs) timed on the LOBPCG by tools/ab_option.py, interleaved
# with the default build (REPS rounds) to see through run-to-run drift.
# usage: REPS=2 bash tools/variants_lobpcg.sh "name1:-DFLAG ..." ...
make -j16 >/dev/null 2>&1
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  make -j16 BUILD=build/$name LIB=build/$name/libpcband.so EXTRA="$flags" >/dev/null 2>&1 || echo "build $name failed"
done
for r in $(seq ${REPS:-2}); do
  echo "default $(python tools/ab_option.py --key profile --values 1 --nk 2 | cut -c1-900)"
  for spec in "$@"; do
    name=${spec%%:*}
    echo "$name $(PCBAND_LIB=$PWD/build/$name/libpcband.so python tools/ab_option.py --key profile --values 1 --nk 2 | cut -c1-900)"
  done
done
