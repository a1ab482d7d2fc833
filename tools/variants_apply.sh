# Tuning builds of libpcband (separate build dirs) timed by tools/pass_time.py / tools/apply_time.py.
# usage: bash tools/variants_apply.sh "name1:-DFLAG ..." "name2:..."
make -j16 >/dev/null 2>&1
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  make -j16 BUILD=build/$name LIB=build/$name/libpcband.so EXTRA="$flags" >/dev/null 2>&1 || echo "build $name failed"
done
echo "default $(python tools/apply_time.py C4 15)"
for spec in "$@"; do
  name=${spec%%:*}
  echo "$name $(PCBAND_LIB=$PWD/build/$name/libpcband.so python tools/apply_time.py C4 15)"
done
