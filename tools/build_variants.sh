# Build tuning variants of libpcband: var/<name>/libpcband.so (objects in build/<name>).
# usage: bash tools/build_variants.sh "name1:-DFLAG=1 -DOTHER" "name2:..."
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  mkdir -p var/$name build/$name
  make -j32 BUILD=build/$name LIB=var/$name/libpcband.so EXTRA="$flags" > build/$name/make.log 2>&1 || echo "build $name failed"
done
ls var/*/libpcband.so
