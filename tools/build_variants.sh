# Build tuning variants of libpcband: var/<name>/libpcband.so (objects in /tmp/pcb_build/<name>).
# usage: bash tools/build_variants.sh "name1:-DFLAG=1 -DOTHER" "name2:..."
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  mkdir -p var/$name /tmp/pcb_build/$name
  make -j32 BUILD=/tmp/pcb_build/$name LIB=var/$name/libpcband.so EXTRA="$flags" > /tmp/pcb_build/$name/make.log 2>&1 || echo "build $name failed"
done
ls var/*/libpcband.so
