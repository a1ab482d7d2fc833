# Variant builds (var/<name>/libpcband.so, made with make BUILD=build/<name> LIB=var/<name>/libpcband.so
# EXTRA="-D...") timed by tools/bench_block.py against the default build, REPS rounds.
# usage (on the GPU box): VARIANTS="a b" WHICH="0 3" bash tools/vrun.sh
cd ${GRAFT_REPO_ROOT:-.}
for r in $(seq ${REPS:-2}); do
  echo "default $(python tools/bench_block.py --which ${WHICH:-0 3})"
  for v in $VARIANTS; do echo "$v $(PCBAND_LIB=$PWD/var/$v/libpcband.so python tools/bench_block.py --which ${WHICH:-0 3})"; done
done
