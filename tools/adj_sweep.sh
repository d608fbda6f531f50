# A/B sweep of adjoint variants (tools/build_variant.sh) over brick heights.
#   BZS="64 96 128" tools/adj_sweep.sh build/libkct_a*.so
BZS=${BZS:-"96 128 192 256"}
for lib in "$@"; do
  for bz in $BZS; do
    r=$(KCT_ADJ_BZ=$bz KCT_LIB_PATH=$lib timeout 120 python tools/kprof.py --reps 3 2>&1 | tail -1)
    echo "$lib bz=$bz $r"
  done
done
