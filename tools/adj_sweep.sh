for lib in build/libkct_*.so; do
  for bz in 96 128 192 256; do
    if [ $bz = 0 ]; then unset KCT_ADJ_BZ; else export KCT_ADJ_BZ=$bz; fi
    r=$(KCT_LIB_PATH=$lib timeout 120 python tools/kprof.py --reps 2 2>&1 | tail -1)
    echo "$lib bz=$bz $r"
  done
done
