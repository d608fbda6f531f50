for lib in paper_2509_08574_b200/libkct.so build/libkct_fm*.so; do
  for c in 2 3 4; do
    r=$(KCT_FWD_C=$c KCT_LIB_PATH=$lib timeout 120 python tools/kprof.py --reps 3 2>&1 | tail -1); echo "$lib C=$c $r"
  done
done
