for lib in paper_2509_08574_b200/libkct.so build/libkct_fw*.so; do
  r=$(KCT_LIB_PATH=$lib timeout 120 python tools/kprof.py --reps 3 2>&1 | tail -1); echo "$lib $r"
done
