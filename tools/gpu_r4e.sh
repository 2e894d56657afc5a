# round 2 (4e): PASS1 forced on the 512-thread launch: filter-only time vs the inline build
for lib in p1 q2; do
  for cfg in "4"; do
    for sk in 0 1 2; do
    echo "$lib skip$sk cfg $cfg | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4e_ab.txt
    done
  done
done
cat gpurun_out/r4e_ab.txt
