# round 2 (4t): the PASS1 streaming phase alone on the 512-thread launch (pa) and PASS1 with candidate
# tiles decided at once (pb) vs the inline build (m)
for cfg in "4" "4 --mode nearest"; do
  echo "pa skip2 cfg $cfg | $(SPIN_DEBUG_SKIP=2 SPIN_LIB_PATH=abbuild/pa/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-60)" >> gpurun_out/r4t_ab.txt
  for lib in m pb; do
    for sk in 0 2; do
      echo "$lib skip$sk cfg $cfg | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-60)" >> gpurun_out/r4t_ab.txt
    done
  done
done
cat gpurun_out/r4t_ab.txt
